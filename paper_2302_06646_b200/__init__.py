"""paper_2302_06646_b200 — B200-native FlashButterfly long convolution.

A drop-in for the reference longconv hot path (regularized_long_conv and its
backward, conv through the butterfly / three-pass engines, the learned
butterfly): CUDA kernels for sm_100a behind the C ABI in
include/flashbutterfly.h, with this package as the host-side mirror of the
reference interface.
"""
from .longconv import (  # noqa: F401
    ConvMode,
    Engine,
    HostRunner,
    InitKind,
    LongConvPlan,
    RegularizationConfig,
    SmoothDomain,
    init_kernels,
    long_conv,
    regularized_long_conv,
    regularized_long_conv_backward,
)
from ._lib import DimensionError, FBError, PlanError  # noqa: F401
from .learned import (  # noqa: F401
    LearnedButterflyPlan,
    LearnedLongConvPlan,
    learned_butterfly,
    learned_long_conv,
)

__all__ = [
    "ConvMode", "Engine", "HostRunner", "InitKind", "LongConvPlan", "init_kernels", "RegularizationConfig", "SmoothDomain", "long_conv",
    "regularized_long_conv", "regularized_long_conv_backward", "DimensionError", "FBError",
    "PlanError", "LearnedButterflyPlan", "learned_butterfly", "LearnedLongConvPlan", "learned_long_conv",
]
