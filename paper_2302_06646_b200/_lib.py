"""ctypes binding of the C ABI in include/flashbutterfly.h.

Loads the in-tree ``libflashbutterfly.so``.  There is no fallback: if the
library is missing or no CUDA device is present, every call raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# FB_LIB_PATH: experiment builds only (e.g. an instrumented library); the
# product always loads the in-tree libflashbutterfly.so
LIB_PATH = Path(os.environ.get("FB_LIB_PATH") or Path(__file__).resolve().parent / "libflashbutterfly.so")

FB_OK, FB_ERR_DIM, FB_ERR_PLAN, FB_ERR_CUDA, FB_ERR_NCCL, FB_ERR_ARG, FB_ERR_UNSUPPORTED = range(7)
FB_MODE_CIRCULAR, FB_MODE_CAUSAL = 0, 1
FB_ENGINE_AUTO, FB_ENGINE_SINGLE, FB_ENGINE_THREE, FB_ENGINE_SINGLE_SIMT = 0, 1, 2, 3
FB_F32, FB_BF16, FB_F16 = 0, 1, 2
FB_SMOOTH_TIME, FB_SMOOTH_FREQUENCY = 0, 1

# Every symbol include/flashbutterfly.h declares (tests check the export list).
EXPORTED = [
    "fb_plan_create", "fb_plan_destroy", "fb_plan_get_info", "fb_kernel_prep", "fb_plan_copy_kbar",
    "fb_workspace_size", "fb_fwd", "fb_bwd", "fb_learned_plan_create", "fb_learned_plan_destroy",
    "fb_learned_plan_factors", "fb_learned_plan_engine", "fb_learned_workspace_size", "fb_learned_fwd", "fb_learned_bwd",
    "fb_last_error", "fb_version", "fb_host_runner_create", "fb_host_runner_destroy",
    "fb_host_runner_chunk_heads", "fb_host_runner_run", "fb_saved_size", "fb_fwd_save",
    "fb_bwd_saved", "fb_shard_plan_create", "fb_shard_plan_destroy", "fb_shard_plan_dims",
    "fb_shard_columns", "fb_shard_rows", "fb_plan_profile_events", "fb_dft_plan_create",
    "fb_dft_plan_destroy", "fb_dft_plan_factors", "fb_dft_workspace_size", "fb_dft", "fb_conv_rows",
    "fb_conv_rows_spectrum", "fb_init_kernels", "fb_shard_rows_pairs", "fb_shard_rows_bwd",
    "fb_shard_stage",
    "fb_shard_columns_from_signals", "fb_shard_columns_to_signals", "fb_lconv_plan_create",
    "fb_lconv_plan_destroy", "fb_lconv_plan_dims", "fb_lconv_workspace_size", "fb_lconv_fwd", "fb_lconv_bwd",
]


class FBError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[fb error {code}] {msg}")
        self.code = code


class DimensionError(FBError, ValueError):
    """FB_ERR_DIM — mirrors longconv::DimensionError (errors.hpp:10-12)."""


class PlanError(FBError, ValueError):
    """FB_ERR_PLAN — mirrors longconv::PlanError (errors.hpp:15-17)."""


class RegConfig(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("smooth_width", C.c_int64),
                ("dropout_rate", C.c_double), ("smooth_domain", C.c_int), ("seed", C.c_uint64)]


class PlanInfo(C.Structure):
    _fields_ = [("N", C.c_int64), ("H", C.c_int64), ("n", C.c_int64), ("l", C.c_int64),
                ("m", C.c_int64), ("engine", C.c_int), ("dtype", C.c_int), ("mode", C.c_int),
                ("tensor_cores", C.c_int)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(
                f"{LIB_PATH} is missing — build it with `python -m paper_2302_06646_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        vp, i64, sz = C.c_void_p, C.c_int64, C.c_size_t
        L.fb_plan_create.argtypes = [C.POINTER(vp), i64, i64, C.c_int, C.c_int, C.c_int, C.c_int]
        L.fb_plan_destroy.argtypes = [vp]
        L.fb_plan_get_info.argtypes = [vp, C.POINTER(PlanInfo)]
        L.fb_kernel_prep.argtypes = [vp, vp, vp, C.POINTER(RegConfig), C.c_int, vp]
        L.fb_plan_copy_kbar.argtypes = [vp, vp, vp]
        L.fb_workspace_size.argtypes = [vp, i64]
        L.fb_workspace_size.restype = sz
        L.fb_fwd.argtypes = [vp, vp, vp, i64, vp, vp]
        L.fb_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, vp, vp]
        L.fb_learned_plan_create.argtypes = [C.POINTER(vp), i64, i64, i64, C.c_int, C.c_int]
        L.fb_learned_plan_destroy.argtypes = [vp]
        L.fb_learned_plan_factors.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
        L.fb_learned_plan_engine.argtypes = [vp, C.POINTER(C.c_int)]
        L.fb_learned_workspace_size.argtypes = [vp, i64]
        L.fb_learned_workspace_size.restype = sz
        L.fb_learned_fwd.argtypes = [vp, vp, vp, vp, i64, vp, vp]
        L.fb_learned_bwd.argtypes = [vp, vp, vp, vp, vp, vp, i64, vp, vp]
        L.fb_shard_plan_create.argtypes = [C.POINTER(vp), i64, C.c_int]
        L.fb_shard_plan_destroy.argtypes = [vp]
        L.fb_shard_plan_dims.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.fb_shard_columns.argtypes = [vp, vp, vp, i64, i64, i64, C.c_int, vp]
        L.fb_shard_rows.argtypes = [vp, vp, vp, vp, i64, i64, C.c_int, C.c_float, vp]
        L.fb_saved_size.argtypes = [vp, i64]
        L.fb_saved_size.restype = sz
        L.fb_fwd_save.argtypes = [vp, vp, vp, vp, i64, vp, vp]
        L.fb_bwd_saved.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, i64, vp, vp]
        L.fb_host_runner_create.argtypes = [C.POINTER(vp), i64, i64, C.c_int, C.c_int, C.c_int,
                                             C.c_int, i64, i64]
        L.fb_host_runner_destroy.argtypes = [vp]
        L.fb_host_runner_chunk_heads.argtypes = [vp]
        L.fb_host_runner_chunk_heads.restype = i64
        L.fb_host_runner_run.argtypes = [vp, C.POINTER(RegConfig), C.c_int, vp, vp, vp, vp, vp,
                                         vp, vp, vp, vp]
        L.fb_plan_profile_events.argtypes = [vp, C.c_int, vp, vp]
        L.fb_dft_plan_create.argtypes = [C.POINTER(vp), i64, i64, C.c_int]
        L.fb_dft_plan_destroy.argtypes = [vp]
        L.fb_dft_plan_factors.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.fb_dft_workspace_size.argtypes = [vp, i64, i64]
        L.fb_dft_workspace_size.restype = sz
        L.fb_dft.argtypes = [vp, vp, vp, i64, C.c_int, vp, vp]
        L.fb_conv_rows.argtypes = [vp, vp, vp, vp, i64, i64, i64, C.c_int, vp, vp]
        L.fb_conv_rows_spectrum.argtypes = [vp, vp, vp, vp, i64, i64, i64, C.c_int, vp, vp]
        L.fb_shard_rows_pairs.argtypes = [vp, vp, vp, i64, i64, i64, vp]
        L.fb_shard_rows_bwd.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, vp]
        L.fb_shard_columns_from_signals.argtypes = [vp, vp, C.c_int, vp, i64, i64, i64, i64, i64, vp]
        L.fb_shard_columns_to_signals.argtypes = [vp, vp, vp, C.c_int, vp, vp, i64, i64, i64, i64, i64, vp]
        L.fb_shard_stage.argtypes = [vp, vp, i64, i64, i64, C.c_int, C.c_int, vp]
        L.fb_lconv_plan_create.argtypes = [C.POINTER(vp), i64, i64, i64, C.c_int, C.c_int]
        L.fb_lconv_plan_destroy.argtypes = [vp]
        L.fb_lconv_plan_dims.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.fb_lconv_workspace_size.argtypes = [vp, i64]
        L.fb_lconv_workspace_size.restype = sz
        L.fb_lconv_fwd.argtypes = [vp] * 7 + [i64, vp, vp]
        L.fb_lconv_bwd.argtypes = [vp] * 12 + [i64, vp, vp]
        L.fb_init_kernels.argtypes = [C.c_int, i64, i64, C.c_uint64, vp, vp, vp, vp, C.c_int, vp]
        L.fb_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == FB_OK:
        return
    msg = lib().fb_last_error().decode()
    cls = {FB_ERR_DIM: DimensionError, FB_ERR_PLAN: PlanError}.get(rc, FBError)
    raise cls(rc, msg)
