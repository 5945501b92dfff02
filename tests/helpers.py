"""Shared helpers for GPU parity tests: reference-RNG inputs rounded to the
I/O dtype, fed identically to the CUDA path and the fp64 oracle."""
from __future__ import annotations

import numpy as np
import torch

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2, torch.float16: 2e-2}  # north_star bars


def rounded(x: np.ndarray, dtype: torch.dtype):
    """(torch tensor on cuda in dtype, the same values as fp64 numpy)."""
    t = torch.tensor(x, dtype=torch.float64).to(dtype)
    return t.cuda(), t.double().numpy()


def layer_inputs(lc, B, H, N, dtype, seeds=(1, 2, 3), kind=1):
    u = lc.signal_batch(seeds[0], B, H, N)
    dy = lc.signal_batch(seeds[1], B, H, N)
    K, D = lc.init_kernels(kind, H, N, seeds[2])
    tu, u64 = rounded(u, dtype)
    tdy, dy64 = rounded(dy, dtype)
    tK, K64 = rounded(K, torch.float32)
    tD, D64 = rounded(D, torch.float32)
    return dict(tu=tu, tdy=tdy, tK=tK, tD=tD, u=u64, dy=dy64, K=K64, D=D64)


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().double().cpu().numpy()
