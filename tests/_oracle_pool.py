"""Per-head oracle workers for the full-configuration parity tests
(tests/test_gpu_full.py).  Test infrastructure only: imports numpy and the
oracle, never torch, so a `spawn` process pool can run one head per task on
every host core.

Inputs follow SURVEY.md §8(c) (the reference RNG, rng.cpp:57-69):
u[b,h,:] = standard_normal_draws(SeededRng(1).child(b*H+h), N), dy with seed 2;
the 16-bit product sees those values rounded to bf16, so the oracle runs on
the same rounded values."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.oracle import LcOracle  # noqa: E402

_LC = None


def _lc():
    global _LC
    if _LC is None:
        _LC = LcOracle()
    return _LC


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round to bfloat16 (nearest even); the raw 16-bit patterns."""
    f = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (f + np.uint32(0x7FFF) + ((f >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def bf16_value(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def layer_head(args):
    """One head of the layer: reference-RNG signals (bf16-rounded), then the
    fp64 regularizers, forward, backward and regularizer chain rule."""
    h, B, H, N, K_h, D_h, lam, p = args
    lc = _lc()
    ub = np.stack([bf16_bits(lc.normal_draws(1, b * H + h, N)) for b in range(B)])
    gb = np.stack([bf16_bits(lc.normal_draws(2, b * H + h, N)) for b in range(B)])
    u = bf16_value(ub)[:, None, :]
    dy = bf16_value(gb)[:, None, :]
    K = K_h[None, :]
    D = np.array([D_h])
    Kbar = lc.regularize_bank(K, lam, p)
    y = lc.long_conv_forward(u, Kbar, D)
    du, dKbar, dD = lc.long_conv_backward(u, dy, Kbar, D)
    dK = lc.regularizer_backward(K, lam, p, dKbar)
    return (h, ub, gb, y[:, 0].astype(np.float32), du[:, 0].astype(np.float32),
            dK[0], float(dD[0]))


def learned_head(args):
    """One head of the learned butterfly: blocks =
    from_plan(build_plan(n, 16)) + 0.1 (N + iN) from SeededRng(4).child(h)
    (draws interleaved re, im per entry); x, g complex normal from seeds 5 and
    6, stream b*H + h, interleaved re, im; x and g bf16-rounded."""
    h, B, H, n, r = args
    lc = _lc()
    base = lc.learned_init(n, r)
    d = lc.normal_draws(4, h, 2 * base.size)
    blocks = base + 0.1 * (d[0::2] + 1j * d[1::2])
    xb = np.stack([bf16_bits(lc.normal_draws(5, b * H + h, 2 * n)) for b in range(B)])
    gb = np.stack([bf16_bits(lc.normal_draws(6, b * H + h, 2 * n)) for b in range(B)])
    xs, gs = bf16_value(xb), bf16_value(gb)
    ys, dxs, db = [], [], 0
    for b in range(B):
        x = xs[b, 0::2] + 1j * xs[b, 1::2]
        g = gs[b, 0::2] + 1j * gs[b, 1::2]
        ys.append(lc.learned_forward(blocks, x, r))
        dbb, dx = lc.learned_gradients(blocks, x, g, r)
        dxs.append(dx)
        db = db + dbb
    return (h, blocks, xb, gb, np.array(ys).astype(np.complex64), np.array(dxs).astype(np.complex64),
            db)
