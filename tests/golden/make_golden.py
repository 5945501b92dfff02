"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Every array in the fixtures is an output of the reference library itself
(through oracle/ref_capi.cpp), on inputs drawn with the reference's own
SeededRng streams.  tests/test_oracle.py pins our C
restatement (oracle/lc_oracle.c) against these files, so the restatement is
checked even on machines without /root/reference.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import RefOracle  # noqa: E402

OUT = Path(__file__).resolve().parent
LAM, P = 0.003, 1  # SURVEY.md §8d (lambda from PAPER.md:1803)


def layer_case(ref, B, H, N, causal=True, rate=0.0, training=False, seed=0, engines=(1,)):
    u = ref.signal_batch(1, B, H, N)
    dy = ref.signal_batch(2, B, H, N)
    K, D = ref.init_kernels(1, H, N, 3)
    out = dict(u=u, dy=dy, K=K, D=D, lam=LAM, p=P, rate=rate, training=int(training),
               seed=seed, causal=int(causal))
    Kbar = ref.regularize_bank(K, LAM, P, rate, 0, seed, training)
    out["Kbar"] = Kbar
    for e in engines:
        out[f"y_engine{e}"] = ref.regularized_long_conv(u, K, D, LAM, P, rate, 0, seed,
                                                        causal=causal, training=training,
                                                        engine=e)
    if causal:
        du, dKbar, dD = ref.long_conv_backward(u, dy, Kbar, D)
        out.update(du=du, dKbar=dKbar, dD=dD)
        out["dK"] = ref.regularizer_backward(K, LAM, P, dKbar, rate, seed, training)
    return out


def main():
    ref = RefOracle()
    rng = np.random.default_rng(0)
    cases = {}
    # config 1: B=1 H=1 N=1024 causal, fwd + bwd, all three engines
    cases["layer_b1h1n1024"] = layer_case(ref, 1, 1, 1024, engines=(0, 1, 2))
    # odd batch, several heads, causal
    cases["layer_b3h4n256"] = layer_case(ref, 3, 4, 256, engines=(0, 1, 2))
    # circular mode
    cases["layer_b2h2n128_circ"] = layer_case(ref, 2, 2, 128, causal=False, engines=(0, 1, 2))
    # training-mode dropout (rate 0.2, seed 7)
    cases["layer_b2h3n64_drop"] = layer_case(ref, 2, 3, 64, rate=0.2, training=True, seed=7,
                                             engines=(0, 1))
    # transforms
    x = ref.signal_batch(5, 1, 1, 2 * 8192).reshape(-1)
    xc = x[0::2] + 1j * x[1::2]
    cases["apply_plan_8192"] = dict(x=xc, fwd=ref.apply_plan(xc), inv=ref.apply_plan(xc, inverse=True),
                                    factors=np.array(ref.plan_factors(8192)))
    xs = xc[:96]
    cases["apply_plan_96_r16"] = dict(x=xs, fwd=ref.apply_plan(xs), factors=np.array(ref.plan_factors(96)))
    # three-pass circular conv n=4096, l=256, m=16 (and the d_k layout)
    n, l, m = 4096, 256, 16
    u = xc[:n]
    k = xc[n:2 * n]
    cases["three_pass_4096"] = dict(u=u, k=k, l=l, m=m, y=ref.conv_three_pass(u, k, l, m),
                                    dk=ref.three_pass_dk(k, l, m), sweeps=ref.last_sweeps)
    # real packed, both modes
    ur, kr = x[:512], x[512:1024]
    cases["real_packed_512"] = dict(u=ur, k=kr, causal=ref.conv_real_packed(ur, kr, True),
                                    circular=ref.conv_real_packed(ur, kr, False))
    # learned butterfly n=1024 r=16 ([16,16,4]) with perturbed blocks
    n = 1024
    bl = ref.learned_init(n, 16)
    pert = 0.1 * (rng.standard_normal(bl.size) + 1j * rng.standard_normal(bl.size))
    blocks = bl + pert
    xl = xc[:n]
    gl = xc[n:2 * n]
    db, dx = ref.learned_gradients(blocks, xl, gl, 16)
    cases["learned_1024"] = dict(blocks=blocks, x=xl, g=gl, y=ref.learned_forward(blocks, xl, 16),
                                 dblocks=db, dx=dx, init=bl)
    n = 64
    bl = ref.learned_init(n, 4)
    blocks = bl + 0.1 * (rng.standard_normal(bl.size) + 1j * rng.standard_normal(bl.size))
    db, dx = ref.learned_gradients(blocks, xc[:n], xc[n:2 * n], 4)
    cases["learned_64_r4"] = dict(blocks=blocks, x=xc[:n], g=xc[n:2 * n],
                                  y=ref.learned_forward(blocks, xc[:n], 4), dblocks=db, dx=dx)
    # regularizers incl. smooth_frequency
    kk = ref.signal_batch(9, 1, 1, 64).reshape(-1)
    cases["regularizers_64"] = dict(k=kk, squash=ref.squash(kk, 0.2), smooth=ref.smooth(kk, 2),
                                    smooth_freq=ref.smooth_frequency(kk, 2))
    # rng streams
    cases["rng"] = dict(normal=ref.normal_draws(1, 0, 16), uniform=ref.uniform_draws(7, 3, 16))
    for name, d in cases.items():
        np.savez_compressed(OUT / f"{name}.npz", **{k: np.asarray(v) for k, v in d.items()})
        print(name, sum(np.asarray(v).nbytes for v in d.values()))


if __name__ == "__main__":
    main()
