"""BASELINE config 5-4M (N = 4,194,304) against the fp64 oracle.

One channel pair (B = 2, H = 1) at the full sequence length, inputs rounded
to bf16 (so the same fp64 values feed the fp32 runs, the bf16 run and the
oracle, computed once for the module):

* the single-GPU three-pass plan (n = 8M = l 8192 x m 1024: big-column
  passes 1/3, rows on tcgen05 for bf16), fp32 at 1e-5 and bf16 at 2e-2;
* the sequence-sharded four-step (seqshard: fb_shard_columns /
  fb_shard_rows, regularizer and its chain rule on the sharded layout) at
  world 1 on the GPU, fp32 at 1e-5, forward + backward down to dK.
"""
import numpy as np
import pytest
import torch

from helpers import to_np
from oracle.oracle import rel_l2

pytestmark = pytest.mark.gpu

fb = pytest.importorskip("paper_2302_06646_b200")

N4M = 1 << 22
LAM, P = 0.003, 1


@pytest.fixture(scope="module")
def case4m(lc):
    B, H, N = 2, 1, N4M
    bf = lambda a: torch.tensor(a).to(torch.bfloat16).double().numpy()  # noqa: E731
    u = bf(lc.signal_batch(1, B, H, N))
    dy = bf(lc.signal_batch(2, B, H, N))
    K, D = lc.init_kernels(1, H, N, 3)
    K = K.astype(np.float32).astype(np.float64)
    D = D.astype(np.float32).astype(np.float64)
    Kbar = lc.regularize_bank(K, LAM, P)
    y = lc.long_conv_forward(u, Kbar, D)
    du, dKbar, dD = lc.long_conv_backward(u, dy, Kbar, D)
    dK = lc.regularizer_backward(K, LAM, P, dKbar)
    return dict(u=u, dy=dy, K=K, D=D, Kbar=Kbar, y=y, du=du, dKbar=dKbar, dD=dD, dK=dK)


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
def test_three_pass_4m(case4m, dtype, tol):
    c = case4m
    B, H, N = 2, 1, N4M
    plan = fb.LongConvPlan(N, H, fb.ConvMode.CAUSAL, dtype, fb.Engine.AUTO)
    assert plan.engine == fb.Engine.THREE_PASS and plan.m == 1024
    cfg = fb.RegularizationConfig(lambda_=LAM, smooth_width=P)
    dev = lambda a, dt: torch.tensor(a, dtype=torch.float64).to(dt).cuda()  # noqa: E731
    plan.prep(dev(c["K"], torch.float32), dev(c["D"], torch.float32), cfg)
    y, saved = plan.forward(dev(c["u"], dtype), save=True)
    du, dK, dD = plan.backward(dev(c["dy"], dtype), dev(c["u"], dtype), saved=saved)
    torch.cuda.synchronize()
    errs = {"y": rel_l2(to_np(y), c["y"]), "du": rel_l2(to_np(du), c["du"]),
            "dK": rel_l2(to_np(dK), c["dK"]), "dD": rel_l2(to_np(dD), c["dD"]),
            "kbar": rel_l2(to_np(plan.kbar()), c["Kbar"])}
    print(f"N=4M three-pass {dtype}:", errs)
    assert all(e <= tol for e in errs.values()), errs


def test_seqshard_4m_world1(case4m):
    """Sequence-sharded layer at one rank: sharded regularize, kernel spectrum,
    forward, backward (du, dKbar, dD) and the regularizer chain rule to dK."""
    from paper_2302_06646_b200 import seqshard as ss

    c = case4m
    B, H, N = 2, 1, N4M
    l = 8192
    m = 2 * N // l
    sh = ss.SeqShard(l=l, m=m, world=1, rank=0)
    cols = lambda a: torch.tensor(a, dtype=torch.float32, device="cuda").reshape(  # noqa: E731
        *a.shape[:-1], m // 2, l)
    gp = ss.GpuPasses(2 * N)
    kbar = ss.sharded_regularize(cols(c["K"]), LAM, P, sh)
    D = torch.tensor(c["D"], dtype=torch.float32, device="cuda")
    y = ss.sharded_long_conv(cols(c["u"]), kbar, D, sh, gp)
    du, dkbar, dD = ss.sharded_long_conv_backward(cols(c["dy"]), cols(c["u"]), kbar, D, sh, gp)
    dK = ss.sharded_regularizer_backward(cols(c["K"]), dkbar, LAM, P, sh)
    torch.cuda.synchronize()
    errs = {"kbar": rel_l2(to_np(kbar).reshape(H, N), c["Kbar"]),
            "y": rel_l2(to_np(y).reshape(B, H, N), c["y"]),
            "du": rel_l2(to_np(du).reshape(B, H, N), c["du"]),
            "dKbar": rel_l2(to_np(dkbar).reshape(H, N), c["dKbar"]),
            "dK": rel_l2(to_np(dK).reshape(H, N), c["dK"]),
            "dD": rel_l2(to_np(dD), c["dD"])}
    print("N=4M seqshard world 1:", errs)
    assert all(e <= 1e-5 for e in errs.values()), errs


@pytest.mark.parametrize("N", [65536, 262144])
def test_three_pass_big_m_bf16(lc, N):
    """bf16 three-pass at m = 16 .. 64 with an odd batch (zero partner) — the
    column-size ladder between config 3 and N = 4M (m = 1024 above)."""
    from helpers import layer_inputs
    from test_gpu_layer import CFG, assert_parity, oracle_layer, run_layer

    inp = layer_inputs(lc, 3, 1, N, torch.bfloat16)
    cfg = fb.RegularizationConfig(**CFG)
    plan, got = run_layer(inp, N, 1, torch.bfloat16, cfg, engine=2)
    assert plan.m == 2 * N // 8192
    assert_parity(got, oracle_layer(lc, inp, cfg), 2e-2, keys=("y", "du", "dK", "dD"))
