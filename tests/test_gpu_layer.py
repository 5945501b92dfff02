"""GPU parity of the layer (K1 + K2/K3 forward, K4 backward) through the C ABI
against the fp64 oracle (oracle/lc_oracle.c, pinned to the reference) and
the reference-generated golden fixtures.

Bars (BASELINE.json north_star): relative L2 <= 1e-5 in fp32 mode,
<= 2e-2 in bf16/fp16 tensor mode, for y, du, dK (and dD)."""
import numpy as np
import pytest
import torch

from conftest import golden
from helpers import TOL, layer_inputs, rounded, to_np
from oracle.oracle import rel_l2

pytestmark = pytest.mark.gpu

fb = pytest.importorskip("paper_2302_06646_b200")


def run_layer(inp, N, H, dtype, cfg, mode=1, engine=0, training=False):
    plan = fb.LongConvPlan(N, H, fb.ConvMode(mode), dtype, fb.Engine(engine))
    plan.prep(inp["tK"], inp["tD"], cfg, training)
    y = plan.forward(inp["tu"])
    du, dK, dD, dKbar = plan.backward(inp["tdy"], inp["tu"], want_dkbar=True)
    torch.cuda.synchronize()
    return plan, dict(y=to_np(y), du=to_np(du), dK=to_np(dK), dD=to_np(dD), dKbar=to_np(dKbar),
                      kbar=to_np(plan.kbar()))


def oracle_layer(lc, inp, cfg, causal=True, training=False):
    lam, p = cfg.lambda_, cfg.smooth_width
    Kbar = lc.regularize_bank(inp["K"], lam, p, cfg.dropout_rate, int(cfg.smooth_domain), cfg.seed,
                              training)
    y = lc.long_conv_forward(inp["u"], Kbar, inp["D"], causal)
    du, dKbar, dD = lc.long_conv_backward(inp["u"], inp["dy"], Kbar, inp["D"], causal)
    if cfg.smooth_domain == 0:
        dK = lc.regularizer_backward(inp["K"], lam, p, dKbar, cfg.dropout_rate, cfg.seed, training)
    else:
        dK = None
    return dict(y=y, du=du, dK=dK, dD=dD, dKbar=dKbar, kbar=Kbar)


def assert_parity(got, want, tol, keys=("y", "du", "dK", "dD", "dKbar", "kbar")):
    errs = {k: rel_l2(got[k], want[k]) for k in keys if want.get(k) is not None}
    assert all(e <= tol for e in errs.values()), errs
    return errs


CFG = dict(lambda_=0.003, smooth_width=1)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
def test_config1_single_channel(lc, dtype):
    # BASELINE config 1: B=1 H=1 N=1024 causal fwd+bwd vs the CPU oracle
    inp = layer_inputs(lc, 1, 1, 1024, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    _, got = run_layer(inp, 1024, 1, dtype, cfg)
    assert_parity(got, oracle_layer(lc, inp, cfg), TOL[dtype])


@pytest.mark.parametrize("B,H,N", [(2, 3, 128), (3, 4, 256), (4, 2, 1000), (2, 2, 4096),
                                   (5, 3, 64), (1, 2, 4), (2, 1, 1)])
def test_single_pass_shapes_fp32(lc, B, H, N):
    inp = layer_inputs(lc, B, H, N, torch.float32)
    cfg = fb.RegularizationConfig(**CFG)
    _, got = run_layer(inp, N, H, torch.float32, cfg, engine=1)
    assert_parity(got, oracle_layer(lc, inp, cfg), 1e-5)


@pytest.mark.parametrize("N", [8, 64, 256, 1024])
def test_circular_mode_fp32(lc, N):
    inp = layer_inputs(lc, 3, 2, N, torch.float32)
    cfg = fb.RegularizationConfig(**CFG)
    _, got = run_layer(inp, N, 2, torch.float32, cfg, mode=0)
    assert_parity(got, oracle_layer(lc, inp, cfg, causal=False), 1e-5)


@pytest.mark.parametrize("N", [256, 512, 1024, 2048, 4096])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("B,H", [(3, 2), (8, 3)])
def test_circular_mode_tensor_cores(lc, dtype, B, H, N):
    """16-bit circular mode (n = N, no zero padding) on the radix-16 tcgen05
    single pass."""
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    plan, got = run_layer(inp, N, H, dtype, cfg, mode=0)
    assert plan.tensor_cores
    assert_parity(got, oracle_layer(lc, inp, cfg, causal=False), TOL[dtype])


def test_dropout_training_mode(lc):
    # on-device xoshiro256++ stream must reproduce the reference mask exactly
    inp = layer_inputs(lc, 2, 3, 512, torch.float32)
    cfg = fb.RegularizationConfig(lambda_=0.003, smooth_width=1, dropout_rate=0.2, seed=7)
    _, got = run_layer(inp, 512, 3, torch.float32, cfg, training=True)
    want = oracle_layer(lc, inp, cfg, training=True)
    assert np.array_equal(got["kbar"] == 0, want["kbar"] == 0)
    assert_parity(got, want, 1e-5)


@pytest.mark.parametrize("kind,H,N,seed", [(1, 3, 4096, 3), (0, 5, 20001, 11), (1, 2, 1, 0),
                                           (1, 7, 131072, 42)])
def test_init_kernels_on_device(lc, kind, H, N, seed):
    """init_kernels (regularize.cpp:73-91) on the device: the reference's
    xoshiro256++ streams, split over threads by GF(2) jump-ahead (chunks of
    512 draws; odd N ends on a cached-sine-free pair), fp64 Box-Muller."""
    K64, D64 = fb.init_kernels(fb.InitKind(kind), H, N, seed, dtype=torch.float64)
    K32, D32 = fb.init_kernels(fb.InitKind(kind), H, N, seed)
    Kw, Dw = lc.init_kernels(kind, H, N, seed)
    K64, D64 = to_np(K64), to_np(D64)
    # device fp64 libm vs glibc: a last-ulp difference at most
    assert np.max(np.abs(K64 - Kw) / np.maximum(np.abs(Kw), 1e-300)) < 1e-13
    assert np.max(np.abs(D64 - Dw) / np.maximum(np.abs(Dw), 1e-300)) < 1e-13
    assert np.mean(to_np(K32) == Kw.astype(np.float32)) > 0.9999
    assert np.array_equal(to_np(D32), Dw.astype(np.float32))


def test_dropout_mask_long_streams(lc):
    """Dropout keep flags over many jump-ahead chunks per head (N = 20000, not
    a multiple of the 512-draw chunk) equal the reference's sequential walk."""
    H, N = 3, 20000
    K = torch.randn(H, N, device="cuda")
    D = torch.zeros(H, device="cuda")
    cfg = fb.RegularizationConfig(dropout_rate=0.3, seed=123)
    plan = fb.LongConvPlan(N, H, fb.ConvMode.CAUSAL, torch.float32, fb.Engine.AUTO)
    plan.prep(K, D, cfg, True)
    kbar = to_np(plan.kbar())
    want = lc.regularize_bank(to_np(K), 0.0, 0, 0.3, 0, 123, True)
    assert np.array_equal(kbar == 0, want == 0)
    assert rel_l2(kbar, want) < 1e-6


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
def test_dropout_training_three_pass(lc, dtype, tol):
    """Three-pass training step with kernel dropout: the prep (mask, Kbar,
    kernel spectrum) runs on the plan's auxiliary stream and the dK tail
    (regularizer chain rule through the mask) forks off the backward; two
    steps back to back on one plan, each against the oracle."""
    N, H, B = 16384, 3, 3
    plan = None
    for seed in (7, 8):
        inp = layer_inputs(lc, B, H, N, dtype, seeds=(seed, seed + 10, seed + 20))
        cfg = fb.RegularizationConfig(lambda_=0.003, smooth_width=1, dropout_rate=0.2, seed=seed)
        if plan is None:
            plan = fb.LongConvPlan(N, H, fb.ConvMode.CAUSAL, dtype, fb.Engine.THREE_PASS)
        plan.prep(inp["tK"], inp["tD"], cfg, True)
        y = plan.forward(inp["tu"])
        du, dK, dD = plan.backward(inp["tdy"], inp["tu"])
        torch.cuda.synchronize()
        got = dict(y=to_np(y), du=to_np(du), dK=to_np(dK), dD=to_np(dD), kbar=to_np(plan.kbar()))
        want = oracle_layer(lc, inp, cfg, training=True)
        assert np.array_equal(got["kbar"] == 0, want["kbar"] == 0)
        assert_parity(got, want, tol, keys=("y", "du", "dK", "dD", "kbar"))


def test_smooth_frequency(lc):
    inp = layer_inputs(lc, 2, 2, 256, torch.float32)
    cfg = fb.RegularizationConfig(lambda_=0.01, smooth_width=2,
                                  smooth_domain=fb.SmoothDomain.FREQUENCY)
    _, got = run_layer(inp, 256, 2, torch.float32, cfg)
    want = oracle_layer(lc, inp, cfg)
    assert_parity(got, want, 1e-5, keys=("y", "du", "dD", "dKbar", "kbar"))
    # chain rule: smooth_frequency(k) = k * w (Dirichlet window) is self-adjoint
    t = np.arange(256)
    w = (1 + 2 * sum(np.cos(2 * np.pi * d * t / 256) for d in (1, 2))) / 5
    dK = (want["kbar"] != 0) * want["dKbar"] * w
    assert rel_l2(got["dK"], dK) < 1e-5


@pytest.mark.parametrize("name", ["layer_b1h1n1024", "layer_b3h4n256", "layer_b2h2n128_circ",
                                  "layer_b2h3n64_drop"])
def test_against_reference_golden(name):
    """Directly against outputs of the unmodified reference (tests/golden)."""
    g = golden(name)
    causal, training = bool(g["causal"]), bool(g["training"])
    B, H, N = g["u"].shape
    cfg = fb.RegularizationConfig(lambda_=float(g["lam"]), smooth_width=int(g["p"]),
                                  dropout_rate=float(g["rate"]), seed=int(g["seed"]))
    # fp32 inputs: compare against the reference evaluated on fp64 inputs,
    # so the bar absorbs the input rounding (rel ~6e-8)
    inp = dict(tu=torch.tensor(g["u"], dtype=torch.float32).cuda(),
               tdy=torch.tensor(g["dy"], dtype=torch.float32).cuda(),
               tK=torch.tensor(g["K"], dtype=torch.float32).cuda(),
               tD=torch.tensor(g["D"], dtype=torch.float32).cuda())
    _, got = run_layer(inp, N, H, torch.float32, cfg, mode=int(causal), training=training)
    assert rel_l2(got["y"], g["y_engine1"]) < 1e-5
    if causal:
        for k in ("du", "dK", "dD"):
            assert rel_l2(got[k], g[k]) < 1e-5, k


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_deterministic(lc, dtype):
    inp = layer_inputs(lc, 6, 4, 2048, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    _, a = run_layer(inp, 2048, 4, dtype, cfg)
    _, b = run_layer(inp, 2048, 4, dtype, cfg)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_autograd_long_conv(lc):
    B, H, N = 2, 3, 512
    inp = layer_inputs(lc, B, H, N, torch.float32)
    u = inp["tu"].clone().requires_grad_(True)
    K = inp["tK"].clone().requires_grad_(True)
    D = inp["tD"].clone().requires_grad_(True)
    cfg = fb.RegularizationConfig(**CFG)
    y = fb.long_conv(u, K, D, cfg)
    y.backward(inp["tdy"])
    want = oracle_layer(lc, inp, cfg)
    assert rel_l2(to_np(y), want["y"]) < 1e-5
    assert rel_l2(to_np(u.grad), want["du"]) < 1e-5
    assert rel_l2(to_np(K.grad), want["dK"]) < 1e-5
    assert rel_l2(to_np(D.grad), want["dD"]) < 1e-5


def test_dimension_errors():
    with pytest.raises(fb.DimensionError):
        plan = fb.LongConvPlan(64, 2)
        plan.prep(torch.zeros(3, 64, device="cuda"), torch.zeros(3, device="cuda"),
                  fb.RegularizationConfig())
    plan = fb.LongConvPlan(64, 2)
    plan.prep(torch.zeros(2, 64, device="cuda"), torch.zeros(2, device="cuda"),
              fb.RegularizationConfig())
    with pytest.raises(fb.DimensionError):
        plan.forward(torch.zeros(1, 3, 64, device="cuda"))
    with pytest.raises(fb.DimensionError):
        fb.LongConvPlan(64, 2).prep(torch.zeros(2, 64, device="cuda"),
                                    torch.zeros(2, device="cuda"),
                                    fb.RegularizationConfig(lambda_=-1.0))


# ------------------------------------------------------------ tcgen05 single-pass
@pytest.mark.parametrize("N", [4096, 2048, 1024, 512, 256, 128])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("B,H", [(2, 2), (3, 3), (5, 1), (16, 3), (8, 5)])
def test_tensor_core_single_pass(lc, dtype, B, H, N):
    """N = 4096, and N = 2048 on the same n = 8192 transform (16 data rows);
    N = 128 / 256 / 512 / 1024 on the radix-16 stages (fb_learned_tc.cu short single pass)."""
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    plan, got = run_layer(inp, N, H, dtype, cfg, engine=1)
    assert plan.tensor_cores, "16-bit causal N=4096 / 2048 must run on tcgen05"
    assert_parity(got, oracle_layer(lc, inp, cfg), TOL[dtype])


@pytest.mark.parametrize("B,H,N", [(32, 20, 4096), (9, 37, 4096), (64, 6, 4096), (9, 37, 2048)])
def test_tensor_core_persistent_shares(lc, B, H, N):
    """Pair counts above the SM count: the persistent CTAs' shares straddle
    head boundaries (several head segments per CTA, several CTAs per head),
    which exercises the k_f' reloads and the dK-partial bookkeeping."""
    dtype = torch.bfloat16
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    plan, got = run_layer(inp, N, H, dtype, cfg, engine=1)
    assert plan.tensor_cores
    assert_parity(got, oracle_layer(lc, inp, cfg), TOL[dtype], keys=("y", "du", "dK", "dD"))


@pytest.mark.parametrize("dtype,B,H", [(torch.bfloat16, 3, 3), (torch.float16, 2, 2),
                                       (torch.bfloat16, 32, 48), (torch.bfloat16, 9, 37)])
@pytest.mark.parametrize("saved", [True, False])
def test_tensor_core_v2_design(lc, monkeypatch, dtype, B, H, saved):
    """The 128 x 64 TMEM-resident single-pass design (fb_tc2.cu, opt-in via
    FB_TC2=1 at plan creation): odd batches, multi-segment CTA shares, the
    training step (saved U) and the recompute path."""
    monkeypatch.setenv("FB_TC2", "1")
    N = 4096
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    plan = fb.LongConvPlan(N, H, fb.ConvMode.CAUSAL, dtype, fb.Engine.BUTTERFLY)
    assert plan.tensor_cores
    plan.prep(inp["tK"], inp["tD"], cfg)
    if saved:
        y, sv = plan.forward(inp["tu"], save=True)
        du, dK, dD = plan.backward(inp["tdy"], inp["tu"], saved=sv)
    else:
        y = plan.forward(inp["tu"])
        du, dK, dD = plan.backward(inp["tdy"], inp["tu"])
    torch.cuda.synchronize()
    got = dict(y=to_np(y), du=to_np(du), dK=to_np(dK), dD=to_np(dD))
    assert_parity(got, oracle_layer(lc, inp, cfg), TOL[dtype], keys=("y", "du", "dK", "dD"))


def test_tensor_core_deterministic(lc):
    B, H, N = 32, 20, 4096
    inp = layer_inputs(lc, B, H, N, torch.bfloat16)
    cfg = fb.RegularizationConfig(**CFG)
    _, a = run_layer(inp, N, H, torch.bfloat16, cfg, engine=1)
    _, b = run_layer(inp, N, H, torch.bfloat16, cfg, engine=1)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_tensor_core_matches_simt(lc):
    """tcgen05 path vs the fp32 CUDA-core path on identical bf16 inputs."""
    B, H, N = 4, 2, 4096
    inp = layer_inputs(lc, B, H, N, torch.bfloat16)
    cfg = fb.RegularizationConfig(**CFG)
    _, a = run_layer(inp, N, H, torch.bfloat16, cfg, engine=1)
    _, b = run_layer(inp, N, H, torch.bfloat16, cfg, engine=3)
    for k in ("y", "du", "dK", "dD"):
        assert rel_l2(a[k], b[k]) < 2e-2, k


def test_config2_heads_sample_tensor_core(lc):
    """BASELINE config 2 (B=32 H=256 N=4096 bf16) on tcgen05; a head sample
    (all batches, so dK is complete) against the fp64 oracle."""
    B, H, N = 32, 256, 4096
    dtype = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(7)
    u = torch.randn(B, H, N, device="cuda", generator=g).to(dtype)
    dy = torch.randn(B, H, N, device="cuda", generator=g).to(dtype)
    K, D = lc.init_kernels(1, H, N, 3)
    tK = torch.tensor(K, dtype=torch.float32, device="cuda")
    tD = torch.tensor(D, dtype=torch.float32, device="cuda")
    cfg = fb.RegularizationConfig(**CFG)
    plan = fb.LongConvPlan(N, H, fb.ConvMode.CAUSAL, dtype)
    assert plan.tensor_cores
    plan.prep(tK, tD, cfg)
    y = plan.forward(u)
    du, dK, dD = plan.backward(dy, u)
    torch.cuda.synchronize()
    heads = [0, 131, 255]
    sub = dict(u=to_np(u[:, heads]), dy=to_np(dy[:, heads]), K=to_np(tK[heads]), D=to_np(tD[heads]))
    want = oracle_layer(lc, sub, cfg)
    got = dict(y=to_np(y[:, heads]), du=to_np(du[:, heads]), dK=to_np(dK[heads]),
               dD=to_np(dD[heads]))
    errs = assert_parity(got, want, 2e-2, keys=("y", "du", "dK", "dD"))
    print("config2 tcgen05 rel-L2:", errs)


# ------------------------------------------------------------ three-pass (K3/K4b)
@pytest.mark.parametrize("B,H,N,mode", [(2, 2, 8192, 1), (3, 2, 16384, 1), (2, 1, 65536, 1),
                                        (2, 2, 16384, 0)])
def test_three_pass_fp32(lc, B, H, N, mode):
    inp = layer_inputs(lc, B, H, N, torch.float32)
    cfg = fb.RegularizationConfig(**CFG)
    plan, got = run_layer(inp, N, H, torch.float32, cfg, mode=mode, engine=2)
    assert plan.engine == fb.Engine.THREE_PASS and plan.m == (2 * N if mode else N) // 8192
    assert_parity(got, oracle_layer(lc, inp, cfg, causal=bool(mode)), 1e-5)


@pytest.mark.parametrize("B,H,N", [(2, 1, 131072), (3, 1, 262144), (3, 2, 131072)])
def test_three_pass_tiled_columns_fp32(lc, B, H, N):
    """m = 2N / 8192 > 16: passes 1/3 run as smem-tiled batched column FFTs."""
    inp = layer_inputs(lc, B, H, N, torch.float32)
    cfg = fb.RegularizationConfig(**CFG)
    plan, got = run_layer(inp, N, H, torch.float32, cfg, engine=2)
    assert plan.m == 2 * N // 8192 and plan.m > 16
    assert_parity(got, oracle_layer(lc, inp, cfg), 1e-5)


@pytest.mark.slow
def test_sweep_1m_bf16(lc):
    """Top of the BASELINE sweep: N = 2^20 (m = 256 columns), one pair, bf16."""
    B, H, N = 2, 1, 1 << 20
    inp = layer_inputs(lc, B, H, N, torch.bfloat16)
    cfg = fb.RegularizationConfig(**CFG)
    plan, got = run_layer(inp, N, H, torch.bfloat16, cfg)
    assert plan.engine == fb.Engine.THREE_PASS and plan.m == 256
    assert_parity(got, oracle_layer(lc, inp, cfg), 2e-2, keys=("y", "du", "dK", "dD"))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_three_pass_16bit(lc, dtype):
    inp = layer_inputs(lc, 3, 2, 32768, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    _, got = run_layer(inp, 32768, 2, dtype, cfg, engine=2)
    assert_parity(got, oracle_layer(lc, inp, cfg), 2e-2)


@pytest.mark.parametrize("B,H,N,mode,dtype", [(2, 2, 8192, 1, torch.bfloat16),
                                              (1, 3, 16384, 0, torch.bfloat16),
                                              (5, 2, 65536, 1, torch.bfloat16),
                                              (4, 3, 16384, 1, torch.bfloat16),
                                              (3, 1, 131072, 1, torch.bfloat16),
                                              (2, 1, 262144, 1, torch.bfloat16),
                                              (3, 2, 16384, 1, torch.float16),
                                              (2, 2, 65536, 0, torch.float16),
                                              (3, 1, 131072, 1, torch.float16),
                                              (4, 2, 131072, 1, torch.bfloat16),
                                              (1, 2, 262144, 1, torch.float16),
                                              (2, 1, 524288, 1, torch.bfloat16),
                                              (3, 1, 524288, 1, torch.float16)])
def test_three_pass_bf16_tc_rows(lc, B, H, N, mode, dtype):
    """16-bit three-pass with pass 2 on tcgen05 (m = 2 .. 128: register
    column pass 1 for m <= 16, the tcgen05 column GEMM for causal m = 32 ..
    128, writing planar rows; causal and circular; odd B = a
    zero partner channel; fp16 I/O with bf16 rows): recompute and saved-U
    backward agree bit for bit, both within the 16-bit bar of the oracle."""
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    plan, got = run_layer(inp, N, H, dtype, cfg, mode=mode, engine=2)
    assert plan.engine == fb.Engine.THREE_PASS
    assert_parity(got, oracle_layer(lc, inp, cfg, causal=bool(mode)), 2e-2,
                  keys=("y", "du", "dK", "dD"))
    y, saved = plan.forward(inp["tu"], save=True)
    du, dK, dD = plan.backward(inp["tdy"], None, saved=saved)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(y), got["y"])
    assert np.array_equal(to_np(du), got["du"])


def test_config3_heads_sample(lc):
    """BASELINE config 3 shape (B=16 H=128 N=65536 bf16, three-pass) on the
    GPU; a sample of heads (all batches, so dK is complete) vs the oracle."""
    B, H, N = 16, 128, 65536
    dtype = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(5)
    u = torch.randn(B, H, N, device="cuda", generator=g).to(dtype)
    dy = torch.randn(B, H, N, device="cuda", generator=g).to(dtype)
    K, D = lc.init_kernels(1, H, N, 3)
    tK = torch.tensor(K, dtype=torch.float32, device="cuda")
    tD = torch.tensor(D, dtype=torch.float32, device="cuda")
    cfg = fb.RegularizationConfig(**CFG)
    plan = fb.LongConvPlan(N, H, fb.ConvMode.CAUSAL, dtype, fb.Engine.AUTO)
    assert plan.engine == fb.Engine.THREE_PASS and plan.m == 16
    plan.prep(tK, tD, cfg)
    y = plan.forward(u)
    du, dK, dD = plan.backward(dy, u)
    torch.cuda.synchronize()
    heads = [0, 77]
    sub = dict(u=to_np(u[:, heads]), dy=to_np(dy[:, heads]), K=to_np(tK[heads]), D=to_np(tD[heads]))
    want = oracle_layer(lc, sub, cfg)
    got = dict(y=to_np(y[:, heads]), du=to_np(du[:, heads]), dK=to_np(dK[heads]),
               dD=to_np(dD[heads]))
    assert_parity(got, want, 2e-2, keys=("y", "du", "dK", "dD"))


# ------------------------------------------------------------ host-buffer runner
@pytest.mark.parametrize("dtype,H,hc,training,N", [(torch.bfloat16, 12, 4, False, 4096),
                                                   (torch.float32, 6, 2, True, 4096),
                                                   (torch.bfloat16, 4, 2, False, 16384),
                                                   # H / hc >= 4: small first / last chunks
                                                   (torch.bfloat16, 32, 8, True, 4096),
                                                   (torch.float32, 16, 4, False, 4096)])
def test_host_runner_matches_device_path(lc, dtype, H, hc, training, N):
    """fb_host_runner (pinned host buffers, heads in pipelined chunks) gives
    the device path's results: y / du per channel bit-identical, dK / dD up to
    the fixed-order partial grouping and the saved-transform rounding (three-
    pass); dropout streams follow the global head."""
    B = 5
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(lambda_=0.003, smooth_width=1,
                                  dropout_rate=0.2 if training else 0.0, seed=7)
    _, want = run_layer(inp, N, H, dtype, cfg, training=training)
    r = fb.HostRunner(N, H, B, dtype, heads_per_chunk=hc)
    assert r.chunk_heads == hc
    pin = lambda t: t.cpu().contiguous().pin_memory()  # noqa: E731
    y, du, dK, dD = r.run(pin(inp["tu"]), pin(inp["tdy"]), pin(inp["tK"]), pin(inp["tD"]), cfg,
                          training=training)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(y), want["y"])
    assert np.array_equal(to_np(du), want["du"])
    tol = 1e-6 if N <= 8192 else 1e-2  # three-pass: U saved in the I/O precision
    assert rel_l2(to_np(dK), want["dK"]) < tol
    assert rel_l2(to_np(dD), want["dD"]) < tol


@pytest.mark.parametrize("B,H,dtype,N", [(32, 20, torch.bfloat16, 4096), (7, 3, torch.bfloat16, 4096),
                                         (6, 4, torch.float16, 4096), (7, 3, torch.bfloat16, 2048)])
def test_tensor_core_saved_transform(lc, B, H, dtype, N):
    """fb_fwd_save / fb_bwd_saved (the backward reads the forward's transform
    of u) gives bit-identical results to the recompute path: it parks exactly
    the same bf16 values."""
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    plan, want = run_layer(inp, N, H, dtype, cfg, engine=1)
    assert plan.saved_size(B) == ((B + 1) // 2) * H * 8192 * 4
    y, saved = plan.forward(inp["tu"], save=True)
    du, dK, dD = plan.backward(inp["tdy"], None, saved=saved)
    torch.cuda.synchronize()
    for k, v in (("y", y), ("du", du), ("dK", dK), ("dD", dD)):
        assert np.array_equal(to_np(v), want[k]), k


# ------------------------------------------------------------ sequence-sharded four-step
@pytest.mark.parametrize("m", [16, 64])
def test_four_step_gpu_passes_single_rank(m):
    """seqshard.four_step_conv with the GPU local passes (fb_shard_*) at one
    rank (the exchange is the identity) against numpy's circular convolution;
    the multi-rank exchange itself is covered by the gloo tests on CPU."""
    from paper_2302_06646_b200 import seqshard as ss

    l = 8192
    n, Cn = l * m, 3
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((Cn, n)) + 1j * rng.standard_normal((Cn, n))).astype(np.complex64)
    k = np.zeros((Cn, n), np.float32)
    k[:, : n // 2] = rng.standard_normal((Cn, n // 2)) * np.exp(-np.arange(n // 2) / 500.0)
    want = np.fft.ifft(np.fft.fft(x.astype(np.complex128), axis=1) * np.fft.fft(k, axis=1), axis=1)
    sh = ss.SeqShard(l=l, m=m, world=1, rank=0)
    gp = ss.GpuPasses(n)
    kcols = ss.scatter_tau(torch.from_numpy(k).cuda(), sh)[:, : m // 2]  # the causal half
    kf2 = gp.spectrum_rows(kcols, sh)
    khat = np.fft.fft(k.astype(np.float64), axis=1)
    s_idx, a_idx = np.arange(l), np.arange(m)
    kf2_want = khat[:, a_idx[:, None] + m * s_idx[None, :]]
    assert rel_l2(kf2.cpu().numpy(), kf2_want) < 1e-5
    xc = ss.scatter_tau(torch.from_numpy(x).cuda(), sh)
    for chunks in (1, 2):
        y = ss.four_step_conv(xc, sh, gp, chunks=chunks)
        got = ss.gather_tau([y.cpu()], sh).numpy()
        assert rel_l2(got, want) < 1e-5, chunks


def test_shard_stage_layouts():
    """fb_shard_stage (the all-to-all send / receive layouts): out[b][a][x] =
    in[a][b][x], exact in f32, bf16-rounded on a bf16 wire and back."""
    from paper_2302_06646_b200 import seqshard as ss

    gp = ss.GpuPasses(8192 * 16)
    A, Bd, X = 6, 4, 96
    t = torch.randn(A, Bd, X, dtype=torch.complex64, device="cuda")
    want = t.permute(1, 0, 2).contiguous().reshape(-1)
    assert torch.equal(gp.stage(t, A, Bd, X, "f32"), want)
    wire = gp.stage(t, A, Bd, X, "bf16")
    assert wire.dtype == torch.bfloat16 and wire.numel() == 2 * A * Bd * X
    back = gp.stage(wire, Bd, A, X, "f32")  # [A][Bd][X] again, f32
    ref = torch.view_as_complex(torch.view_as_real(t).bfloat16().float()).reshape(-1)
    assert torch.equal(back, ref)


@pytest.mark.parametrize("dtype,N", [(torch.float32, 16384), (torch.bfloat16, 32768),
                                     (torch.float16, 32768)])
def test_three_pass_saved_transform(lc, dtype, N):
    """Three-pass training step: the forward keeps its pass-2 row spectra of u
    and the backward runs passes 1/2 on dy only (dD from the lag-0 dKbar).
    y and du are bit-identical to the recompute path; dK and dD match the
    oracle at the mode's bar."""
    B, H = 3, 2
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    plan, want = run_layer(inp, N, H, dtype, cfg, engine=2)
    assert plan.saved_size(B) > 0
    y, saved = plan.forward(inp["tu"], save=True)
    du, dK, dD = plan.backward(inp["tdy"], None, saved=saved)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(y), want["y"])
    assert np.array_equal(to_np(du), want["du"])
    ref = oracle_layer(lc, inp, cfg)
    assert_parity(dict(y=to_np(y), du=to_np(du), dK=to_np(dK), dD=to_np(dD)), ref, TOL[dtype],
                  keys=("y", "du", "dK", "dD"))


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
def test_sharded_long_conv_layer_single_rank(lc, dtype, tol):
    """seqshard.sharded_long_conv (pairs of real channels, causal crop, D u)
    at one rank against the fp64 layer oracle (N = 65536: l = 8192, m = 16);
    bf16 signals in and out (fp32 complex intermediates)."""
    from paper_2302_06646_b200 import seqshard as ss

    B, H, N = 3, 2, 65536
    l, m = 8192, 16
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    kbar = lc.regularize_bank(inp["K"], cfg.lambda_, cfg.smooth_width)
    want = lc.long_conv_forward(inp["u"], kbar, inp["D"])
    sh = ss.SeqShard(l=l, m=m, world=1, rank=0)
    u_cols = inp["tu"].reshape(B, H, m // 2, l)
    k_cols = torch.tensor(kbar, dtype=torch.float32, device="cuda").reshape(H, m // 2, l)
    y = ss.sharded_long_conv(u_cols, k_cols, inp["tD"], sh, ss.GpuPasses(2 * N))
    torch.cuda.synchronize()
    assert y.dtype == dtype
    assert rel_l2(to_np(y.reshape(B, H, N)), want) < tol


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
def test_sharded_long_conv_backward_single_rank(lc, dtype, tol):
    """seqshard.sharded_long_conv_backward on the GPU passes at one rank vs the
    fp64 backward oracle (du, dKbar, dD); bf16 signals in the 16-bit case."""
    from paper_2302_06646_b200 import seqshard as ss

    B, H, N = 3, 2, 65536
    l, m = 8192, 16
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    kbar = lc.regularize_bank(inp["K"], cfg.lambda_, cfg.smooth_width)
    du_w, dkbar_w, dD_w = lc.long_conv_backward(inp["u"], inp["dy"], kbar, inp["D"])
    sh = ss.SeqShard(l=l, m=m, world=1, rank=0)
    cols = lambda t: t.reshape(*t.shape[:-1], m // 2, l)  # noqa: E731
    kt = torch.tensor(kbar, dtype=torch.float32, device="cuda")
    du, dkbar, dD = ss.sharded_long_conv_backward(cols(inp["tdy"]), cols(inp["tu"]), cols(kt),
                                                  inp["tD"], sh, ss.GpuPasses(2 * N))
    torch.cuda.synchronize()
    assert rel_l2(to_np(du.reshape(B, H, N)), du_w) < tol
    assert rel_l2(to_np(dkbar.reshape(H, N)), dkbar_w) < tol
    assert rel_l2(to_np(dD), dD_w) < tol


@pytest.mark.parametrize("dtype,world", [(torch.bfloat16, 4), (torch.float32, 2)])
def test_head_sharding_product(lc, dtype, world):
    """B*H sharding as bench.py --gpus P runs it (seqshard.head_shard, no
    collective): each 'rank' builds its own plan on its head slice; the
    concatenated y / du / dK / dD equal the unsharded plan's bit for bit
    (channels are independent, dK / dD are head-local) and match the oracle."""
    from paper_2302_06646_b200.seqshard import head_shard

    B, H, N = 6, 8, 4096
    inp = layer_inputs(lc, B, H, N, dtype)
    cfg = fb.RegularizationConfig(**CFG)
    _, want = run_layer(inp, N, H, dtype, cfg, engine=1)
    parts = []
    for r in range(world):
        hs = head_shard(H, world, r)
        sub = dict(tu=inp["tu"][:, hs].contiguous(), tdy=inp["tdy"][:, hs].contiguous(),
                   tK=inp["tK"][hs].contiguous(), tD=inp["tD"][hs].contiguous())
        parts.append(run_layer(sub, N, hs.stop - hs.start, dtype, cfg, engine=1)[1])
    for k, ax in (("y", 1), ("du", 1), ("dK", 0), ("dD", 0)):
        assert np.array_equal(np.concatenate([p[k] for p in parts], axis=ax), want[k]), k
    assert_parity(want, oracle_layer(lc, inp, cfg), TOL[dtype], keys=("y", "du", "dK", "dD"))
