"""GPU parity of the learned butterfly (K5) through the C ABI against the
reference fixtures (tests/golden) and the fp64 oracle."""
import numpy as np
import pytest
import torch

from conftest import golden
from oracle.oracle import rel_l2

pytestmark = pytest.mark.gpu
fb = pytest.importorskip("paper_2302_06646_b200")


def cplx(a, shape):
    return torch.tensor(np.asarray(a, dtype=np.complex128).reshape(shape), dtype=torch.complex64).cuda()


def to16(t, dtype):
    return torch.view_as_real(t).to(dtype).contiguous()


def from16(t):
    return torch.view_as_complex(t.float().contiguous()).cpu().numpy().astype(np.complex128)


@pytest.mark.parametrize("name,r", [("learned_1024", 16), ("learned_64_r4", 4)])
def test_against_reference_golden(name, r):
    g = golden(name)
    n = g["x"].size
    plan = fb.LearnedButterflyPlan(n, r, 1, torch.complex64)
    blocks = cplx(g["blocks"], (1, -1))
    x = cplx(g["x"], (1, 1, n))
    up = cplx(g["g"], (1, 1, n))
    y = plan.forward(blocks, x)
    db, dx = plan.gradients(blocks, x, up)
    torch.cuda.synchronize()
    assert rel_l2(y.cpu().numpy().ravel(), g["y"]) < 1e-5
    assert rel_l2(dx.cpu().numpy().ravel(), g["dx"]) < 1e-5
    assert rel_l2(db.cpu().numpy().ravel(), g["dblocks"]) < 1e-5


def test_dft_init_is_fft_and_zero_blocks():
    n, H, B = 1024, 3, 2
    plan = fb.LearnedButterflyPlan(n, 16, H)
    assert plan.factors == [16, 16, 4] and plan.param_count == 528
    x = torch.randn(B, H, n, dtype=torch.complex64, device="cuda")
    y = plan.forward(plan.dft_blocks(), x)
    ref = torch.fft.fft(x.cpu().to(torch.complex128))
    assert rel_l2(y.cpu().numpy(), ref.numpy()) < 1e-5
    z = plan.forward(torch.zeros(H, 528, dtype=torch.complex64, device="cuda"), x)
    assert torch.count_nonzero(z) == 0


def batch_case(lc, B, H, n, r, seed=4):
    rng = np.random.default_rng(seed)
    base = lc.learned_init(n, r)
    blocks = base[None, :] + 0.1 * (rng.standard_normal((H, base.size))
                                    + 1j * rng.standard_normal((H, base.size)))
    x = rng.standard_normal((B, H, n)) + 1j * rng.standard_normal((B, H, n))
    g = rng.standard_normal((B, H, n)) + 1j * rng.standard_normal((B, H, n))
    return blocks, x, g


def oracle_batch(lc, blocks, x, g, r, heads):
    B = x.shape[0]
    ys, dxs, dbs = [], [], []
    for h in heads:
        db = 0
        for b in range(B):
            ys.append(lc.learned_forward(blocks[h], x[b, h], r))
            d, dxr = lc.learned_gradients(blocks[h], x[b, h], g[b, h], r)
            dxs.append(dxr)
            db = db + d
        dbs.append(db)
    return np.array(ys), np.array(dxs), np.array(dbs)


@pytest.mark.parametrize("n,r", [(1024, 16), (96, 16), (64, 4), (4096, 16)])
def test_batched_fp32(lc, n, r):
    B, H = 3, 4
    blocks, x, g = batch_case(lc, B, H, n, r)
    plan = fb.LearnedButterflyPlan(n, r, H)
    assert plan.engine != "tcgen05"  # fp32 stays on the CUDA cores (1e-5 bar)
    tb, tx, tg = cplx(blocks, blocks.shape), cplx(x, x.shape), cplx(g, g.shape)
    y = plan.forward(tb, tx).cpu().numpy()
    db, dx = plan.gradients(tb, tx, tg)
    heads = list(range(H))
    ry, rdx, rdb = oracle_batch(lc, blocks, x, g, r, heads)
    order = [(b, h) for h in heads for b in range(B)]
    assert rel_l2(np.array([y[b, h] for b, h in order]), ry) < 1e-5
    assert rel_l2(np.array([dx.cpu().numpy()[b, h] for b, h in order]), rdx) < 1e-5
    assert rel_l2(db.cpu().numpy(), rdb) < 1e-5


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_config4_shape_16bit(lc, dtype):
    """BASELINE config 4 (B=8 H=768 n=1024 WikiText-shaped) in the 16-bit
    mode; oracle on a sample of heads (all b, so dblocks are complete)."""
    B, H, n, r = 8, 768, 1024, 16
    blocks, x, g = batch_case(lc, B, H, n, r, seed=6)
    plan = fb.LearnedButterflyPlan(n, r, H, dtype)
    tb = cplx(blocks, blocks.shape)
    tx = to16(cplx(x, x.shape), dtype)
    tg = to16(cplx(g, g.shape), dtype)
    y = from16(plan.forward(tb, tx))
    db, dx = plan.gradients(tb, tx, tg)
    dx = from16(dx)
    heads = [0, 301, 767]
    # oracle on the same 16-bit-rounded inputs
    xr = from16(tx)
    gr = from16(tg)
    ry, rdx, rdb = oracle_batch(lc, blocks, xr, gr, r, heads)
    order = [(b, h) for h in heads for b in range(B)]
    assert rel_l2(np.array([y[b, h] for b, h in order]), ry) < 2e-2
    assert rel_l2(np.array([dx[b, h] for b, h in order]), rdx) < 2e-2
    assert rel_l2(db.cpu().numpy()[heads], rdb) < 2e-2


@pytest.mark.parametrize("n,B", [(32, 5), (64, 3), (128, 2), (256, 7), (512, 9), (1024, 1), (1024, 6),
                                 (1024, 10), (2048, 3), (2048, 19), (4096, 3)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_tensor_core_chains_16bit(lc, n, B, dtype):
    """The tcgen05 kernels (fb_learned_tc.cu) own the 16-bit chains
    [16] * S + [FL] (n = 32 .. 4096); B not a multiple of the CTA's
    4096 / n rows, so the last row group is partial."""
    H, r = 3, 16
    blocks, x, g = batch_case(lc, B, H, n, r, seed=n + B)
    plan = fb.LearnedButterflyPlan(n, r, H, dtype)
    assert plan.engine == "tcgen05"
    tb = cplx(blocks, blocks.shape)
    tx = to16(cplx(x, x.shape), dtype)
    tg = to16(cplx(g, g.shape), dtype)
    y = from16(plan.forward(tb, tx))
    db, dx = plan.gradients(tb, tx, tg)
    dx = from16(dx)
    heads = list(range(H))
    ry, rdx, rdb = oracle_batch(lc, blocks, from16(tx), from16(tg), r, heads)
    order = [(b, h) for h in heads for b in range(B)]
    ey = rel_l2(np.array([y[b, h] for b, h in order]), ry)
    edx = rel_l2(np.array([dx[b, h] for b, h in order]), rdx)
    edb = rel_l2(db.cpu().numpy(), rdb)
    print(f"n={n} B={B} {dtype}: y {ey:.2e} dx {edx:.2e} dblocks {edb:.2e}")
    assert ey < 2e-2 and edx < 2e-2 and edb < 2e-2
    # again: bit-identical (fixed-order in-kernel reduction, counters reset)
    db2, dx2 = plan.gradients(tb, tx, tg)
    assert torch.equal(db2, db) and np.array_equal(from16(dx2), dx)


def test_autograd():
    n, H, B = 256, 2, 3
    plan = fb.LearnedButterflyPlan(n, 16, H)
    blocks = (plan.dft_blocks() + 0.05 * torch.randn(H, plan.param_count, dtype=torch.complex64,
                                                       device="cuda")).requires_grad_(True)
    x = torch.randn(B, H, n, dtype=torch.complex64, device="cuda", requires_grad=True)
    y = fb.learned_butterfly(x, blocks, 16)
    up = torch.randn_like(y)
    y.backward(up)
    db, dx = plan.gradients(blocks.detach(), x.detach(), up)
    assert torch.allclose(x.grad, dx) and torch.allclose(blocks.grad, db)


# ------------------------------------------------------------ learned-butterfly long convolution
def _lconv_oracle(lc, u, kbar, D, Wf, Wi, r, causal):
    """fp64 composition of the reference's learned_forward / learned_gradients
    (oracle rows): y = Re IL(Wi, L(Wf, pad u) L(Wf, pad k))[:N] + D u and its
    backward for dy (IL(W, z) = conj(L(W, conj z)) / n)."""
    B, H, N = u.shape
    n = 2 * N if causal else N

    def pad(x):
        z = np.zeros(n, np.complex128)
        z[:N] = x
        return z
    out = {}

    def fwd(dy=None):
        y = np.zeros((B, H, N))
        du = np.zeros((B, H, N))
        dk = np.zeros((H, N))
        dD = np.zeros(H)
        dWf = np.zeros_like(Wf)
        dWi = np.zeros_like(Wi)
        for h in range(H):
            Kf = lc.learned_forward(Wf[h], pad(kbar[h]), r)
            gK = np.zeros(n, np.complex128)
            for b in range(B):
                U = lc.learned_forward(Wf[h], pad(u[b, h]), r)
                Zc = np.conj(U * Kf)
                V = lc.learned_forward(Wi[h], Zc, r)
                y[b, h] = V.real[:N] / n + D[h] * u[b, h]
                if dy is None:
                    continue
                g = pad(dy[b, h]) / n
                db, G = lc.learned_gradients(Wi[h], Zc, g, r)
                dWi[h] += db
                gZ = np.conj(G)
                db, dX = lc.learned_gradients(Wf[h], pad(u[b, h]), gZ * np.conj(Kf), r)
                dWf[h] += db
                du[b, h] = dX.real[:N] + D[h] * dy[b, h]
                gK += gZ * np.conj(U)
                dD[h] += np.dot(dy[b, h], u[b, h])
            if dy is not None:
                db, dXk = lc.learned_gradients(Wf[h], pad(kbar[h]), gK, r)
                dWf[h] += db
                dk[h] = dXk.real[:N]
        return y, du, dk, dD, dWf, dWi
    return fwd


@pytest.mark.parametrize("B,H,N,r,causal", [(2, 2, 64, 4, True), (3, 1, 96, 16, False), (2, 3, 512, 16, True)])
def test_learned_long_conv(lc, B, H, N, r, causal):
    """The learned-butterfly long convolution on the device
    vs the fp64 composition of the reference's learned operator: y, du, dKbar,
    dD and both block gradients, with perturbed (non-DFT) blocks; and at the DFT
    initialisation it is the regular layer."""
    rng = np.random.default_rng(B * 100 + N)
    plan = fb.LearnedLongConvPlan(N, H, r, 1 if causal else 0)
    W0 = plan.dft_blocks().cpu().numpy().astype(np.complex128)
    P = W0.shape[1]
    Wf = W0 + 0.1 * (rng.standard_normal((H, P)) + 1j * rng.standard_normal((H, P)))
    Wi = W0 + 0.1 * (rng.standard_normal((H, P)) + 1j * rng.standard_normal((H, P)))
    u = rng.standard_normal((B, H, N)).astype(np.float32).astype(np.float64)
    dy = rng.standard_normal((B, H, N)).astype(np.float32).astype(np.float64)
    kbar = (rng.standard_normal((H, N)) * np.exp(-np.arange(N) / 30.0)).astype(np.float32).astype(np.float64)
    D = rng.standard_normal(H).astype(np.float32).astype(np.float64)
    Wf = Wf.astype(np.complex64).astype(np.complex128)
    Wi = Wi.astype(np.complex64).astype(np.complex128)
    t = lambda a, dt=torch.float32: torch.tensor(a, dtype=dt).cuda()  # noqa: E731
    y = plan.forward(t(u), t(kbar), t(D), t(Wf, torch.complex64), t(Wi, torch.complex64))
    du, dk, dD, dWf, dWi = plan.backward(t(dy), t(u), t(kbar), t(D), t(Wf, torch.complex64),
                                         t(Wi, torch.complex64))
    torch.cuda.synchronize()
    yw, duw, dkw, dDw, dWfw, dWiw = _lconv_oracle(lc, u, kbar, D, Wf, Wi, r, causal)(dy)
    got = dict(y=y, du=du, dk=dk, dD=dD, dWf=dWf, dWi=dWi)
    want = dict(y=yw, du=duw, dk=dkw, dD=dDw, dWf=dWfw, dWi=dWiw)
    errs = {k: rel_l2(got[k].cpu().numpy().astype(np.complex128 if k.startswith("dW") else np.float64), want[k])
            for k in got}
    assert all(e < 1e-5 for e in errs.values()), errs
    # DFT blocks: the layer itself (regularized_long_conv with Kbar, D)
    y0 = plan.forward(t(u), t(kbar), t(D), t(W0, torch.complex64), t(W0, torch.complex64))
    want0 = lc.long_conv_forward(u, kbar, D, causal)
    assert rel_l2(y0.cpu().numpy(), want0) < 1e-5


def test_learned_long_conv_autograd():
    """torch.autograd through fb.learned_long_conv matches the plan's backward."""
    B, H, N, r = 2, 2, 64, 4
    plan = fb.LearnedLongConvPlan(N, H, r)
    W0 = plan.dft_blocks()
    g = torch.Generator(device="cuda").manual_seed(3)
    u = torch.randn(B, H, N, device="cuda", generator=g, requires_grad=True)
    kb = torch.randn(H, N, device="cuda", generator=g, requires_grad=True)
    D = torch.randn(H, device="cuda", generator=g, requires_grad=True)
    Wf = (W0 + 0.05 * torch.randn(W0.shape, dtype=torch.complex64, device="cuda", generator=g)).requires_grad_()
    Wi = (W0 + 0.05 * torch.randn(W0.shape, dtype=torch.complex64, device="cuda", generator=g)).requires_grad_()
    y = fb.learned_long_conv(u, kb, D, Wf, Wi, r)
    dy = torch.randn_like(y)
    (y * dy).sum().backward()
    du, dk, dD, dWf, dWi = plan.backward(dy, u, kb, D, Wf, Wi)
    for a, b in ((u.grad, du), (kb.grad, dk), (D.grad, dD), (Wf.grad, dWf), (Wi.grad, dWi)):
        assert torch.allclose(a, b, rtol=1e-5, atol=1e-6)
