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
