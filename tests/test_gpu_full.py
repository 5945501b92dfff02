"""Whole-configuration parity at BASELINE.json's headline shapes: every head
and batch of configs 2, 3 and 4, inputs from the reference RNG (SURVEY.md
§8(c): u / dy from SeededRng(1) / (2) children b*H + h, K and D from
init_kernels(kGeometric, seed 3)), the CUDA path against the fp64 oracle.
The oracle runs one head per task on all host cores (tests/_oracle_pool.py,
a spawn pool that never imports torch).  Bar: relative L2 <= 2e-2 (16-bit
I/O, BASELINE.json north_star), over the whole tensors."""
import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest
import torch

import _oracle_pool as pool
from oracle.oracle import LcOracle, rel_l2

pytestmark = pytest.mark.gpu
fb = pytest.importorskip("paper_2302_06646_b200")

LAM, P = 0.003, 1


def _map(fn, tasks):
    workers = max(1, min(len(tasks), os.cpu_count() or 1))
    with ProcessPoolExecutor(workers, mp_context=mp.get_context("spawn")) as ex:
        return list(ex.map(fn, tasks, chunksize=max(1, len(tasks) // (4 * workers))))


def _bf16(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def _layer_case(B, H, N):
    K, D = LcOracle().init_kernels(1, H, N, 3)
    K32, D32 = K.astype(np.float32), D.astype(np.float32)
    res = _map(pool.layer_head, [(h, B, H, N, K32[h].astype(np.float64), float(D32[h]), LAM, P)
                                 for h in range(H)])
    res.sort(key=lambda t: t[0])
    u = np.stack([r[1] for r in res], axis=1)   # [B, H, N] bf16 bits
    dy = np.stack([r[2] for r in res], axis=1)
    want = dict(y=np.stack([r[3] for r in res], axis=1), du=np.stack([r[4] for r in res], axis=1),
                dK=np.stack([r[5] for r in res]), dD=np.array([r[6] for r in res]))
    return _bf16(u), _bf16(dy), torch.from_numpy(K32).cuda(), torch.from_numpy(D32).cuda(), want


@pytest.mark.parametrize("B,H,N,engine", [(32, 256, 4096, "tcgen05 single pass"),
                                          (16, 128, 65536, "three-pass, rows on tcgen05")])
def test_full_config_layer(B, H, N, engine):
    tu, tdy, tK, tD, want = _layer_case(B, H, N)
    plan = fb.LongConvPlan(N, H, fb.ConvMode.CAUSAL, torch.bfloat16)
    if N == 4096:
        assert plan.tensor_cores
    plan.prep(tK, tD, fb.RegularizationConfig(lambda_=LAM, smooth_width=P))
    y = plan.forward(tu)
    du, dK, dD = plan.backward(tdy, tu)
    torch.cuda.synchronize()
    got = dict(y=y.float().cpu().numpy(), du=du.float().cpu().numpy(), dK=dK.cpu().numpy(),
               dD=dD.cpu().numpy())
    errs = {k: rel_l2(got[k].astype(np.float64), want[k].astype(np.float64)) for k in want}
    print(f"B={B} H={H} N={N} ({engine}), all heads:", errs)
    assert all(e < 2e-2 for e in errs.values()), errs


def test_full_config4_learned():
    B, H, n, r = 8, 768, 1024, 16
    res = _map(pool.learned_head, [(h, B, H, n, r) for h in range(H)])
    res.sort(key=lambda t: t[0])
    blocks = torch.tensor(np.stack([t[1] for t in res]), dtype=torch.complex64).cuda()
    x = _bf16(np.stack([t[2] for t in res], axis=1)).view(B, H, n, 2)
    g = _bf16(np.stack([t[3] for t in res], axis=1)).view(B, H, n, 2)
    plan = fb.LearnedButterflyPlan(n, r, H, torch.bfloat16)
    assert plan.engine == "tcgen05"
    y = torch.view_as_complex(plan.forward(blocks, x).float().contiguous())
    db, dx = plan.gradients(blocks, x, g)
    dx = torch.view_as_complex(dx.float().contiguous())
    torch.cuda.synchronize()
    ry = np.stack([t[4] for t in res], axis=1)  # [B, H, n]
    rdx = np.stack([t[5] for t in res], axis=1)
    rdb = np.stack([t[6] for t in res])
    errs = dict(y=rel_l2(y.cpu().numpy().astype(np.complex128), ry.astype(np.complex128)),
                dx=rel_l2(dx.cpu().numpy().astype(np.complex128), rdx.astype(np.complex128)),
                dblocks=rel_l2(db.cpu().numpy().astype(np.complex128), rdb))
    print(f"config 4 (B={B} H={H} n={n}), all heads:", errs)
    assert all(e < 2e-2 for e in errs.values()), errs
