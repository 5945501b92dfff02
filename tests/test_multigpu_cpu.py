"""Multi-rank host logic on CPU (gloo, world size 2 and 4):

* B*H sharding: every rank runs its head slice with no collective and the
  concatenation equals the unsharded layer (oracle compute per rank);
* sequence-sharded four-step (config 5-4M): the two all-to-all transposes of
  paper_2302_06646_b200.seqshard move the data so that, with a numpy
  restatement of the three local passes, the sharded circular convolution
  equals the single-process one.
"""
import os
import tempfile

import numpy as np
import pytest
import torch

from paper_2302_06646_b200 import seqshard as ss

L_COLS, M_ROWS = 64, 16  # n = l * m = 1024


class NumpyPasses:
    """numpy / torch restatement of the local passes (three_pass.cpp:225-254)
    and of the glue kernels (fb_shard_pack / _unpack / _stage / _real_rows,
    fb_shard_rows_bwd) on a rank's slice: test infrastructure standing in for
    seqshard.GpuPasses on CPU ranks."""

    def __init__(self, kf2_full):
        self.kf2 = kf2_full  # [C][m][l] = K_hat[a + m s] (per channel), or set by spectrum_rows

    def _kf2(self):
        return self.kf2.numpy() if isinstance(self.kf2, torch.Tensor) else self.kf2

    def pass1(self, x, sh):
        n = sh.l * sh.m
        X = np.fft.fft(x.numpy(), axis=1)  # over c: sum_c w_m^(a c)
        tau = np.arange(sh.tau0, sh.tau0 + sh.lp)
        a = np.arange(sh.m)[:, None]
        return torch.from_numpy(X * np.exp(-2j * np.pi * a * tau[None, :] / n)).to(torch.complex64)

    def _rows_kf2(self, sh):
        kf2 = self._kf2()
        # full-height kf2 (unsharded problem) or this rank's rows
        return kf2[:, sh.a0:sh.a0 + sh.mp, :] if kf2.shape[1] == sh.m else kf2

    def pass2(self, rows, sh):
        kf2 = self._rows_kf2(sh)
        P = rows.shape[0] // kf2.shape[0]  # kernel rows shared by the channel pairs of a head
        Z = np.fft.fft(rows.numpy(), axis=2) * np.tile(kf2, (P, 1, 1))
        return torch.from_numpy(np.fft.ifft(Z, axis=2) * sh.l).to(torch.complex64)

    def pass3(self, w, sh):
        n = sh.l * sh.m
        tau = np.arange(sh.tau0, sh.tau0 + sh.lp)
        a = np.arange(sh.m)[:, None]
        W = w.numpy() * np.exp(2j * np.pi * a * tau[None, :] / n)
        return torch.from_numpy(np.fft.ifft(W, axis=1) * sh.m / n).to(torch.complex64)

    def rows_fft(self, rows, sh):
        return torch.from_numpy(np.fft.fft(rows.numpy(), axis=2)).to(torch.complex64)

    def rows_bwd(self, dy_rows, u_rows, sh):
        kf2 = self._rows_kf2(sh)
        H = kf2.shape[0]
        P = dy_rows.shape[0] // H
        DY = np.fft.fft(dy_rows.numpy(), axis=2)
        U = np.fft.fft(u_rows.numpy(), axis=2)
        du = np.fft.ifft(DY * np.conj(np.tile(kf2, (P, 1, 1))), axis=2) * sh.l
        S = (np.conj(U) * DY).reshape(P, H, sh.mp, sh.l).sum(0)
        wdk = np.fft.ifft(S, axis=2) * sh.l
        return torch.from_numpy(du).to(torch.complex64), torch.from_numpy(wdk).to(torch.complex64)

    def stage(self, t, A, Bd, X, wire):
        t = t.reshape(-1)
        if t.dtype == torch.bfloat16:
            t = torch.view_as_complex(t.float().reshape(-1, 2).contiguous())
        v = t.reshape(A, Bd, X).permute(1, 0, 2).contiguous().reshape(-1)
        return torch.view_as_real(v).to(torch.bfloat16).reshape(-1) if wire == "bf16" else v

    def pack(self, sig, m):
        B, H, half, lp = sig.shape
        P = (B + 1) // 2
        f = sig.float()
        if B % 2:
            f = torch.cat([f, torch.zeros_like(f[:1])], 0)
        x = torch.zeros(P, H, m, lp, dtype=torch.complex64)
        x[:, :, :half] = torch.complex(f[0::2], f[1::2])
        return x.reshape(P * H, m, lp)

    def unpack(self, y, B, H, half, skip=None, D=None, dtype=torch.float32):
        P = (B + 1) // 2
        y = y.reshape(P, H, -1, y.shape[-1])[:, :, :half]
        out = torch.stack([y.real, y.imag], 1).reshape(2 * P, H, half, y.shape[-1])[:B]
        if skip is not None:
            out = out + D.float().view(1, H, 1, 1) * skip.float()
        return out.to(dtype)

    def pass1_signals(self, sig, sh):
        return self.pass1(self.pack(sig, sh.m), sh)

    def pass3_signals(self, w, sh, B, H, half, skip=None, D=None, dtype=torch.float32):
        return self.unpack(self.pass3(w, sh), B, H, half, skip, D, dtype)

    def real_rows(self, y, half):
        return y.real[:, :half].contiguous().float()

    def spectrum_rows(self, kbar_cols, sh, group=None, wire="f32"):
        """The sharded kernel spectrum, as GpuPasses.spectrum_rows does it."""
        rows = ss.columns_to_rows(self.pass1(self.pack(kbar_cols.float().unsqueeze(0), sh.m), sh), sh, group,
                                  self, wire)
        self.kf2 = np.fft.fft(rows.numpy(), axis=2)
        return torch.from_numpy(self.kf2).to(torch.complex64)


def _problem(C=3, seed=0):
    rng = np.random.default_rng(seed)
    n = L_COLS * M_ROWS
    x = (rng.standard_normal((C, n)) + 1j * rng.standard_normal((C, n))).astype(np.complex64)
    k = rng.standard_normal((C, n)).astype(np.float32)
    khat = np.fft.fft(k, axis=1)
    s = np.arange(L_COLS)
    a = np.arange(M_ROWS)
    kf2 = khat[:, a[:, None] + M_ROWS * s[None, :]]  # [C][m][l] = K_hat[a + m s]
    want = np.fft.ifft(np.fft.fft(x, axis=1) * khat, axis=1)
    return x, kf2, want


def _problem_pairs(P=3, H=2, seed=1):
    """P channel pairs per head, H heads (pair-major channels), per-head kernels."""
    rng = np.random.default_rng(seed)
    n = L_COLS * M_ROWS
    x = (rng.standard_normal((P * H, n)) + 1j * rng.standard_normal((P * H, n))).astype(np.complex64)
    k = rng.standard_normal((H, n)).astype(np.float32)
    khat = np.fft.fft(k, axis=1)
    s = np.arange(L_COLS)
    a = np.arange(M_ROWS)
    kf2 = khat[:, a[:, None] + M_ROWS * s[None, :]]
    want = np.fft.ifft(np.fft.fft(x, axis=1) * np.tile(khat, (P, 1)), axis=1)
    return x, kf2, want


def _seq_worker(rank, world):
    chunks = int(os.environ.get("FB_TEST_CHUNKS", "1"))
    x, kf2, _ = _problem() if chunks == 1 else _problem_pairs()
    sh = ss.SeqShard(L_COLS, M_ROWS, world, rank)
    cols = ss.scatter_tau(torch.from_numpy(x), sh)
    y = ss.four_step_conv(cols, sh, NumpyPasses(kf2), chunks=chunks)
    np.save(os.path.join(os.environ["FB_TEST_DIR"], f"seq_{world}_{rank}.npy"), y.numpy())


@pytest.mark.parametrize("world,chunks", [(2, 1), (4, 1), (2, 3)])
def test_seq_sharded_four_step_gloo(world, chunks, monkeypatch):
    """The two all-to-all transposes (and, chunks > 1, the pipelined exchange:
    per-channel-chunk asynchronous all-to-alls) move the data so that the
    sharded circular convolution equals the single-process one."""
    d = tempfile.mkdtemp()
    monkeypatch.setenv("FB_TEST_DIR", d)
    monkeypatch.setenv("FB_TEST_CHUNKS", str(chunks))
    ss.run_ranks(world, _seq_worker, port=29571 + world + 10 * chunks)
    x, _, want = _problem() if chunks == 1 else _problem_pairs()
    sh = ss.SeqShard(L_COLS, M_ROWS, world, 0)
    parts = [torch.from_numpy(np.load(os.path.join(d, f"seq_{world}_{r}.npy"))) for r in range(world)]
    got = ss.gather_tau(parts, sh).numpy()
    assert np.abs(got - want).max() / np.abs(want).max() < 1e-5


def test_transposes_are_inverse_single_rank():
    # world 1: no exchange, identity layouts
    sh = ss.SeqShard(8, 4, 1, 0)
    x = torch.randn(2, 4, 8, dtype=torch.complex64)
    assert torch.equal(ss.scatter_tau(x.reshape(2, 32), sh), x)


def _head_worker(rank, world):
    from oracle.oracle import LcOracle

    lc = LcOracle()
    B, H, N = 2, 8, 256
    u = lc.signal_batch(1, B, H, N)
    K, D = lc.init_kernels(1, H, N, 3)
    sl = ss.head_shard(H, world, rank)
    y = lc.regularized_long_conv(u[:, sl], K[sl], D[sl], 0.003, 1)
    gathered = [torch.zeros(B, H // world, N, dtype=torch.float64) for _ in range(world)]
    torch.distributed.all_gather(gathered, torch.from_numpy(y))
    if rank == 0:
        np.save(os.path.join(os.environ["FB_TEST_DIR"], f"heads_{world}.npy"),
                torch.cat(gathered, dim=1).numpy())


@pytest.mark.parametrize("world", [2, 4])
def test_head_sharding_gloo(world, monkeypatch, lc):
    d = tempfile.mkdtemp()
    monkeypatch.setenv("FB_TEST_DIR", d)
    ss.run_ranks(world, _head_worker, port=29581 + world)
    B, H, N = 2, 8, 256
    u = lc.signal_batch(1, B, H, N)
    K, D = lc.init_kernels(1, H, N, 3)
    want = lc.regularized_long_conv(u, K, D, 0.003, 1)
    assert np.array_equal(np.load(os.path.join(d, f"heads_{world}.npy")), want)


def _layer_worker(rank, world):
    from oracle.oracle import LcOracle

    lc = LcOracle()
    B, H, N = 3, 2, L_COLS * M_ROWS // 2
    u = lc.signal_batch(1, B, H, N)
    K, D = lc.init_kernels(1, H, N, 3)
    kbar = lc.regularize_bank(K, 0.003, 1)
    sh = ss.SeqShard(L_COLS, M_ROWS, world, rank)
    u_cols = torch.from_numpy(u.reshape(B, H, M_ROWS // 2, L_COLS)[..., sh.tau0:sh.tau0 + sh.lp])
    k_cols = torch.from_numpy(kbar.reshape(H, M_ROWS // 2, L_COLS)[..., sh.tau0:sh.tau0 + sh.lp])
    y = ss.sharded_long_conv(u_cols.float(), k_cols.float(), torch.from_numpy(D).float(), sh,
                             NumpyPasses(None))
    np.save(os.path.join(os.environ["FB_TEST_DIR"], f"layer_{world}_{rank}.npy"), y.numpy())


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_layer_gloo(world, monkeypatch, lc):
    """seqshard.sharded_long_conv (pair packing, causal crop, D u, sharded kernel
    spectrum) across ranks equals the fp64 layer oracle."""
    d = tempfile.mkdtemp()
    monkeypatch.setenv("FB_TEST_DIR", d)
    ss.run_ranks(world, _layer_worker, port=29591 + world)
    B, H, N = 3, 2, L_COLS * M_ROWS // 2
    u = lc.signal_batch(1, B, H, N)
    K, D = lc.init_kernels(1, H, N, 3)
    kbar = lc.regularize_bank(K, 0.003, 1)
    want = lc.long_conv_forward(u.astype(np.float32).astype(np.float64), kbar, D.astype(np.float32))
    parts = [np.load(os.path.join(d, f"layer_{world}_{r}.npy")) for r in range(world)]
    got = np.concatenate(parts, axis=-1).reshape(B, H, N)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5


def _layer_bwd_worker(rank, world):
    from oracle.oracle import LcOracle

    lc = LcOracle()
    B, H, N = 3, 2, L_COLS * M_ROWS // 2
    u = lc.signal_batch(1, B, H, N)
    dy = lc.signal_batch(2, B, H, N)
    K, D = lc.init_kernels(1, H, N, 3)
    kbar = lc.regularize_bank(K, 0.003, 1)
    sh = ss.SeqShard(L_COLS, M_ROWS, world, rank)
    cols = lambda a: torch.from_numpy(a.reshape(*a.shape[:-1], M_ROWS // 2, L_COLS)[..., sh.tau0:sh.tau0 + sh.lp]).float()  # noqa: E731
    du, dkbar, dD = ss.sharded_long_conv_backward(cols(dy), cols(u), cols(kbar),
                                                  torch.from_numpy(D).float(), sh, NumpyPasses(None))
    d = os.environ["FB_TEST_DIR"]
    np.save(os.path.join(d, f"bdu_{world}_{rank}.npy"), du.numpy())
    np.save(os.path.join(d, f"bdk_{world}_{rank}.npy"), dkbar.numpy())
    np.save(os.path.join(d, f"bdd_{world}_{rank}.npy"), dD.numpy())


@pytest.mark.parametrize("world", [2])
def test_sharded_layer_backward_gloo(world, monkeypatch, lc):
    d = tempfile.mkdtemp()
    monkeypatch.setenv("FB_TEST_DIR", d)
    ss.run_ranks(world, _layer_bwd_worker, port=29601 + world)
    B, H, N = 3, 2, L_COLS * M_ROWS // 2
    u = lc.signal_batch(1, B, H, N).astype(np.float32).astype(np.float64)
    dy = lc.signal_batch(2, B, H, N).astype(np.float32).astype(np.float64)
    K, D = lc.init_kernels(1, H, N, 3)
    kbar = lc.regularize_bank(K, 0.003, 1)
    du_w, dkbar_w, dD_w = lc.long_conv_backward(u, dy, kbar, D.astype(np.float32))
    cat = lambda name: np.concatenate([np.load(os.path.join(d, f"{name}_{world}_{r}.npy"))  # noqa: E731
                                       for r in range(world)], axis=-1)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(cat("bdu").reshape(B, H, N), du_w) < 1e-5
    assert rel(cat("bdk").reshape(H, N), dkbar_w) < 1e-5
    for r in range(world):
        assert rel(np.load(os.path.join(d, f"bdd_{world}_{r}.npy")), dD_w) < 1e-5


def _reg_worker(rank, world):
    """Sharded regularize_bank + chain rule with the +-p halo exchange."""
    from oracle.oracle import LcOracle

    lc = LcOracle()
    H, N, p = 3, L_COLS * M_ROWS // 2, int(os.environ["FB_TEST_P"])
    K, _ = lc.init_kernels(1, H, N, 3)
    dkbar = lc.signal_batch(4, 1, H, N)[0]
    sh = ss.SeqShard(L_COLS, M_ROWS, world, rank)
    cols = lambda a: torch.from_numpy(a.reshape(H, M_ROWS // 2, L_COLS)[..., sh.tau0:sh.tau0 + sh.lp])  # noqa: E731
    kb = ss.sharded_regularize(cols(K), 0.003, p, sh)
    dk = ss.sharded_regularizer_backward(cols(K), cols(dkbar), 0.003, p, sh)
    d = os.environ["FB_TEST_DIR"]
    np.save(os.path.join(d, f"rkb_{world}_{rank}.npy"), kb.numpy())
    np.save(os.path.join(d, f"rdk_{world}_{rank}.npy"), dk.numpy())


@pytest.mark.parametrize("world,p", [(1, 1), (2, 1), (4, 1), (2, 3), (4, 16)])
def test_sharded_regularizer_halo_gloo(world, p, monkeypatch, lc):
    """sharded_regularize / sharded_regularizer_backward (halo of p columns per
    slice edge, wrapping to the neighbouring row at the first / last rank)
    reproduce regularize_bank and its chain rule on the gathered bank; p = 16
    is the whole slice at world 4 (lp = 16)."""
    d = tempfile.mkdtemp()
    monkeypatch.setenv("FB_TEST_DIR", d)
    monkeypatch.setenv("FB_TEST_P", str(p))
    if world == 1:
        _reg_worker(0, 1)
    else:
        ss.run_ranks(world, _reg_worker, port=29611 + 7 * world + p)
    H, N = 3, L_COLS * M_ROWS // 2
    K, _ = lc.init_kernels(1, H, N, 3)
    dkbar = lc.signal_batch(4, 1, H, N)[0]
    kb_w = lc.regularize_bank(K, 0.003, p)
    dk_w = lc.regularizer_backward(K, 0.003, p, dkbar)
    cat = lambda name: np.concatenate([np.load(os.path.join(d, f"{name}_{world}_{r}.npy"))  # noqa: E731
                                       for r in range(world)], axis=-1).reshape(H, N)
    # fp64 in the reference's summation order, rounded once to fp32
    assert np.array_equal(cat("rkb"), kb_w.astype(np.float32))
    assert np.array_equal(cat("rdk"), dk_w.astype(np.float32))
