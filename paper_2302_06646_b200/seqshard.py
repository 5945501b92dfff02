"""Sequence-sharded four-step long convolution.

For N beyond one GPU's appetite the transform length n = 2N = l * m is split
across P ranks in the *block-cyclic tau layout*: with t = c * l + tau
(c < m rows, tau < l columns; the three-pass indexing of
three_pass.cpp:225-254), rank r owns the columns tau in
[r * l/P, (r+1) * l/P) of every row.  Then

    pass 1 (local)   X1[a][tau] = w_n^(-a tau) sum_c w_m^(-a c) x[c l + tau]
    all-to-all       column slices  ->  row slices (rank r owns rows a in
                     [r * m/P, (r+1) * m/P), all tau)
    pass 2 (local)   W[a] = IFFT_l(FFT_l(X1[a]) * Kf2[a])
    all-to-all       row slices  ->  column slices
    pass 3 (local)   y[c l + tau] = sum_a w_m^(+a c) w_n^(+a tau) W[a][tau]

so the forward costs exactly two all-to-alls, each moving (P-1)/P of the
intermediate (one `all_to_all_single` over NCCL / NVLink, equal splits).
The exchange is implemented here; the local passes are supplied by the
caller (`LocalPasses`): on the GPU they are the three-pass column/row
kernels, in the CPU tests a numpy restatement checks the data movement.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Protocol

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class SeqShard:
    """Geometry of one rank's share of an n = l * m transform."""

    l: int
    m: int
    world: int
    rank: int

    def __post_init__(self):
        if self.l % self.world or self.m % self.world:
            raise ValueError("l and m must be divisible by the world size")

    @property
    def lp(self) -> int:  # local columns
        return self.l // self.world

    @property
    def mp(self) -> int:  # local rows after the transpose
        return self.m // self.world

    @property
    def tau0(self) -> int:
        return self.rank * self.lp

    @property
    def a0(self) -> int:
        return self.rank * self.mp


def scatter_tau(x: torch.Tensor, shard: SeqShard) -> torch.Tensor:
    """Global [..., n] (t = c l + tau) -> this rank's columns [..., m, lp]."""
    v = x.reshape(*x.shape[:-1], shard.m, shard.l)
    return v[..., shard.tau0:shard.tau0 + shard.lp].contiguous()


def gather_tau(parts: list[torch.Tensor], shard: SeqShard) -> torch.Tensor:
    """Inverse of scatter_tau over all ranks' [..., m, lp] parts."""
    v = torch.cat(parts, dim=-1)
    return v.reshape(*v.shape[:-2], shard.m * shard.l)


def _a2a(x: torch.Tensor, group=None, world: int = 2) -> torch.Tensor:
    if world == 1:  # one rank: the transpose moves nothing (no process group needed)
        return x
    out = torch.empty_like(x)
    dist.all_to_all_single(out, x, group=group)
    return out


def columns_to_rows(x1: torch.Tensor, shard: SeqShard, group=None) -> torch.Tensor:
    """[C, m, lp] complex (all rows, my columns) -> [C, mp, l] (my rows, all columns)."""
    C = x1.shape[0]
    P, mp, lp = shard.world, shard.mp, shard.lp
    send = x1.reshape(C, P, mp, lp).permute(1, 0, 2, 3).contiguous()  # [dest][C][mp][lp]
    recv = _a2a(torch.view_as_real(send), group, P)                     # [src][C][mp][lp][2]
    recv = torch.view_as_complex(recv)
    return recv.permute(1, 2, 0, 3).reshape(C, mp, P * lp).contiguous()


def rows_to_columns(rows: torch.Tensor, shard: SeqShard, group=None) -> torch.Tensor:
    """[C, mp, l] (my rows, all columns) -> [C, m, lp] (all rows, my columns)."""
    C = rows.shape[0]
    P, mp, lp = shard.world, shard.mp, shard.lp
    send = rows.reshape(C, mp, P, lp).permute(2, 0, 1, 3).contiguous()  # [dest][C][mp][lp]
    recv = torch.view_as_complex(_a2a(torch.view_as_real(send), group, P))  # [src][C][mp][lp]
    return recv.permute(1, 0, 2, 3).reshape(C, P * mp, lp).contiguous()


class LocalPasses(Protocol):
    def pass1(self, x_cols: torch.Tensor, shard: SeqShard) -> torch.Tensor: ...
    def pass2(self, rows: torch.Tensor, shard: SeqShard) -> torch.Tensor: ...
    def pass3(self, w_cols: torch.Tensor, shard: SeqShard) -> torch.Tensor: ...


def four_step_conv(x_cols: torch.Tensor, shard: SeqShard, passes: LocalPasses,
                   group=None) -> torch.Tensor:
    """Circular convolution of length n = l m of the sharded signals
    x_cols [C, m, lp] (complex; two real channels per complex as elsewhere)
    with the kernel held by `passes`; returns this rank's output columns."""
    x1 = passes.pass1(x_cols, shard)
    rows = columns_to_rows(x1, shard, group)
    rows = passes.pass2(rows, shard)
    w = rows_to_columns(rows, shard, group)
    return passes.pass3(w, shard)


class GpuPasses:
    """The three local passes on this rank's GPU with this package's kernels
    (fb_shard_columns / fb_shard_rows in libflashbutterfly.so): complex64
    [C, m, lp] column slices and [C, mp, l] row slices, l = 8192.  `kf2` holds
    this rank's rows of the kernel spectrum, kf2[c][a - a0][s] = K_hat[a + m s]."""

    def __init__(self, n: int, kf2: torch.Tensor | None = None, device=None):
        import ctypes as C

        from . import _lib

        self._C, self._lib = C, _lib
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.device, self.n = dev, int(n)
        h = C.c_void_p()
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().fb_shard_plan_create(C.byref(h), self.n, dev.index or 0))
        self._h = h
        l, m = C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().fb_shard_plan_dims(h, C.byref(l), C.byref(m)))
        self.l, self.m = l.value, m.value
        self.kf2 = kf2

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.lib().fb_shard_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def _p(self, t):
        return self._C.c_void_p(t.data_ptr()) if t is not None else self._C.c_void_p(0)

    def _stream(self):
        return self._C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _cols(self, x: torch.Tensor, sh: SeqShard, inverse: int) -> torch.Tensor:
        x = x.contiguous()
        if x.dtype != torch.complex64 or tuple(x.shape[1:]) != (sh.m, sh.lp):
            raise ValueError(f"expected complex64 [C, {sh.m}, {sh.lp}], got {x.dtype} {list(x.shape)}")
        out = torch.empty_like(x)
        self._lib.check(self._lib.lib().fb_shard_columns(self._h, self._p(x), self._p(out), x.shape[0],
                                                         sh.tau0, sh.lp, inverse, self._stream()))
        return out

    def pass1(self, x_cols: torch.Tensor, sh: SeqShard) -> torch.Tensor:
        return self._cols(x_cols, sh, 0)

    def pass3(self, w_cols: torch.Tensor, sh: SeqShard) -> torch.Tensor:
        return self._cols(w_cols, sh, 1)

    def pass2(self, rows: torch.Tensor, sh: SeqShard) -> torch.Tensor:
        rows = rows.contiguous()
        kf2 = self.kf2.contiguous()
        self._lib.check(self._lib.lib().fb_shard_rows(self._h, self._p(rows), self._p(kf2), None,
                                                      rows.shape[0], sh.mp, 0, 1.0, self._stream()))
        return rows

    def rows_fft(self, rows: torch.Tensor, sh: SeqShard) -> torch.Tensor:
        """FFT_l of each row [C, mp, l] (fb_shard_rows, spectrum mode)."""
        rows = rows.contiguous()
        out = torch.empty_like(rows)
        self._lib.check(self._lib.lib().fb_shard_rows(self._h, self._p(rows), None, self._p(out),
                                                      rows.shape[0], sh.mp, 1, 1.0, self._stream()))
        return out

    def rows_ifft(self, rows: torch.Tensor, sh: SeqShard) -> torch.Tensor:
        """Unnormalised inverse FFT_l of each row: conj(FFT_l(conj(rows)))."""
        return torch.conj(self.rows_fft(torch.conj(rows).resolve_conj(), sh)).resolve_conj()

    def spectrum_rows(self, kbar_cols: torch.Tensor, sh: SeqShard, group=None) -> torch.Tensor:
        """This rank's kernel-spectrum rows from its real kernel columns
        kbar_cols [C, m, lp] (float32; zero-padded causal kernels): pass 1,
        the transpose, then the row FFTs — the sharded build_three_pass
        (three_pass.cpp:197-203).  Sets and returns self.kf2."""
        x = torch.complex(kbar_cols.float(), torch.zeros_like(kbar_cols, dtype=torch.float32))
        rows = columns_to_rows(self.pass1(x, sh), sh, group)
        kf2 = torch.empty_like(rows)
        self._lib.check(self._lib.lib().fb_shard_rows(self._h, self._p(rows), None, self._p(kf2),
                                                      rows.shape[0], sh.mp, 1, 1.0, self._stream()))
        self.kf2 = kf2
        return kf2


def sharded_long_conv(u_cols: torch.Tensor, kbar_cols: torch.Tensor, D: torch.Tensor,
                      shard: SeqShard, passes: "GpuPasses", group=None) -> torch.Tensor:
    """The layer forward y = conv_causal(u, Kbar) + D u (regularize.cpp:185-187)
    with the sequence sharded: rank r holds the tau-slice [tau0, tau0 + lp) of
    every data row c < m/2 of t = c l + tau (N = n / 2 causal; rows c >= m/2
    are the zero pad and are not stored).
      u_cols [B, H, m/2, lp] real, kbar_cols [H, m/2, lp] fp32 (regularized),
      D [H]  ->  y_cols [B, H, m/2, lp] (u's dtype).
    Two real channels ride as re / im of one complex transform (batch-pair
    packing, as on a single GPU); the kernel spectrum is built sharded with the
    same passes (two all-to-alls), the convolution costs two more."""
    B, H, half, lp = u_cols.shape
    m = shard.m
    if half * 2 != m or lp != shard.lp or kbar_cols.shape != (H, half, lp):
        raise ValueError("sharded_long_conv: expected u [B, H, m/2, lp] and Kbar [H, m/2, lp]")
    dev = u_cols.device
    kpad = torch.zeros(H, m, lp, dtype=torch.float32, device=dev)
    kpad[:, :half] = kbar_cols.float()
    kf2 = passes.spectrum_rows(kpad, shard, group)  # [H, mp, l]
    P = (B + 1) // 2
    uf = u_cols.float()
    if B % 2:
        uf = torch.cat([uf, torch.zeros_like(uf[:1])], 0)
    x = torch.zeros(P, H, m, lp, dtype=torch.complex64, device=dev)
    x[:, :, :half] = torch.complex(uf[0::2], uf[1::2])
    passes.kf2 = kf2.repeat(P, 1, 1)  # channel (p, h) uses head h's rows
    y = four_step_conv(x.reshape(P * H, m, lp), shard, passes, group).reshape(P, H, m, lp)
    y = y[:, :, :half]
    out = torch.stack([y.real, y.imag], 1).reshape(2 * P, H, half, lp)[:B]
    out = out + D.float().view(1, H, 1, 1) * u_cols.float()
    return out.to(u_cols.dtype)


def _pack_pairs(sig_cols: torch.Tensor, m: int) -> torch.Tensor:
    """[B, H, m/2, lp] real -> [P*H, m, lp] complex (channels 2p, 2p+1 -> re, im;
    rows c >= m/2 are the causal zero pad)."""
    B, H, half, lp = sig_cols.shape
    P = (B + 1) // 2
    f = sig_cols.float()
    if B % 2:
        f = torch.cat([f, torch.zeros_like(f[:1])], 0)
    x = torch.zeros(P, H, m, lp, dtype=torch.complex64, device=sig_cols.device)
    x[:, :, :half] = torch.complex(f[0::2], f[1::2])
    return x.reshape(P * H, m, lp)


def _unpack_pairs(y: torch.Tensor, B: int, H: int, half: int) -> torch.Tensor:
    P = (B + 1) // 2
    y = y.reshape(P, H, -1, y.shape[-1])[:, :, :half]
    return torch.stack([y.real, y.imag], 1).reshape(2 * P, H, half, y.shape[-1])[:B]


def sharded_long_conv_backward(dy_cols: torch.Tensor, u_cols: torch.Tensor,
                               kbar_cols: torch.Tensor, D: torch.Tensor, shard: SeqShard,
                               passes: "GpuPasses", group=None):
    """Backward of sharded_long_conv (SURVEY.md §8c formulas, sequence sharded):
      du     = corr(dy, Kbar) + D dy   -> IFFT(DY conj(K_hat)), causal crop
      dKbar  = sum_b corr(dy_b, u_b)   -> Re IFFT(sum_pairs conj(U) DY), lag < N
      dD     = dKbar[0]                 (lag 0, held by the rank with tau0 = 0)
    Layouts as in sharded_long_conv; returns (du_cols [B, H, m/2, lp],
    dkbar_cols [H, m/2, lp] fp32, dD [H] fp32).  The chain rule through the
    regularizers to dK is sharded_regularizer_backward (halo exchange of the
    +-p smoothing neighbours across slices)."""
    B, H, half, lp = u_cols.shape
    m = shard.m
    dev = u_cols.device
    kpad = torch.zeros(H, m, lp, dtype=torch.float32, device=dev)
    kpad[:, :half] = kbar_cols.float()
    kf2 = passes.spectrum_rows(kpad, shard, group)  # [H, mp, l] (K_hat rows)
    P = (B + 1) // 2
    xdy = _pack_pairs(dy_cols, m)
    xu = _pack_pairs(u_cols, m)
    # row spectra of dy and u (pass 1, transpose, row FFT)
    DY = passes.rows_fft(columns_to_rows(passes.pass1(xdy, shard), shard, group), shard)
    U = passes.rows_fft(columns_to_rows(passes.pass1(xu, shard), shard, group), shard)
    # du: DY conj(K_hat), inverse rows, transpose back, pass 3
    kc = torch.conj(kf2).resolve_conj().repeat(P, 1, 1)
    du_rows = passes.rows_ifft(DY * kc, shard)
    du = _unpack_pairs(passes.pass3(rows_to_columns(du_rows, shard, group), shard), B, H, half)
    du = du + D.float().view(1, H, 1, 1) * dy_cols.float()
    # dKbar: sum over the pairs of each head, then the inverse transform
    S = (torch.conj(U) * DY).reshape(P, H, shard.mp, shard.l).sum(0)
    dk = passes.pass3(rows_to_columns(passes.rows_ifft(S, shard), shard, group), shard)
    dkbar = dk.real[:, :half].contiguous()
    dD = dkbar[:, 0, 0].clone() if shard.tau0 == 0 else torch.zeros(H, device=dev)
    if shard.world > 1:
        dist.all_reduce(dD, group=group)
    return du.to(dy_cols.dtype), dkbar, dD


def _halo(x_cols: torch.Tensor, p: int, shard: SeqShard, group=None) -> torch.Tensor:
    """[H, rows, lp] slices of t = c l + tau -> [H, rows, lp + 2p] with the p
    neighbours on either side of every row of the slice: the left halo of row
    c comes from rank r-1's last p columns of row c (rank 0: rank P-1's row
    c-1), the right halo from rank r+1's first p columns of row c (rank P-1:
    rank 0's row c+1); zero beyond t = 0 and t = rows * l (the zero-padded
    window of regularize.cpp:22-34)."""
    H, R, lp = x_cols.shape
    if p == 0:
        return x_cols
    if p > lp:
        raise ValueError(f"smooth width {p} exceeds the slice width {lp}")
    edges = torch.cat([x_cols[..., :p], x_cols[..., lp - p:]], -1).contiguous()  # [H, R, 2p]
    P, r = shard.world, shard.rank
    if P == 1:
        parts = [edges]
    else:
        parts = [torch.empty_like(edges) for _ in range(P)]
        dist.all_gather(parts, edges, group=group)
    zrow = torch.zeros_like(edges[:, :1, :p])
    lft = parts[r - 1][..., p:] if r > 0 else torch.cat([zrow, parts[P - 1][:, :-1, p:]], 1)
    rgt = parts[r + 1][..., :p] if r < P - 1 else torch.cat([parts[0][:, 1:, :p], zrow], 1)
    return torch.cat([lft, x_cols, rgt], -1)


def _smooth_sharded(x_cols: torch.Tensor, p: int, shard: SeqShard, group=None) -> torch.Tensor:
    """smooth (regularize.cpp:22-34): zero-padded window mean over |j - i| <= p,
    on the sharded layout (halo exchange of p columns per slice edge)."""
    if p == 0:
        return x_cols.clone()
    xp = _halo(x_cols, p, shard, group)
    lp = x_cols.shape[-1]
    acc = xp[..., 0:lp].clone()
    for d in range(1, 2 * p + 1):
        acc += xp[..., d:d + lp]
    return acc * (1.0 / (2 * p + 1))


def sharded_regularize(k_cols: torch.Tensor, lam: float, p: int, shard: SeqShard,
                       group=None) -> torch.Tensor:
    """regularize_bank (regularize.cpp:93-107, time-domain smooth, no dropout)
    on the sharded layout: Kbar = squash(smooth(K)).  k_cols [H, m/2, lp]
    (raw kernels, any float dtype) -> fp32 Kbar slices; computed in fp64."""
    s = _smooth_sharded(k_cols.double(), p, shard, group)
    mag = s.abs() - lam
    return torch.where(mag > 0, torch.copysign(mag, s), torch.zeros_like(s)).float()


def sharded_regularizer_backward(k_cols: torch.Tensor, dkbar_cols: torch.Tensor, lam: float,
                                 p: int, shard: SeqShard, group=None) -> torch.Tensor:
    """Chain rule of sharded_regularize: smooth is a symmetric
    zero-padded band (self-adjoint) and squash' = 1[|smooth(K)| > lam], so
    dK = smooth(1[|smooth(K)| > lam] * dKbar) — two halo exchanges.  Returns
    fp32 dK slices [H, m/2, lp] w.r.t. the raw K."""
    s = _smooth_sharded(k_cols.double(), p, shard, group)
    g = torch.where(s.abs() > lam, dkbar_cols.double(), torch.zeros_like(s))
    return _smooth_sharded(g, p, shard, group).float()


def head_shard(H: int, world: int, rank: int) -> slice:
    """Heads owned by `rank` under B*H sharding (contiguous, no collective:
    K, D, dK, dD are head-local, regularize.cpp:177-188)."""
    if H % world:
        raise ValueError(f"H={H} must be divisible by the world size {world}")
    per = H // world
    return slice(rank * per, (rank + 1) * per)


def _rank_entry(rank, world, port, fn, backend):
    import os

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        fn(rank, world)
    finally:
        dist.destroy_process_group()


def run_ranks(world: int, fn: Callable[[int, int], None], port: int = 29561,
              backend: str = "gloo") -> None:
    """Spawn `world` ranks on 127.0.0.1 and run fn(rank, world) in each
    (fn must be a picklable top-level function)."""
    import torch.multiprocessing as mp

    mp.spawn(_rank_entry, args=(world, port, fn, backend), nprocs=world, join=True)
