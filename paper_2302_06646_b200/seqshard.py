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


def _a2a(x: torch.Tensor, group=None, world: int = 2, async_op: bool = False):
    """Equal-split all-to-all of a flat staging buffer (rank-major blocks)."""
    if world == 1:  # one rank: the transpose moves nothing (no process group needed)
        return (x, None) if async_op else x
    out = torch.empty_like(x)
    work = dist.all_to_all_single(out, x, group=group, async_op=async_op)
    return (out, work) if async_op else out


# The all-to-all transposes.  The local re-layouts around the exchange are
# `passes.stage` calls (GpuPasses: the fb_shard_stage kernel, which also
# converts to the wire type — "bf16" halves the NVLink bytes of each exchange).
# (one rank: both layouts are the identity, nothing is staged or exchanged)
def _c2r_send(x1, shard, passes, wire):
    if shard.world == 1:
        return x1
    C = x1.shape[0]
    return passes.stage(x1, C, shard.world, shard.mp * shard.lp, wire)   # [dest][C][mp lp]


def _c2r_recv(recv, C, shard, passes):
    P, mp, lp = shard.world, shard.mp, shard.lp
    if P == 1:
        return recv.reshape(C, mp, lp)
    return passes.stage(recv, P, C * mp, lp, "f32").reshape(C, mp, P * lp)  # [C][mp][src lp]


def _r2c_send(rows, shard, passes, wire):
    if shard.world == 1:
        return rows
    C = rows.shape[0]
    return passes.stage(rows, C * shard.mp, shard.world, shard.lp, wire)  # [dest][C mp][lp]


def _r2c_recv(recv, C, shard, passes):
    P, mp, lp = shard.world, shard.mp, shard.lp
    if P == 1:
        return recv.reshape(C, mp, lp)
    return passes.stage(recv, P, C, mp * lp, "f32").reshape(C, P * mp, lp)  # [C][src mp][lp]


def columns_to_rows(x1: torch.Tensor, shard: SeqShard, group=None, passes=None,
                    wire: str = "f32") -> torch.Tensor:
    """[C, m, lp] complex (all rows, my columns) -> [C, mp, l] (my rows, all columns)."""
    C = x1.shape[0]
    return _c2r_recv(_a2a(_c2r_send(x1, shard, passes, wire), group, shard.world), C, shard, passes)


def rows_to_columns(rows: torch.Tensor, shard: SeqShard, group=None, passes=None,
                    wire: str = "f32") -> torch.Tensor:
    """[C, mp, l] (my rows, all columns) -> [C, m, lp] (all rows, my columns)."""
    C = rows.shape[0]
    return _r2c_recv(_a2a(_r2c_send(rows, shard, passes, wire), group, shard.world), C, shard, passes)


class LocalPasses(Protocol):
    def pass1(self, x_cols: torch.Tensor, shard: SeqShard) -> torch.Tensor: ...
    def pass2(self, rows: torch.Tensor, shard: SeqShard) -> torch.Tensor: ...
    def pass3(self, w_cols: torch.Tensor, shard: SeqShard) -> torch.Tensor: ...
    def stage(self, t: torch.Tensor, A: int, Bd: int, X: int, wire: str) -> torch.Tensor: ...


def four_step_conv(x_cols: torch.Tensor | None, shard: SeqShard, passes: LocalPasses,
                   group=None, wire: str = "f32", chunks: int = 1, C: int | None = None,
                   first=None, last=None):
    """Circular convolution of length n = l m of the sharded signals
    x_cols [C, m, lp] (complex; two real channels per complex as elsewhere)
    with the kernel held by `passes`; returns this rank's output columns.
    `chunks` > 1 splits the channels (whole pairs) so that chunk i's
    all-to-alls (NCCL, asynchronous) overlap the local passes of its
    neighbours.  `first(a, b)` / `last(w, a, b)` replace pass 1 / pass 3 of
    channels [a, b) (the layer's fused signal-side passes); the outputs of
    `last` are concatenated along dim 0."""
    C = x_cols.shape[0] if C is None else C
    first = first or (lambda a, b: passes.pass1(x_cols[a:b], shard))
    last = last or (lambda w, a, b: passes.pass3(w, shard))
    # chunks of whole channel pairs (the kernel rows are shared per head)
    H = passes.kf2.shape[0] if getattr(passes, "kf2", None) is not None else C
    units = max(1, C // H)
    chunks = max(1, min(chunks, units))
    bounds = [H * (units * i // chunks) for i in range(chunks)] + [C]
    parts = [(a, b) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    P = shard.world
    sent = []
    for a, b in parts:  # pass 1 + the outbound exchange, issued back to back
        sent.append(_a2a(_c2r_send(first(a, b), shard, passes, wire), group, P, True))
    back = []
    for (a, b), (recv, work) in zip(parts, sent):
        if work is not None:
            work.wait()
        rows = passes.pass2(_c2r_recv(recv, b - a, shard, passes), shard)
        back.append(_a2a(_r2c_send(rows, shard, passes, wire), group, P, True))
    out = []
    for (a, b), (recv, work) in zip(parts, back):
        if work is not None:
            work.wait()
        out.append(last(_r2c_recv(recv, b - a, shard, passes), a, b))
    return out[0] if len(out) == 1 else torch.cat(out, 0)


class GpuPasses:
    """The local passes and the glue on this rank's GPU with this package's
    kernels (libflashbutterfly.so: fb_shard_columns(_from_signals /
    _to_signals: pair packing and the D u skip fused) / fb_shard_rows_pairs /
    fb_shard_rows_bwd for the passes, fb_shard_stage for the all-to-all
    layouts): complex64 [C, m, lp] column slices and [C, mp, l]
    row slices, l = 8192, C = P * H channels (pair-major).  `kf2` holds this
    rank's rows of the kernel spectrum, kf2[h][a - a0][s] = K_hat[a + m s],
    shared by the P channel pairs of head h."""

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

    def _call(self, name, *args):
        self._lib.check(getattr(self._lib.lib(), name)(*args))

    def _cols(self, x: torch.Tensor, sh: SeqShard, inverse: int) -> torch.Tensor:
        x = x.contiguous()
        if x.dtype != torch.complex64 or tuple(x.shape[1:]) != (sh.m, sh.lp):
            raise ValueError(f"expected complex64 [C, {sh.m}, {sh.lp}], got {x.dtype} {list(x.shape)}")
        out = torch.empty_like(x)
        self._call("fb_shard_columns", self._h, self._p(x), self._p(out), x.shape[0], sh.tau0, sh.lp,
                   inverse, self._stream())
        return out

    def pass1(self, x_cols: torch.Tensor, sh: SeqShard) -> torch.Tensor:
        return self._cols(x_cols, sh, 0)

    def pass3(self, w_cols: torch.Tensor, sh: SeqShard) -> torch.Tensor:
        return self._cols(w_cols, sh, 1)

    def pass1_signals(self, sig: torch.Tensor, sh: SeqShard) -> torch.Tensor:
        """Pass 1 of the channel pairs straight from real signals [B, H, m/2, lp]
        (pairs packed on the fly, causal zero rows implied) -> [P*H, m, lp]."""
        sig = sig.contiguous()
        B, H, half, lp = sig.shape
        out = torch.empty(((B + 1) // 2) * H, sh.m, lp, dtype=torch.complex64, device=self.device)
        self._call("fb_shard_columns_from_signals", self._h, self._p(sig), self._DT[sig.dtype], self._p(out),
                   B, H, half, sh.tau0, lp, self._stream())
        return out

    def pass3_signals(self, w: torch.Tensor, sh: SeqShard, B: int, H: int, half: int, skip=None, D=None,
                      dtype=torch.float32) -> torch.Tensor:
        """Pass 3 of [P*H, m, lp] straight into real signals [B, H, m/2, lp]
        (+ D[h] skip), in `dtype`."""
        w = w.contiguous()
        out = torch.empty(B, H, half, sh.lp, dtype=dtype, device=self.device)
        if skip is not None:
            skip = skip.to(dtype).contiguous()
            D = D.float().contiguous()
        self._call("fb_shard_columns_to_signals", self._h, self._p(w), self._p(out), self._DT[dtype],
                   self._p(skip), self._p(D), B, H, half, sh.tau0, sh.lp, self._stream())
        return out

    def pass2(self, rows: torch.Tensor, sh: SeqShard) -> torch.Tensor:
        """Rows [P*H, mp, l] in place against the heads' kernel rows (no copies per pair)."""
        rows = rows.contiguous()
        H = self.kf2.shape[0]
        self._call("fb_shard_rows_pairs", self._h, self._p(rows), self._p(self.kf2.contiguous()),
                   rows.shape[0] // H, H, sh.mp, self._stream())
        return rows

    def rows_bwd(self, dy_rows: torch.Tensor, u_rows: torch.Tensor, sh: SeqShard):
        """du rows = IFFT(DY conj(kf2)) in place, and the heads' dK spectrum rows
        IFFT(sum_pairs conj(U) DY) [H, mp, l] (fused, fixed order)."""
        H = self.kf2.shape[0]
        dy_rows, u_rows = dy_rows.contiguous(), u_rows.contiguous()
        wdk = torch.empty(H, sh.mp, sh.l, dtype=torch.complex64, device=self.device)
        self._call("fb_shard_rows_bwd", self._h, self._p(dy_rows), self._p(u_rows),
                   self._p(self.kf2.contiguous()), self._p(wdk), dy_rows.shape[0] // H, H, sh.mp,
                   self._stream())
        return dy_rows, wdk

    def rows_fft(self, rows: torch.Tensor, sh: SeqShard) -> torch.Tensor:
        """FFT_l of each row [C, mp, l] (fb_shard_rows, spectrum mode)."""
        rows = rows.contiguous()
        out = torch.empty_like(rows)
        self._call("fb_shard_rows", self._h, self._p(rows), None, self._p(out), rows.shape[0], sh.mp, 1,
                   self._C.c_float(1.0), self._stream())
        return out

    def stage(self, t: torch.Tensor, A: int, Bd: int, X: int, wire: str) -> torch.Tensor:
        """out[b][a][x] = t[a][b][x] (complex elements) as a flat wire buffer."""
        t = t.contiguous()
        in_dt = self._lib.FB_F32 if t.dtype == torch.complex64 else self._lib.FB_BF16
        if wire == "f32":
            out = torch.empty(A * Bd * X, dtype=torch.complex64, device=self.device)
            out_dt = self._lib.FB_F32
        else:
            out = torch.empty(2 * A * Bd * X, dtype=torch.bfloat16, device=self.device)
            out_dt = self._lib.FB_BF16
        self._call("fb_shard_stage", self._p(t), self._p(out), A, Bd, X, in_dt, out_dt, self._stream())
        return out

    _DT = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}

    def spectrum_rows(self, kbar_cols: torch.Tensor, sh: SeqShard, group=None,
                      wire: str = "f32") -> torch.Tensor:
        """This rank's kernel-spectrum rows from its real kernel columns
        kbar_cols [H, m/2, lp] (regularized, the causal zero rows implied):
        pass 1, the transpose, then the row FFTs — the sharded build_three_pass
        (three_pass.cpp:197-203).  Sets and returns self.kf2 [H, mp, l]."""
        x = self.pass1_signals(kbar_cols.float().unsqueeze(0), sh)  # one "batch": re = Kbar, im = 0
        rows = columns_to_rows(x, sh, group, self, wire)
        self.kf2 = self.rows_fft(rows, sh)
        return self.kf2


def sharded_long_conv(u_cols: torch.Tensor, kbar_cols: torch.Tensor, D: torch.Tensor,
                      shard: SeqShard, passes: "GpuPasses", group=None, wire: str = "f32",
                      chunks: int = 1) -> torch.Tensor:
    """The layer forward y = conv_causal(u, Kbar) + D u (regularize.cpp:185-187)
    with the sequence sharded: rank r holds the tau-slice [tau0, tau0 + lp) of
    every data row c < m/2 of t = c l + tau (N = n / 2 causal; rows c >= m/2
    are the zero pad and are not stored).
      u_cols [B, H, m/2, lp] real, kbar_cols [H, m/2, lp] fp32 (regularized),
      D [H]  ->  y_cols [B, H, m/2, lp] (u's dtype).
    Two real channels ride as re / im of one complex transform (batch-pair
    packing, as on a single GPU); the kernel spectrum is built sharded with the
    same passes (two all-to-alls), the convolution costs two more.  All glue
    (packing, staging, unpack with D u) runs in the passes' kernels."""
    B, H, half, lp = u_cols.shape
    if half * 2 != shard.m or lp != shard.lp or kbar_cols.shape != (H, half, lp):
        raise ValueError("sharded_long_conv: expected u [B, H, m/2, lp] and Kbar [H, m/2, lp]")
    passes.spectrum_rows(kbar_cols, shard, group, wire)  # [H, mp, l]

    def first(a, b):  # channels [a, b) = pairs [a/H, b/H) = batches [2a/H, 2b/H)
        return passes.pass1_signals(u_cols[2 * a // H:min(B, 2 * b // H)], shard)

    def last(w, a, b):
        b0, b1 = 2 * a // H, min(B, 2 * b // H)
        return passes.pass3_signals(w, shard, b1 - b0, H, half, skip=u_cols[b0:b1], D=D, dtype=u_cols.dtype)

    return four_step_conv(None, shard, passes, group, wire, chunks, C=((B + 1) // 2) * H, first=first,
                          last=last)


def sharded_long_conv_backward(dy_cols: torch.Tensor, u_cols: torch.Tensor,
                               kbar_cols: torch.Tensor, D: torch.Tensor, shard: SeqShard,
                               passes: "GpuPasses", group=None, wire: str = "f32"):
    """Backward of sharded_long_conv (SURVEY.md §8c formulas, sequence sharded):
      du     = corr(dy, Kbar) + D dy   -> IFFT(DY conj(K_hat)), causal crop
      dKbar  = sum_b corr(dy_b, u_b)   -> Re IFFT(sum_pairs conj(U) DY), lag < N
      dD     = dKbar[0]                 (lag 0, held by the rank with tau0 = 0)
    Layouts as in sharded_long_conv; returns (du_cols [B, H, m/2, lp],
    dkbar_cols [H, m/2, lp] fp32, dD [H] fp32).  The row pass (both spectra,
    du rows, the dK spectrum summed over pairs in a fixed order, its inverse)
    is one fused kernel (fb_shard_rows_bwd).  The chain rule through the
    regularizers to dK is sharded_regularizer_backward (halo exchange)."""
    B, H, half, lp = u_cols.shape
    dev = u_cols.device
    passes.spectrum_rows(kbar_cols, shard, group, wire)  # [H, mp, l] (K_hat rows)
    rdy = columns_to_rows(passes.pass1_signals(dy_cols, shard), shard, group, passes, wire)
    ru = columns_to_rows(passes.pass1_signals(u_cols, shard), shard, group, passes, wire)
    du_rows, wdk = passes.rows_bwd(rdy, ru, shard)
    du = passes.pass3_signals(rows_to_columns(du_rows, shard, group, passes, wire), shard, B, H, half,
                              skip=dy_cols, D=D, dtype=dy_cols.dtype)
    # the dK rows: one "batch" per head, the real part is dKbar
    dkbar = passes.pass3_signals(rows_to_columns(wdk, shard, group, passes, wire), shard, 1, H, half)[0]
    dD = dkbar[:, 0, 0].clone() if shard.tau0 == 0 else torch.zeros(H, device=dev)
    if shard.world > 1:
        dist.all_reduce(dD, group=group)
    return du, dkbar, dD


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
