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


def _a2a(x: torch.Tensor, group=None) -> torch.Tensor:
    out = torch.empty_like(x)
    dist.all_to_all_single(out, x, group=group)
    return out


def columns_to_rows(x1: torch.Tensor, shard: SeqShard, group=None) -> torch.Tensor:
    """[C, m, lp] complex (all rows, my columns) -> [C, mp, l] (my rows, all columns)."""
    C = x1.shape[0]
    P, mp, lp = shard.world, shard.mp, shard.lp
    send = x1.reshape(C, P, mp, lp).permute(1, 0, 2, 3).contiguous()  # [dest][C][mp][lp]
    recv = _a2a(torch.view_as_real(send), group)                        # [src][C][mp][lp][2]
    recv = torch.view_as_complex(recv)
    return recv.permute(1, 2, 0, 3).reshape(C, mp, P * lp).contiguous()


def rows_to_columns(rows: torch.Tensor, shard: SeqShard, group=None) -> torch.Tensor:
    """[C, mp, l] (my rows, all columns) -> [C, m, lp] (all rows, my columns)."""
    C = rows.shape[0]
    P, mp, lp = shard.world, shard.mp, shard.lp
    send = rows.reshape(C, mp, P, lp).permute(2, 0, 1, 3).contiguous()  # [dest][C][mp][lp]
    recv = torch.view_as_complex(_a2a(torch.view_as_real(send), group))  # [src][C][mp][lp]
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
