"""Multi-GPU layer: one process per GPU (torch.distributed; NCCL on B200s).

SURVEY.md section 8e:
  * configs 2-4 (independent vectors / images): the batch is sharded across
    ranks (`shard_batch`); there is no data-path collective.
  * config 5 (one 4096^2 image, 50 x U*U): rows are partitioned across ranks
    and every separable pass exchanges an all-to-all transpose
    (`RowPartitioned2D`).  With A = U W^-1 the N x M 1D composed operator:

        forward  Y = A X A^T :  rows  T = X_r A^T      (local, M/P x N)
                                all-to-all  T -> T_c    (M x N/P, columns)
                                cols  Y_c = A T_c       (local, N x N/P)
        adjoint  X = A^T Y A :  cols  T_c = A^T Y_c     (local, M x N/P)
                                all-to-all  T_c -> T    (M/P x N, rows)
                                rows  X_r = T A          (local, M/P x M)

    so the normal operator U*U keeps X row-partitioned and moves 2 x M x N
    doubles through the network per iteration.

    With the banded normal form (A*A = N1 (x) N1, N1 = W (U*U) W^-1 applied
    by `apply_normal_1d` to rows), an iteration is
        rows X_r <- X_r N1  (local),  distributed transpose,
        rows     <- . N1    (local),  distributed transpose back,
    moving 2 x M^2 doubles per iteration instead of 2 x M x N.

The local 1D passes are a callable `apply_1d(batch_rows, adjoint) -> rows`
(the GPU ComposedOp on CUDA tensors in production; any host implementation
in the CPU tests), so the partition / exchange logic is backend-neutral and
is tested with the gloo backend at world_size 2.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_batch(batch: int, rank: int, world: int) -> Tuple[int, int]:
    """(start, count) of the contiguous batch slice owned by `rank`."""
    base, rem = divmod(batch, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def _all_to_all_blocks(blocks, group=None):
    """Exchange equal-size blocks: blocks[q] goes to rank q; returns the
    blocks received, indexed by source rank."""
    world = len(blocks)
    send = torch.cat([b.reshape(-1) for b in blocks])
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    n = send.numel() // world
    return [recv[q * n:(q + 1) * n] for q in range(world)]


class RowPartitioned2D:
    """Separable 2D operator Y = A X A^T with X row-partitioned over ranks.

    apply_1d(v, adjoint): applies A (adjoint=False: length M -> N) or A^T
    (length N -> M) to each row of the 2D tensor v."""

    def __init__(self, M: int, N: int, apply_1d: Callable[[torch.Tensor, bool], torch.Tensor],
                 group=None, apply_normal_1d: Optional[Callable[[torch.Tensor], torch.Tensor]] = None):
        self.M, self.N = M, N
        self.apply_1d = apply_1d
        self.apply_normal_1d = apply_normal_1d
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if M % self.world or N % self.world:
            raise ValueError("M and N must be divisible by the world size")
        self.mr, self.nc = M // self.world, N // self.world

    def forward(self, x_rows: torch.Tensor) -> torch.Tensor:
        """x_rows: (M/P, M) local rows of X -> (N, N/P) local columns of Y."""
        P, mr, nc = self.world, self.mr, self.nc
        t = self.apply_1d(x_rows, False)                                     # (M/P, N)
        blocks = [t[:, q * nc:(q + 1) * nc].contiguous() for q in range(P)]
        got = _all_to_all_blocks(blocks, self.group)                           # P x (M/P * N/P)
        t_cols = torch.cat([g.view(mr, nc) for g in got], dim=0)               # (M, N/P)
        y_cols = self.apply_1d(t_cols.t().contiguous(), False)                 # (N/P, N): columns of Y
        return y_cols.t().contiguous()                                         # (N, N/P)

    def adjoint(self, y_cols: torch.Tensor) -> torch.Tensor:
        """y_cols: (N, N/P) local columns of Y -> (M/P, M) local rows of X."""
        P, mr, nc = self.world, self.mr, self.nc
        t_cols = self.apply_1d(y_cols.t().contiguous(), True).t().contiguous()  # (M, N/P)
        blocks = [t_cols[q * mr:(q + 1) * mr, :].contiguous() for q in range(P)]
        got = _all_to_all_blocks(blocks, self.group)
        t_rows = torch.cat([g.view(mr, nc) for g in got], dim=1)               # (M/P, N)
        return self.apply_1d(t_rows, True)                                     # (M/P, M)

    def transpose(self, x_rows: torch.Tensor) -> torch.Tensor:
        """Distributed transpose of the row-partitioned M x M matrix: rank p
        sends block X[p rows, q cols] to rank q and receives X[q rows, p cols]."""
        P, mr = self.world, self.mr
        blocks = [x_rows[:, q * mr:(q + 1) * mr].contiguous() for q in range(P)]
        got = _all_to_all_blocks(blocks, self.group)
        return torch.cat([g.view(mr, mr).t() for g in got], dim=1).contiguous()

    def normal(self, x_rows: torch.Tensor, iters: int = 1) -> torch.Tensor:
        if self.apply_normal_1d is None:
            for _ in range(iters):
                x_rows = self.adjoint(self.forward(x_rows))
            return x_rows
        for _ in range(iters):  # X <- N1 X N1 (N1 symmetric)
            x_rows = self.transpose(self.apply_normal_1d(x_rows))
            x_rows = self.transpose(self.apply_normal_1d(x_rows))
        return x_rows


def gather_rows(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather row blocks into the full matrix (tests / result read-back)."""
    world = dist.get_world_size(group)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, dim=0)


def gather_cols(local: torch.Tensor, group=None) -> torch.Tensor:
    world = dist.get_world_size(group)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, dim=1)


def cuda_normal_1d(op) -> Callable[[torch.Tensor], torch.Tensor]:
    """The production local normal pass: returns N1 applied to every row (1D
    op); the caller's tensor is not modified (cww_normal works in place on a
    copy)."""
    def f(v: torch.Tensor) -> torch.Tensor:
        return op.normal(v.clone(memory_format=torch.contiguous_format), iters=1)
    return f


def cuda_apply_1d(op) -> Callable[[torch.Tensor, bool], torch.Tensor]:
    """The production local pass: a 1D ComposedOp on CUDA tensors (rows)."""
    def f(v: torch.Tensor, adjoint: bool) -> torch.Tensor:
        return op.adjoint(v) if adjoint else op.forward(v)
    return f
