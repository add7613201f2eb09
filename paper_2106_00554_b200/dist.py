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


# ---------------------------------------------------------------------------
# Native multi-GPU entry points (C ABI, csrc/cww_dist.cpp; include/cww_b200.h)
# ---------------------------------------------------------------------------
def _native():
    import ctypes as C
    from . import _load
    L = _load()
    if not getattr(L, "_cww_dist_bound", False):
        vp, sz = C.c_void_p, C.c_size_t
        L.cww_nccl_unique_id.argtypes = [C.c_char_p, sz]
        L.cww_dist_create.argtypes = [vp, C.c_int, C.c_int, C.c_char_p, sz, C.POINTER(vp)]
        L.cww_dist_create_local.argtypes = [vp, C.c_int, C.POINTER(vp)]
        L.cww_dist_destroy.argtypes = [vp]
        L.cww_dist_normal.argtypes = [vp, vp, sz, C.c_int, vp]
        L.cww_dist_normal_local.argtypes = [vp, C.POINTER(vp), sz, C.c_int, vp]
        L.cww_multi_create.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(vp)]
        L.cww_multi_destroy.argtypes = [vp]
        for n in ("cww_multi_forward_host", "cww_multi_adjoint_host"):
            getattr(L, n).argtypes = [vp, vp, sz, vp, sz, sz]
        L._cww_dist_bound = True
    return L


def _desc(spec, j: int, q: int, dim: int, min_level: int, use_idwt: bool, device: int):
    from . import DATA_DIR, _Desc
    return _Desc(int(spec.family), spec.nu, int(spec.boundary), j, q, dim, min_level, 1 if use_idwt else 0, 0,
                 device, DATA_DIR.encode(), None, 0, None, 0)


def nccl_unique_id() -> bytes:
    """128-byte NCCL bootstrap id (rank 0; broadcast it to the other ranks)."""
    import ctypes as C
    from . import _check
    L = _native()
    buf = C.create_string_buffer(128)
    _check(L.cww_nccl_unique_id(buf, 128))
    return buf.raw


class NativeRowPartitioned2D:
    """Config 5 on P GPUs through the C ABI (cww_dist_*): this rank's M/P rows
    of a 2^j x 2^j coefficient image; `normal` applies (U*U)^iters with the
    banded normal form per axis and NCCL all-to-all transposes (grouped
    ncclSend / ncclRecv, pack = local transpose, unpack kernel).

    local=True: `nranks` virtual ranks in this process on one GPU with a
    device-copy exchange (the partition logic on a single GPU)."""

    def __init__(self, spec, j: int, q: int, min_level: int, rank: int = 0, nranks: int = 1,
                 nccl_id: Optional[bytes] = None, device: int = 0, use_idwt: bool = True, local: bool = False):
        import ctypes as C
        from . import _check
        L = _native()
        self.L, self.local, self.nranks, self.rank = L, local, nranks, rank
        self.M = 1 << j
        self.m = self.M // nranks
        d = _desc(spec, j, q, 2, min_level, use_idwt, device)
        h = C.c_void_p()
        if local:
            _check(L.cww_dist_create_local(C.byref(d), nranks, C.byref(h)))
        else:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("nccl_id (128 bytes from nccl_unique_id on rank 0) required")
            _check(L.cww_dist_create(C.byref(d), rank, nranks, nccl_id, 128, C.byref(h)))
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.L.cww_dist_destroy(h)
            self.h = None

    def normal(self, x_rows, iters: int = 1):
        """In place on this rank's rows (an (M/P, M) contiguous float64 CUDA
        tensor); local mode: a list of every virtual rank's rows."""
        import ctypes as C
        from . import _check
        if self.local:
            xs = list(x_rows)
            for x in xs:
                assert x.is_cuda and x.dtype == torch.float64 and x.is_contiguous() and x.numel() == self.m * self.M
            arr = (C.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
            _check(self.L.cww_dist_normal_local(self.h, arr, self.m * self.M, iters,
                                                torch.cuda.current_stream(xs[0].device).cuda_stream))
            return xs
        x = x_rows
        assert x.is_cuda and x.dtype == torch.float64 and x.is_contiguous() and x.numel() == self.m * self.M
        _check(self.L.cww_dist_normal(self.h, x.data_ptr(), x.numel(), iters,
                                      torch.cuda.current_stream(x.device).cuda_stream))
        return x


class MultiDeviceOp:
    """Batch sharding over the devices of one box in one process (cww_multi_*):
    host arrays in, host arrays out; the batch is split into contiguous shards
    (shard_batch), each run on its device from its own host thread."""

    def __init__(self, spec, j: int, q: int, dim: int, min_level: int, devices, use_idwt: bool = True):
        import ctypes as C
        from . import _check
        L = _native()
        self.L = L
        d = _desc(spec, j, q, dim, min_level, use_idwt, -1)
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(L.cww_multi_create(C.byref(d), len(devices), devs, C.byref(h)))
        self.h = h
        M, N = 1 << j, 1 << (j + q)
        self.nin, self.nout = (M, N) if dim == 1 else (M * M, N * N)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.L.cww_multi_destroy(h)
            self.h = None

    def _call(self, a, adjoint: bool):
        import numpy as np
        from . import _check
        a = np.ascontiguousarray(a, dtype=np.float64)
        ni, no = (self.nout, self.nin) if adjoint else (self.nin, self.nout)
        batch = a.size // ni
        o = np.empty(a.shape[:-1] + (no,), dtype=np.float64)
        fn = self.L.cww_multi_adjoint_host if adjoint else self.L.cww_multi_forward_host
        _check(fn(self.h, a.ctypes.data, a.size, o.ctypes.data, o.size, batch))
        return o

    def forward(self, x):
        return self._call(x, False)

    def adjoint(self, y):
        return self._call(y, True)
