"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU layer:
batch sharding (configs 2-4) and the row-partitioned 2D operator with
all-to-all transposes (config 5), checked against the CPU oracle's 2D op.
The local 1D passes use the oracle here (test infrastructure); on B200s they
are the CUDA ComposedOp (paper_2106_00554_b200.dist.cuda_apply_1d)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle_py import Oracle
        from paper_2106_00554_b200.dist import RowPartitioned2D, gather_cols, gather_rows, shard_batch
        o = Oracle()
        fam, nu, bnd, j, qq, r0 = case
        M, N = 1 << j, 1 << (j + qq)
        op1 = o.op(fam, nu, bnd, j, qq, 1, r0)

        def apply_1d(v, adjoint):
            a = v.numpy()
            out = np.stack([op1.adjoint(r) if adjoint else op1.forward(r) for r in a])
            return torch.from_numpy(out)

        # batch sharding covers every item exactly once
        seen = []
        for b in (1, 7, 64):
            s, c = shard_batch(b, rank, world)
            seen.append((b, s, c))
        def normal_1d(v):
            a = v.numpy()
            return torch.from_numpy(np.stack([op1.adjoint(op1.forward(r)) for r in a]))

        d2 = RowPartitioned2D(M, N, apply_1d)
        d2n = RowPartitioned2D(M, N, apply_1d, apply_normal_1d=normal_1d)
        x = torch.from_numpy(o.normals(77, M * M).reshape(M, M))
        xr = x[rank * M // world:(rank + 1) * M // world].contiguous()
        yc = d2.forward(xr)
        y = gather_cols(yc)
        xa = d2.adjoint(yc)
        xn = gather_rows(d2.normal(xr, 2))
        xnb = gather_rows(d2n.normal(xr, 3))  # odd count: transposes must cancel
        xt = gather_rows(d2.transpose(xr))
        xa_full = gather_rows(xa)
        if rank == 0:
            op2 = o.op(fam, nu, bnd, j, qq, 2, r0)
            ref_y = op2.forward(x.numpy().ravel()).reshape(N, N)
            ref_a = op2.adjoint(ref_y.ravel()).reshape(M, M)
            z = x.numpy().ravel()
            for _ in range(2):
                z = op2.adjoint(op2.forward(z))
            z3 = op2.adjoint(op2.forward(z))
            rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
            assert np.array_equal(xt.numpy(), x.numpy().T)
            q.put(("ok", seen, rel(y.numpy(), ref_y), rel(xa_full.numpy(), ref_a),
                   max(rel(xn.numpy().ravel(), z), rel(xnb.numpy().ravel(), z3))))
        else:
            q.put(("ok", seen, 0.0, 0.0, 0.0))
    except Exception as e:  # noqa: BLE001
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [(0, 2, 1, 4, 1, 3), (0, 4, 1, 5, 1, 4), (0, 3, 0, 4, 2, -1)])
def test_row_partitioned_2d_world2(case):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[0] == "ok", r
    counts = {}
    for r in res:
        for b, s, c in r[1]:
            counts.setdefault(b, []).append((s, c))
    for b, parts in counts.items():
        parts.sort()
        assert sum(c for _, c in parts) == b
        assert parts[0][0] == 0 and parts[1][0] == parts[0][1]
    fwd, adj, nrm = max(r[2] for r in res), max(r[3] for r in res), max(r[4] for r in res)
    assert fwd <= 1e-13 and adj <= 1e-13 and nrm <= 1e-13, (fwd, adj, nrm)


def test_shard_batch_uneven():
    from paper_2106_00554_b200.dist import shard_batch
    for world in (1, 2, 3, 8):
        for batch in (0, 1, 5, 32, 64):
            parts = [shard_batch(batch, r, world) for r in range(world)]
            assert sum(c for _, c in parts) == batch
            pos = 0
            for s, c in parts:
                assert s == pos
                pos += c


def _worker_cuda(rank, world, port, case, q):
    """Both ranks on cuda:0 (this box has one GPU): the local passes are the
    production CUDA ComposedOp (dist.cuda_apply_1d / dist.cuda_normal_1d); the
    gloo exchange carries host copies.  The ranks' kernels never wait on each
    other, so sharing one GPU is safe."""
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle_py import Oracle
        import paper_2106_00554_b200 as cw
        from paper_2106_00554_b200.dist import RowPartitioned2D, cuda_apply_1d, cuda_normal_1d, gather_cols, gather_rows
        o = Oracle()
        fam, nu, bnd, j, qq, r0 = case
        M, N = 1 << j, 1 << (j + qq)
        spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
        op1 = cw.ComposedOp(cw.FastOp(spec, j, qq, 1), None, True, None if r0 < 0 else r0)
        dev = torch.device("cuda:0")
        a1, n1 = cuda_apply_1d(op1), cuda_normal_1d(op1)

        def apply_1d(v, adjoint):
            return a1(v.to(dev), adjoint).cpu()

        def normal_1d(v):
            return n1(v.to(dev)).cpu()

        d2 = RowPartitioned2D(M, N, apply_1d)
        d2n = RowPartitioned2D(M, N, apply_1d, apply_normal_1d=normal_1d)
        x = torch.from_numpy(o.normals(78, M * M).reshape(M, M))
        xr = x[rank * M // world:(rank + 1) * M // world].contiguous()
        xr0 = xr.clone()
        y = gather_cols(d2.forward(xr))
        xa = gather_rows(d2.adjoint(d2.forward(xr)))
        xn = gather_rows(d2n.normal(xr, 3))
        assert torch.equal(xr, xr0)  # the caller's rows are not modified
        if rank == 0:
            op2 = o.op(fam, nu, bnd, j, qq, 2, r0)
            ref_y = op2.forward(x.numpy().ravel()).reshape(N, N)
            z = x.numpy().ravel()
            ref_a = op2.adjoint(ref_y.ravel())
            for _ in range(3):
                z = op2.adjoint(op2.forward(z))
            rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
            q.put(("ok", rel(y.numpy(), ref_y), rel(xa.numpy().ravel(), ref_a), rel(xn.numpy().ravel(), z)))
        else:
            q.put(("ok", 0.0, 0.0, 0.0))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put(("err", repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("case", [(0, 2, 1, 7, 1, 3), (0, 4, 1, 8, 1, 4)])
def test_row_partitioned_2d_world2_cuda(case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_cuda, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[0] == "ok", r
    fwd, adj, nrm = max(r[1] for r in res), max(r[2] for r in res), max(r[3] for r in res)
    assert fwd <= 1e-12 and adj <= 1e-12 and nrm <= 1e-12, (fwd, adj, nrm)
