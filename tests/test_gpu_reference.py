"""GPU parity against the compiled, unmodified reference (oracle/_ref/libcwwref.so,
proj/src/{walsh,wavelet,kernel,fastop}.cpp built by oracle/Makefile) at the
bench's exact shapes and FULL batch sizes: every vector of BASELINE configs
1-4 (the batch-dependent grids, edge-sum slots and batch slices of the timed
kernels), and config 5's normal operator at its exact shape (db2, VMP, r0=3,
2D 4096^2, q=1) through the default register-resident row kernel.  Inputs are
the bench's (bench.make_inputs, test_rng seeds).  Tolerance: relative L2 <=
1e-12 per vector (fp64, north_star)."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-12
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def rel_rows(a, b):
    a = np.asarray(a).reshape(len(b), -1)
    b = np.asarray(b).reshape(len(b), -1)
    return max(float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)) for x, y in zip(a, b))


def _op(cfg):
    import bench
    import paper_2106_00554_b200 as cw
    fam, nu, bnd, j, q, dim, r0 = bench.CONFIGS[cfg][:7]
    if nu == 1:
        return cw.HaarFullRankOp(j, q, r0)
    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    return cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, r0)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_full_batch_against_reference(ref, orc, cuda, cfg):
    """Forward and adjoint of the whole bench batch vs the reference library
    (threaded over the batch by ref_bench, as the reference arm times it)."""
    import torch
    import bench
    fam, nu, bnd, j, q, dim, r0, batch = bench.CONFIGS[cfg][:8]
    xs, ys = bench.make_inputs(orc.synth, cfg, 0, batch)
    rop = ref.op(fam, nu, bnd, j, q, dim, r0)
    threads = os.cpu_count() or 1
    want_f = np.empty((batch, rop.nout))
    want_a = np.empty((batch, rop.nin))
    rop.bench(0, xs, want_f, batch, threads)
    rop.bench(1, ys, want_a, batch, threads)
    op = _op(cfg)
    got_f = op.forward(torch.as_tensor(xs, device=cuda)).cpu().numpy()
    got_a = op.adjoint(torch.as_tensor(ys, device=cuda)).cpu().numpy()
    ef, ea = rel_rows(got_f, want_f), rel_rows(got_a, want_a)
    assert ef <= TOL and ea <= TOL, (ef, ea)


@pytest.mark.parametrize("iters", [1, 2])
def test_config5_normal_against_reference(ref, orc, cuda, iters):
    """cww_normal at config 5's exact shape -- the k_normal_rows_reg<2,12,256>
    row kernel that the bench times -- vs the reference's forward_2d/adjoint_2d
    composed `iters` times."""
    import torch
    import bench
    fam, nu, bnd, j, q, dim, r0, batch = bench.CONFIGS[5][:8]
    xs, _ = bench.make_inputs(orc.synth, 5, 0, 1)
    rop = ref.op(fam, nu, bnd, j, q, dim, r0)
    want = np.empty((1, rop.nin))
    rop.bench(2, xs, want, 1, os.cpu_count() or 1, iters)
    op = _op(5)
    x = torch.as_tensor(xs, device=cuda)
    work = torch.empty((1, op.rows()), dtype=torch.float64, device=cuda)
    got = op.normal(x, iters=iters, work=work).cpu().numpy()
    assert rel_rows(got, want) <= TOL


def test_config5_forward_adjoint_against_reference(ref, orc, cuda):
    """Config 5's operator itself (forward U W^-1 and adjoint W U* of the
    4096^2 image, N = 8192^2) vs the reference."""
    import torch
    import bench
    fam, nu, bnd, j, q, dim, r0 = bench.CONFIGS[5][:7]
    xs, _ = bench.make_inputs(orc.synth, 5, 0, 1)
    y = orc.normals(5500, 1 << (2 * (j + q)))[None]
    rop = ref.op(fam, nu, bnd, j, q, dim, r0)
    threads = os.cpu_count() or 1
    want_f = np.empty((1, rop.nout))
    want_a = np.empty((1, rop.nin))
    rop.bench(0, xs, want_f, 1, threads)
    rop.bench(1, y, want_a, 1, threads)
    op = _op(5)
    got_f = op.forward(torch.as_tensor(xs, device=cuda)).cpu().numpy()
    got_a = op.adjoint(torch.as_tensor(y, device=cuda)).cpu().numpy()
    assert rel_rows(got_f, want_f) <= TOL
    assert rel_rows(got_a, want_a) <= TOL


def test_misaligned_buffers(orc, cuda):
    """Caller buffers that are only 8-byte aligned (x + 1 element) on the small
    path (16-byte block loads) and the large path, forward and adjoint."""
    import torch
    import paper_2106_00554_b200 as cw
    for (nu, j, q, r0) in [(4, 10, 2, 4), (2, 6, 1, 3), (3, 14, 2, 4)]:
        spec = cw.WaveletSpec(cw.Family.Daubechies, nu, cw.Boundary.Vmp)
        op = cw.ComposedOp(cw.FastOp(spec, j, q), None, True, r0)
        rop = orc.op(0, nu, 1, j, q, 1, r0)
        B = 3
        xs = np.stack([orc.synth(1, 40 + b, j, r0, 1.0) for b in range(B)])
        ys = np.stack([orc.normals(90 + b, rop.nout) for b in range(B)])
        xb = torch.zeros(B * op.cols() + 1, dtype=torch.float64, device=cuda)
        yb = torch.zeros(B * op.rows() + 1, dtype=torch.float64, device=cuda)
        xb[1:] = torch.as_tensor(xs.ravel(), device=cuda)
        yb[1:] = torch.as_tensor(ys.ravel(), device=cuda)
        fo = torch.empty(B * op.rows() + 1, dtype=torch.float64, device=cuda)
        ao = torch.empty(B * op.cols() + 1, dtype=torch.float64, device=cuda)
        op.forward(xb[1:].view(B, -1), fo[1:].view(B, -1))
        op.adjoint(yb[1:].view(B, -1), ao[1:].view(B, -1))
        torch.cuda.synchronize()
        want_f = np.stack([rop.forward(x) for x in xs])
        want_a = np.stack([rop.adjoint(y) for y in ys])
        assert rel_rows(fo[1:].cpu().numpy(), want_f) <= TOL
        assert rel_rows(ao[1:].cpu().numpy(), want_a) <= TOL


@pytest.mark.parametrize("nu,bnd,q,r0", [(2, 1, 1, 3), (3, 0, 1, -1)])
def test_2d_large_route_against_reference(ref, orc, cuda, nu, bnd, q, r0):
    """The separable 2D operator above 2^12 per axis (j = 13: rows through the
    large path, batched transposes between the passes) vs the reference's
    forward_2d / adjoint_2d (fastop.cpp:196-227)."""
    import torch
    import paper_2106_00554_b200 as cw
    j = 13
    spec = cw.WaveletSpec(cw.Family.Daubechies, nu, cw.Boundary(bnd))
    op = cw.ComposedOp(cw.FastOp(spec, j, q, 2), None, True, None if r0 < 0 else r0)
    rop = ref.op(0, nu, bnd, j, q, 2, r0)
    x = orc.synth(0, 1313, j, max(r0, 0), 0.05, 2)[None]
    y = orc.normals(1314, rop.nout)[None]
    threads = os.cpu_count() or 1
    want_f = np.empty((1, rop.nout))
    want_a = np.empty((1, rop.nin))
    rop.bench(0, x, want_f, 1, threads)
    rop.bench(1, y, want_a, 1, threads)
    got_f = op.forward(torch.as_tensor(x, device=cuda)).cpu().numpy()
    got_a = op.adjoint(torch.as_tensor(y, device=cuda)).cpu().numpy()
    assert rel_rows(got_f, want_f) <= TOL
    assert rel_rows(got_a, want_a) <= TOL
