"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle on
the same seeded inputs.  Tolerance: relative L2 <= 1e-12 (fp64, BASELINE.json
north_star); index / permutation / sign tables bit-exact.  At the full
BASELINE sizes the size-independent properties (adjoint identity, linearity,
normal operator) are checked, plus one full-size vector against the oracle."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-12
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _cw():
    import paper_2106_00554_b200 as cw
    return cw


def make(fam, nu, bnd, j, q, dim=1, r0=-1, use_idwt=True):
    cw = _cw()
    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    if nu == 1:
        return cw.HaarFullRankOp(j, q, 0 if r0 < 0 else r0) if use_idwt else None
    op = cw.FastOp(spec, j, q, dim)
    if not use_idwt:
        return op
    return cw.ComposedOp(op, None, True, None if r0 < 0 else r0)


def gpu(x):
    import torch
    return torch.as_tensor(x, dtype=torch.float64, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


# (family, nu, boundary, j, q, dim, r0) -- small / edge-case coverage
SMALL = [
    (0, 2, 1, 2, 1, 1, -1), (0, 2, 1, 3, 1, 1, -1), (0, 2, 1, 3, 2, 1, -1), (0, 3, 1, 3, 1, 1, -1),
    (0, 4, 1, 3, 1, 1, -1), (0, 5, 1, 4, 1, 1, -1), (0, 6, 1, 4, 2, 1, -1), (0, 2, 1, 5, 1, 1, 3),
    (0, 4, 1, 6, 2, 1, 4), (0, 3, 1, 7, 2, 1, 4), (0, 6, 1, 8, 3, 1, -1), (1, 4, 1, 9, 1, 1, -1),
    (1, 5, 1, 10, 2, 1, 5), (0, 2, 0, 2, 1, 1, -1), (0, 3, 0, 5, 2, 1, -1), (0, 4, 0, 6, 1, 1, 3),
    (1, 6, 0, 7, 3, 1, -1), (0, 2, 0, 9, 1, 1, 0), (0, 4, 1, 10, 1, 1, 4), (0, 2, 1, 12, 1, 1, 3),
    (0, 3, 1, 13, 2, 1, 4), (0, 6, 0, 11, 2, 1, -1), (0, 1, 0, 1, 0, 1, 0), (0, 1, 0, 1, 1, 1, 0),
    (0, 1, 0, 5, 0, 1, 0), (0, 1, 0, 10, 1, 1, 1), (0, 1, 0, 8, 2, 1, 3), (0, 1, 0, 13, 1, 1, 2),
]


@pytest.mark.parametrize("case", SMALL, ids=lambda c: "f%d_nu%d_b%d_j%d_q%d_d%d_r%d" % c)
@pytest.mark.parametrize("use_idwt", [1, 0])
def test_parity_1d(orc, cuda, case, use_idwt):
    fam, nu, bnd, j, q, dim, r0 = case
    if nu == 1 and not use_idwt:
        pytest.skip("Haar op always composes the IDWT")
    ref = orc.op(fam, nu, bnd, j, q, dim, r0)
    op = make(fam, nu, bnd, j, q, dim, r0, bool(use_idwt))
    B = 3
    x = np.stack([orc.normals(100 + b, ref.nin) for b in range(B)])
    y = np.stack([orc.normals(200 + b, ref.nout) for b in range(B)])
    fx = host(op.forward(gpu(x)))
    ay = host(op.adjoint(gpu(y)))
    for b in range(B):
        assert rel(fx[b], ref.forward(x[b], use_idwt)) <= TOL, b
        assert rel(ay[b], ref.adjoint(y[b], use_idwt)) <= TOL, b


TWO_D = [(0, 2, 1, 3, 1, 2, -1), (0, 4, 1, 4, 1, 2, 4), (0, 2, 1, 6, 1, 2, 3), (0, 3, 0, 5, 2, 2, -1),
         (0, 4, 1, 7, 1, 2, 4), (1, 5, 1, 5, 1, 2, -1), (0, 6, 0, 6, 1, 2, -1),
         # j >= 8: column wavelet transforms run as a separate panel pass on the M columns
         (0, 4, 1, 8, 1, 2, 4), (0, 2, 0, 8, 2, 2, -1), (1, 3, 1, 9, 1, 2, 5), (0, 6, 1, 8, 1, 2, -1),
         (0, 2, 1, 10, 1, 2, 3)]


@pytest.mark.parametrize("case", TWO_D, ids=lambda c: "f%d_nu%d_b%d_j%d_q%d_d%d_r%d" % c)
@pytest.mark.parametrize("use_idwt", [1, 0])
def test_parity_2d(orc, cuda, case, use_idwt):
    fam, nu, bnd, j, q, dim, r0 = case
    ref = orc.op(*case)
    op = make(fam, nu, bnd, j, q, dim, r0, bool(use_idwt))
    x = np.stack([orc.normals(300 + b, ref.nin) for b in range(2)])
    y = np.stack([orc.normals(400 + b, ref.nout) for b in range(2)])
    fx, ay = host(op.forward(gpu(x))), host(op.adjoint(gpu(y)))
    for b in range(2):
        assert rel(fx[b], ref.forward(x[b], use_idwt)) <= TOL
        assert rel(ay[b], ref.adjoint(y[b], use_idwt)) <= TOL


# large-M path (two-pass Hadamard with the L2-resident intermediate)
LARGE = [(0, 4, 1, 14, 1, 1, 4), (0, 2, 1, 15, 2, 1, 3), (0, 4, 1, 16, 2, 1, 4), (0, 3, 0, 14, 1, 1, -1),
         (1, 6, 1, 15, 1, 1, -1), (0, 1, 0, 14, 1, 1, 1), (0, 5, 1, 17, 1, 1, -1),
         # edge sums in per-warp slots (2(2nu-1)2^q > 256); multi-launch analysis pyramids;
         # periodic cones down to level 0
         (0, 6, 1, 13, 4, 1, -1), (0, 4, 1, 18, 1, 1, 4), (0, 2, 0, 18, 1, 1, 0), (1, 3, 0, 20, 1, 1, -1),
         # Haar q = 0 (HaarFullRankOp), coarsest level near the top, r0 above the coarse split
         (0, 1, 0, 15, 0, 1, 0), (0, 4, 1, 13, 1, 1, 12), (0, 3, 1, 16, 2, 1, 11)]


@pytest.mark.parametrize("case", LARGE, ids=lambda c: "f%d_nu%d_b%d_j%d_q%d_d%d_r%d" % c)
@pytest.mark.parametrize("use_idwt", [1, 0])
def test_parity_large(orc, cuda, case, use_idwt):
    fam, nu, bnd, j, q, dim, r0 = case
    if nu == 1 and not use_idwt:
        pytest.skip("Haar op always composes the IDWT")
    ref = orc.op(*case)
    op = make(fam, nu, bnd, j, q, dim, r0, bool(use_idwt))
    x = np.stack([orc.normals(500 + b, ref.nin) for b in range(2)])
    y = np.stack([orc.normals(600 + b, ref.nout) for b in range(2)])
    fx, ay = host(op.forward(gpu(x))), host(op.adjoint(gpu(y)))
    for b in range(2):
        assert rel(fx[b], ref.forward(x[b], use_idwt)) <= TOL
        assert rel(ay[b], ref.adjoint(y[b], use_idwt)) <= TOL


# Batches whose xi exceeds 32 MB take the fused routes: the finest synthesis
# level inside forward pass 1, the finest analysis level inside adjoint pass 1
# (chunk-boundary partial sums + fixup).  (family, nu, boundary, j, q, r0, batch)
FUSED = [(0, 3, 1, 17, 2, 4, 40), (0, 2, 0, 17, 1, -1, 36), (0, 4, 1, 18, 1, 17, 20), (1, 5, 1, 19, 1, 6, 9),
         (0, 6, 0, 18, 1, 12, 17)]


@pytest.mark.parametrize("case", FUSED, ids=lambda c: "f%d_nu%d_b%d_j%d_q%d_r%d_B%d" % c)
@pytest.mark.parametrize("offset", [0, 1])
def test_parity_fused_levels(orc, cuda, case, offset):
    """Fused finest wavelet level (large batches), 16-byte aligned buffers and
    buffers one double off (element-wise staging instead of bulk copies)."""
    import torch
    fam, nu, bnd, j, q, r0, B = case
    ref = orc.op(fam, nu, bnd, j, q, 1, r0)
    op = make(fam, nu, bnd, j, q, 1, r0, True)
    x = np.stack([orc.normals(700 + b, ref.nin) for b in range(B)])
    y = np.stack([orc.normals(800 + b, ref.nout) for b in range(B)])
    xb = torch.empty(B * ref.nin + offset, dtype=torch.float64, device="cuda")
    yb = torch.empty(B * ref.nout + offset, dtype=torch.float64, device="cuda")
    xv, yv = xb[offset:].view(B, ref.nin), yb[offset:].view(B, ref.nout)
    xv.copy_(gpu(x))
    yv.copy_(gpu(y))
    fo = torch.empty(B * ref.nout + offset, dtype=torch.float64, device="cuda")[offset:].view(B, ref.nout)
    ao = torch.empty(B * ref.nin + offset, dtype=torch.float64, device="cuda")[offset:].view(B, ref.nin)
    op.forward(xv, fo)
    op.adjoint(yv, ao)
    fx, ay = host(fo), host(ao)
    for b in (0, 1, B // 2, B - 1):
        assert rel(fx[b], ref.forward(x[b], 1)) <= TOL
        assert rel(ay[b], ref.adjoint(y[b], 1)) <= TOL


# ---- subsampled ComposedOp (SamplingMask, fastop.cpp:231-281) --------------
MASKED = [(0, 4, 1, 8, 2, 1, -1, 0.1), (0, 3, 1, 14, 2, 1, 4, 0.3), (1, 2, 0, 9, 1, 1, -1, 0.5),
          (0, 4, 1, 5, 1, 2, -1, 0.2), (0, 2, 1, 6, 1, 2, 3, 0.05), (0, 1, 0, 10, 1, 1, 1, 0.4)]


@pytest.mark.parametrize("case", MASKED, ids=lambda c: "f%d_nu%d_b%d_j%d_q%d_d%d_r%d_%.2f" % c)
@pytest.mark.parametrize("use_idwt", [1, 0])
def test_parity_masked(orc, cuda, case, use_idwt):
    cw = _cw()
    fam, nu, bnd, j, q, dim, r0, frac = case
    if nu == 1 and not use_idwt:
        pytest.skip("Haar op always composes the IDWT")
    ref = orc.op(fam, nu, bnd, j, q, dim, r0)
    rng = np.random.default_rng(j * 31 + nu)
    mask = np.sort(rng.choice(ref.nout, max(1, int(frac * ref.nout)), replace=False)).astype(np.uint64)
    if nu == 1:
        op = cw.ComposedOp.__new__(cw.ComposedOp)  # HaarFullRankOp with a mask: via the handle
        op._h = cw._Handle(cw.WaveletSpec(cw.Family.Daubechies, 1, cw.Boundary.Periodic), j, q, 1, r0,
                           True, mask=mask)
    else:
        spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
        op = cw.ComposedOp(cw.FastOp(spec, j, q, dim), cw.SamplingMask(mask), bool(use_idwt),
                           None if r0 < 0 else r0)
    assert op.rows() == mask.size and op.cols() == ref.nin
    x = np.stack([orc.normals(700 + b, ref.nin) for b in range(2)])
    y = np.stack([orc.normals(800 + b, mask.size) for b in range(2)])
    fx, ay = host(op.forward(gpu(x))), host(op.adjoint(gpu(y)))
    fh = op.forward(x)  # host-pointer path
    for b in range(2):
        assert rel(fx[b], ref.forward_masked(mask, x[b], use_idwt)) <= TOL
        assert rel(ay[b], ref.adjoint_masked(mask, y[b], use_idwt)) <= TOL
        assert rel(fh[b], fx[b]) <= 1e-15
    # normal operator of the subsampled op: A* A = W U* P^T P U W^-1
    if use_idwt and nu > 1:
        xt = gpu(x[:1].copy())
        op.normal(xt, iters=1)
        want = ref.adjoint_masked(mask, ref.forward_masked(mask, x[0]))
        assert rel(host(xt)[0], want) <= TOL


def test_masked_errors(cuda):
    cw = _cw()
    spec = cw.WaveletSpec(cw.Family.Daubechies, 2, cw.Boundary.Vmp)
    op = cw.FastOp(spec, 6, 1)
    with pytest.raises(cw.CwwError, match="sorted and unique"):
        cw.ComposedOp(op, cw.SamplingMask([5, 3]))
    with pytest.raises(cw.CwwError, match="out of range"):
        cw.ComposedOp(op, cw.SamplingMask([1, 128]))
    full = cw.ComposedOp(op, cw.SamplingMask(np.arange(128)))  # full mask = identity
    assert full.rows() == 128


# ---- BASELINE.json configurations ------------------------------------------
CONFIGS = {  # (family, nu, boundary, j, q, dim, r0), (kind, density)
    1: ((0, 1, 0, 10, 1, 1, 1), (0, 1.0)),
    2: ((0, 4, 1, 16, 2, 1, 4), (1, 1.0)),
    3: ((0, 3, 1, 21, 2, 1, 4), (0, 0.1)),
    4: ((0, 4, 1, 10, 1, 2, 4), (1, 0.05)),
    5: ((0, 2, 1, 12, 1, 2, 3), (0, 0.02)),
}


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_config_against_oracle(orc, cuda, cfg):
    (fam, nu, bnd, j, q, dim, r0), (kind, dens) = CONFIGS[cfg]
    ref = orc.op(fam, nu, bnd, j, q, dim, r0)
    op = make(fam, nu, bnd, j, q, dim, r0)
    x = orc.synth(kind, 1000 * cfg, j, r0, dens, dim)
    y = orc.normals(1000 * cfg + 500, ref.nout)
    assert rel(host(op.forward(gpu(x))), ref.forward(x)) <= TOL
    assert rel(host(op.adjoint(gpu(y))), ref.adjoint(y)) <= TOL


def test_config3_one_vector_against_oracle(orc, cuda):
    (fam, nu, bnd, j, q, dim, r0), (kind, dens) = CONFIGS[3]
    ref = orc.op(fam, nu, bnd, j, q, dim, r0)
    op = make(fam, nu, bnd, j, q, dim, r0)
    x = orc.synth(kind, 3000, j, r0, dens)
    assert rel(host(op.forward(gpu(x))), ref.forward(x)) <= TOL
    y = orc.normals(3500, ref.nout)
    assert rel(host(op.adjoint(gpu(y))), ref.adjoint(y)) <= TOL


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_config_properties_full_size(cuda, cfg):
    """Adjoint identity <A x, y> = <x, A* y> and linearity at the full sizes."""
    import torch
    cw = _cw()
    (fam, nu, bnd, j, q, dim, r0), (kind, dens) = CONFIGS[cfg]
    op = make(fam, nu, bnd, j, q, dim, r0)
    B = 2 if cfg in (3, 5) else 4
    x = torch.stack([gpu(cw.synth(kind, 1000 * cfg + b, j, r0, dens, dim)) for b in range(B)])
    g = torch.Generator(device="cuda").manual_seed(cfg)
    y = torch.randn((B, op.rows()), generator=g, dtype=torch.float64, device="cuda")
    Ax, Aty = op.forward(x), op.adjoint(y)
    lhs = (Ax * y).sum(dim=1)
    rhs = (x * Aty).sum(dim=1)
    assert torch.all(torch.abs(lhs - rhs) <= 1e-12 * torch.linalg.norm(Ax, dim=1) * torch.linalg.norm(y, dim=1))
    A2 = op.forward(2.0 * x[:1] - 3.0 * x[1:2])
    assert rel(host(A2), host(2.0 * Ax[:1] - 3.0 * Ax[1:2])) <= 1e-13
    # near-isometry bound ||A x|| <= ||x|| (orthonormal Walsh system, orthogonal W)
    assert torch.all(torch.linalg.norm(Ax, dim=1) <= torch.linalg.norm(x, dim=1) * (1 + 1e-12))


def test_normal_operator_matches_two_calls(cuda):
    import torch
    cw = _cw()
    (fam, nu, bnd, j, q, dim, r0), _ = CONFIGS[5]
    op = make(fam, nu, bnd, 8, q, dim, r0)
    x = gpu(cw.synth(0, 5, 8, r0, 0.02, 2))
    ref = op.adjoint(op.forward(op.adjoint(op.forward(x))))
    out = op.normal(x.clone(), iters=2)
    assert rel(host(out), host(ref)) <= 1e-13
    assert torch.isfinite(out).all()


NORMAL = [(0, 2, 1, 7, 1, 1, 3), (0, 4, 1, 10, 2, 1, 4), (1, 6, 1, 9, 1, 1, -1), (0, 3, 0, 8, 2, 1, -1),
          (0, 1, 0, 8, 1, 1, 2), (0, 4, 1, 12, 1, 1, 4), (0, 2, 1, 6, 1, 2, 3), (0, 4, 1, 7, 1, 2, 4),
          (1, 5, 0, 7, 2, 2, -1), (0, 3, 1, 8, 1, 2, 4)]


@pytest.mark.parametrize("case", NORMAL, ids=lambda c: "f%d_nu%d_b%d_j%d_q%d_d%d_r%d" % c)
@pytest.mark.parametrize("use_idwt", [1, 0])
@pytest.mark.parametrize("iters", [1, 2, 3])
def test_normal_form_matches_forward_adjoint(orc, cuda, case, use_idwt, iters):
    """cww_normal uses the banded normal form (U* U = sum_s C_s^T H^T H C_s
    with H^T H = M I); it must equal repeated adjoint(forward(x)) and the
    oracle's to <= 1e-12 relative."""
    fam, nu, bnd, j, q, dim, r0 = case
    if nu == 1 and not use_idwt:
        pytest.skip("Haar op always composes the IDWT")
    op = make(fam, nu, bnd, j, q, dim, r0, bool(use_idwt))
    ref = orc.op(fam, nu, bnd, j, q, dim, r0)
    x = np.stack([orc.normals(300 + b, ref.nin) for b in range(2)])
    want = gpu(x)
    for _ in range(iters):
        want = op.adjoint(op.forward(want))
    got = op.normal(gpu(x), iters=iters)
    z = x[0]
    for _ in range(iters):
        z = ref.adjoint(ref.forward(z, use_idwt), use_idwt)
    for b in range(2):
        assert rel(host(got)[b], host(want)[b]) <= 1e-12
    assert rel(host(got)[0], z) <= 1e-12


@pytest.mark.parametrize("j,q,dim", [(10, 1, 1), (16, 2, 1), (6, 1, 2)])
def test_cuda_graph_capture(cuda, j, q, dim):
    """cww_forward / cww_adjoint are capturable into a CUDA graph (stream-ordered
    allocations, no host synchronisation): replay reproduces eager calls bitwise."""
    import torch
    cw = _cw()
    op = make(0, 4, 1, j, q, dim, 4)
    x = torch.randn((3, op.cols()), dtype=torch.float64, device="cuda")
    y = torch.randn((3, op.rows()), dtype=torch.float64, device="cuda")
    fo, ao = torch.empty_like(y), torch.empty_like(x)
    op.forward(x, fo)
    op.adjoint(y, ao)
    torch.cuda.synchronize()
    f_ref, a_ref = fo.clone(), ao.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        op.forward(x, fo)
        op.adjoint(y, ao)
    fo.zero_()
    ao.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(fo, f_ref) and torch.equal(ao, a_ref)
    x.mul_(2.0)  # replay reads the current input contents
    g.replay()
    torch.cuda.synchronize()
    assert rel(fo.cpu().numpy(), 2.0 * f_ref.cpu().numpy()) <= 1e-15


def test_host_pointer_path(orc, cuda):
    (fam, nu, bnd, j, q, dim, r0), (kind, dens) = CONFIGS[2]
    ref = orc.op(fam, nu, bnd, 12, q, dim, r0)
    op = make(fam, nu, bnd, 12, q, dim, r0)
    x = np.stack([orc.synth(kind, 7 + b, 12, r0, dens) for b in range(3)])
    fx = op.forward(x)  # numpy in -> the staged host path (cww_forward_host)
    assert isinstance(fx, np.ndarray)
    for b in range(3):
        assert rel(fx[b], ref.forward(x[b])) <= TOL
    y = orc.normals(9, ref.nout)
    assert rel(op.adjoint(y), ref.adjoint(y)) <= TOL


# ---- primitives: integer tables bit-exact, FWHT, DWT -------------------------
@pytest.mark.parametrize("bits", [1, 5, 13, 18, 23])
def test_sequency_perm_bit_exact(orc, cuda, bits):
    cw = _cw()
    got = host(cw.sequency_perm(bits)).astype(np.int64)
    n = np.arange(1 << bits, dtype=np.int64)
    g = n ^ (n >> 1)
    expect = np.zeros_like(g)
    for b in range(bits):
        expect |= ((g >> b) & 1) << (bits - 1 - b)
    assert np.array_equal(got, expect)
    for k in list(range(min(64, 1 << bits))) + [(1 << bits) - 1]:
        assert got[k] == orc.seq_to_nat(k, bits)


def test_walsh_sign_rows_bit_exact(orc, cuda):
    cw = _cw()
    for j in (3, 6, 11):
        ps = list(range(min(1 << j, 40))) + [(1 << j) - 1]
        got = host(cw.walsh_sign_rows(ps, j))
        for i, p in enumerate(ps):
            assert np.array_equal(got[i], orc.sign_row(p, j))


@pytest.mark.parametrize("bits", [3, 10, 13, 14, 16, 21, 23, 24])
def test_fwht(orc, cuda, bits):
    cw = _cw()
    v = np.stack([orc.normals(bits + b, 1 << bits) for b in range(2)])
    s = host(cw.fwht_sequency(gpu(v)))
    n = host(cw.fwht_natural(gpu(v)))
    for b in range(2):
        assert rel(s[b], orc.fwht_sequency(v[b])) <= 1e-14
        assert rel(n[b], orc.fwht_natural(v[b])) <= 1e-14
    ones = host(cw.fwht_sequency(gpu(np.ones(8))))
    assert ones[0] == 8.0 and np.all(ones[1:] == 0.0)


@pytest.mark.parametrize("nu,bnd,j,r0,dim", [(2, 1, 7, 3, 1), (4, 1, 9, 4, 1), (3, 0, 8, -1, 1),
                                             (1, 0, 10, 0, 1), (6, 1, 8, -1, 1), (2, 1, 5, 3, 2),
                                             (4, 1, 6, 4, 2),
                                             # the large-M route (warp pyramids): any j, as dwt_apply
                                             (3, 1, 16, 4, 1), (2, 1, 21, 3, 1), (4, 0, 17, -1, 1),
                                             (1, 0, 14, 0, 1), (5, 1, 13, 11, 1), (2, 1, 13, 3, 2)])
def test_dwt(orc, cuda, nu, bnd, j, r0, dim):
    cw = _cw()
    spec = cw.WaveletSpec(cw.Family.Daubechies, nu, cw.Boundary(bnd))
    n = (1 << j) if dim == 1 else (1 << (2 * j))
    x = orc.normals(77 + nu, n)
    f = host(cw.dwt_apply(spec, j, gpu(x), False, r0, dim))
    i = host(cw.dwt_apply(spec, j, gpu(x), True, r0, dim))
    assert rel(f, orc.dwt(0, nu, bnd, j, x, 0, r0, dim)) <= 1e-14
    assert rel(i, orc.dwt(0, nu, bnd, j, x, 1, r0, dim)) <= 1e-14


def test_kernel_table_matches_oracle(orc, cuda):
    cw = _cw()
    for fam in (0, 1):
        for nu in (2, 3, 4, 5, 6):
            for bnd in (0, 1):
                op = cw.FastOp(cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd)), nu + 3, 2)
                got = op.kernel_table()
                want = orc.kernel_table(fam, nu, bnd, 2)
                for g_, w_ in zip(got, want):
                    assert np.max(np.abs(g_ - w_)) <= 1e-15
                assert [t[:2] for t in op.edge_terms()] == [t[:2] for t in orc.op(fam, nu, bnd, nu + 3, 2).edge_terms()]


def test_dimension_mismatch_raises(cuda):
    cw = _cw()
    op = make(0, 2, 1, 5, 1)
    with pytest.raises(cw.CwwError):
        op.forward(gpu(np.zeros(33)))


# ---- kernel-table cache on op creation (get_kernel_table, kernel.cpp:173-198) ----
def test_op_uses_kernel_cache(orc, cuda, tmp_path):
    import struct
    import zlib
    cw = _cw()
    spec = cw.WaveletSpec(cw.Family.Daubechies, 4, cw.Boundary.Vmp)
    path = tmp_path / cw.kernel_cache_filename(spec, 2)
    op = cw.FastOp(spec, 6, 2, cache_dir=str(tmp_path))  # miss: computed and written back
    assert path.exists()
    gold = os.path.join(os.path.dirname(__file__), "golden", "cwwk_db4_vmp_q2_R14_v1.bin")
    assert path.read_bytes() == open(gold, "rb").read()
    it0 = op.kernel_table()[0]
    # a valid file with different values is loaded instead of recomputing
    body = bytearray(path.read_bytes()[:-4])
    v = struct.unpack_from("<d", body, 32)[0]
    struct.pack_into("<d", body, 32, v + 1.0)
    path.write_bytes(bytes(body) + struct.pack("<I", zlib.crc32(bytes(body)) & 0xFFFFFFFF))
    it1 = cw.FastOp(spec, 6, 2, cache_dir=str(tmp_path)).kernel_table()[0]
    assert it1.ravel()[0] == it0.ravel()[0] + 1.0
    # stale header (R != 14): recomputed and rewritten
    struct.pack_into("<I", body, 24, 12)
    path.write_bytes(bytes(body) + struct.pack("<I", zlib.crc32(bytes(body)) & 0xFFFFFFFF))
    it2 = cw.FastOp(spec, 6, 2, cache_dir=str(tmp_path)).kernel_table()[0]
    assert np.array_equal(it2, it0)
    assert path.read_bytes() == open(gold, "rb").read()


@pytest.mark.parametrize("fam,nu,bnd,q", [(0, 2, 1, 1), (0, 4, 1, 2), (1, 3, 0, 3), (0, 6, 1, 2), (1, 5, 1, 1),
                                          (0, 3, 0, 2)])
def test_gpu_kernel_table_bit_identical(orc, cuda, fam, nu, bnd, q):
    """f4: the kernel-table cascade on the GPU (separately rounded products and
    sums in the host's order) gives the same bits as the host / reference."""
    cw = _cw()
    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    host_t = cw.FastOp(spec, 6, q).kernel_table()
    gpu_t = cw.FastOp(spec, 6, q, gpu_kernel_table=True).kernel_table()
    for a, b in zip(host_t, gpu_t):
        assert np.array_equal(a, b)
    it, le, ri = orc.kernel_table(fam, nu, bnd, q)
    assert np.array_equal(gpu_t[0], it)


def test_pinned_host_async_path(orc, cuda):
    """cww_*_host_async on pinned host tensors (chunk-pipelined copies) gives
    the same results as the device path, on two concurrent streams."""
    import torch
    cw = _cw()
    spec = cw.WaveletSpec(cw.Family.Daubechies, 4, cw.Boundary.Vmp)
    # (9, 37) / (14, 37): chunk-pipelined copies; the tiny ones (<= 256 KB) run
    # zero-copy on the pinned buffers, including 2D and the Haar op (config 1)
    cases = [(cw.ComposedOp(cw.FastOp(spec, j, 2), None, True, 4), B) for j, B in ((9, 37), (14, 37), (10, 1), (6, 5))]
    cases.append((cw.ComposedOp(cw.FastOp(spec, 5, 1, 2), None, True, 4), 2))
    cases.append((cw.HaarFullRankOp(10, 1, 1), 1))
    for op, B in cases:
        x = torch.randn((B, op.cols()), dtype=torch.float64).pin_memory()
        y = torch.randn((B, op.rows()), dtype=torch.float64).pin_memory()
        fo = torch.empty((B, op.rows()), dtype=torch.float64).pin_memory()
        ao = torch.empty((B, op.cols()), dtype=torch.float64).pin_memory()
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        with torch.cuda.stream(s1):
            op.forward(x, fo)
        with torch.cuda.stream(s2):
            op.adjoint(y, ao)
        torch.cuda.synchronize()
        fd = op.forward(x.cuda()).cpu()
        ad = op.adjoint(y.cuda()).cpu()
        assert torch.equal(fo, fd) and torch.equal(ao, ad)


# ---- warp-per-vector kernels (M = 2^10, batches >= 256: the 2D passes) ------
WV = [(0, 4, 1, 10, 1, 1, 4, 1), (0, 2, 0, 10, 2, 1, -1, 1), (1, 6, 1, 10, 1, 1, 9, 1), (0, 3, 1, 10, 3, 1, 5, 1),
      (0, 1, 0, 10, 1, 1, 1, 1), (0, 5, 0, 10, 1, 1, 4, 0), (0, 4, 1, 10, 2, 1, 4, 0)]


@pytest.mark.parametrize("case", WV, ids=lambda c: "f%d_nu%d_b%d_j%d_q%d_d%d_r%d_i%d" % c)
def test_parity_warp_kernels(orc, cuda, case):
    fam, nu, bnd, j, q, dim, r0, use_idwt = case
    ref = orc.op(fam, nu, bnd, j, q, dim, r0)
    op = make(fam, nu, bnd, j, q, dim, r0, bool(use_idwt))
    Bn = 300
    x = np.stack([orc.normals(1100 + b % 7, ref.nin) * (1 + b) for b in range(Bn)])
    y = np.stack([orc.normals(1200 + b % 7, ref.nout) * (1 + b) for b in range(Bn)])
    fx, ay = host(op.forward(gpu(x))), host(op.adjoint(gpu(y)))
    for b in (0, 1, 150, Bn - 1):
        assert rel(fx[b], ref.forward(x[b], use_idwt)) <= TOL
        assert rel(ay[b], ref.adjoint(y[b], use_idwt)) <= TOL


# ---- fp32 I/O mode (north_star: <= 1e-5 against the fp64 oracle) -----------
@pytest.mark.parametrize("case", [(0, 4, 1, 10, 1, 2, 4), (0, 3, 1, 16, 2, 1, 4), (0, 2, 0, 9, 1, 1, -1),
                                  (0, 4, 1, 8, 2, 1, 4)])
def test_fp32_mode(orc, cuda, case):
    import torch
    cw = _cw()
    fam, nu, bnd, j, q, dim, r0 = case
    ref = orc.op(*case)
    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    op = cw.ComposedOp(cw.FastOp(spec, j, q, dim, precision="fp32"), None, True, None if r0 < 0 else r0)
    x = np.stack([orc.normals(900 + b, ref.nin) for b in range(2)])
    y = np.stack([orc.normals(950 + b, ref.nout) for b in range(2)])
    fx = host(op.forward(torch.as_tensor(x, dtype=torch.float32, device="cuda")))
    ay = host(op.adjoint(torch.as_tensor(y, dtype=torch.float32, device="cuda")))
    assert fx.dtype == np.float32 and ay.dtype == np.float32
    for b in range(2):
        assert rel(fx[b], ref.forward(x[b].astype(np.float32).astype(np.float64))) <= 1e-5
        assert rel(ay[b], ref.adjoint(y[b].astype(np.float32).astype(np.float64))) <= 1e-5
    with pytest.raises(cw.CwwError):  # an fp32 op takes float32 buffers only
        op.forward(torch.as_tensor(x, device="cuda"))
