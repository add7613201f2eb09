"""GPU tests of the least-squares driver (the reference
spec's gs_solve): CGLS on the normal equations through the
CUDA operator, checked against the spec's examples and against a dense
least-squares solve built from the CPU oracle (test infrastructure)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _cw():
    import paper_2106_00554_b200 as cw
    return cw


@pytest.mark.parametrize("case", [(0, 4, 1, 8, 1, 1, 4), (0, 3, 1, 14, 2, 1, 4), (0, 2, 0, 9, 1, 1, -1),
                                  (0, 4, 1, 5, 1, 2, 4), (1, 3, 1, 6, 2, 2, -1)])
def test_consistent_system_recovers_x(orc, cuda, case):
    """Spec example: y = forward(x) for random x -> x~ = x to 1e-8."""
    import torch
    cw = _cw()
    fam, nu, bnd, j, q, dim, r0 = case
    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    A = cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, None if r0 < 0 else r0)
    xt = torch.as_tensor(np.stack([orc.normals(40 + b, A.cols()) for b in range(3)]), device="cuda")
    y = A.forward(xt)
    x, iters, res = cw.gs_solve(A, y, residual_tol=1e-13, max_iters=500)
    assert iters > 0 and np.all(res <= 1e-13)
    for b in range(3):
        assert rel(x[b].cpu().numpy(), xt[b].cpu().numpy()) <= 1e-8


def test_matches_dense_least_squares(orc, cuda):
    """Inconsistent data: the GPU CG solution equals the dense LS solution of
    the oracle's matrix (columns = oracle forward of unit vectors)."""
    import torch
    cw = _cw()
    fam, nu, bnd, j, q, r0 = 0, 3, 1, 6, 1, 4
    ref = orc.op(fam, nu, bnd, j, q, 1, r0)
    Ad = np.stack([ref.forward(e) for e in np.eye(ref.nin)], axis=1)
    y = orc.normals(77, ref.nout)
    x_ls = np.linalg.lstsq(Ad, y, rcond=None)[0]
    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    A = cw.ComposedOp(cw.FastOp(spec, j, q, 1), None, True, r0)
    x, iters, res = cw.gs_solve(A, torch.as_tensor(y, device="cuda"), residual_tol=1e-14, max_iters=400)
    assert rel(x.cpu().numpy(), x_ls) <= 1e-10


def test_warm_start_and_non_convergence(orc, cuda):
    import torch
    cw = _cw()
    spec = cw.WaveletSpec(cw.Family.Daubechies, 4, cw.Boundary.Vmp)
    A = cw.ComposedOp(cw.FastOp(spec, 7, 1, 1), None, True, 4)
    xt = torch.as_tensor(orc.normals(5, A.cols()), device="cuda")
    y = A.forward(xt)
    with pytest.raises(cw.CwwError, match="did not converge"):
        cw.gs_solve(A, y, residual_tol=1e-15, max_iters=1)
    x1, it1, res1 = cw.gs_solve(A, y, residual_tol=1e-15, max_iters=1, raise_on_fail=False)
    assert it1 == 1 and res1[0] > 1e-15
    x2, it2, _ = cw.gs_solve(A, y, residual_tol=1e-12, max_iters=500, x0=xt)  # exact start
    assert it2 == 0 and rel(x2.cpu().numpy(), xt.cpu().numpy()) == 0.0


def test_masked_operator_least_squares(orc, cuda):
    """CG on a subsampled op (more samples than unknowns): minimiser of
    ||P A x - P y|| equals the dense masked LS solution."""
    import torch
    cw = _cw()
    fam, nu, bnd, j, q = 0, 2, 1, 5, 2
    ref = orc.op(fam, nu, bnd, j, q, 1, -1)
    rng = np.random.default_rng(3)
    mask = np.sort(rng.choice(ref.nout, 3 * ref.nin, replace=False)).astype(np.uint64)
    Ad = np.stack([ref.forward_masked(mask, e) for e in np.eye(ref.nin)], axis=1)
    y = orc.normals(91, mask.size)
    x_ls = np.linalg.lstsq(Ad, y, rcond=None)[0]
    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    A = cw.ComposedOp(cw.FastOp(spec, j, q, 1), cw.SamplingMask(mask), True)
    x, _, _ = cw.gs_solve(A, torch.as_tensor(y, device="cuda"), residual_tol=1e-14, max_iters=400)
    assert rel(x.cpu().numpy(), x_ls) <= 1e-10
