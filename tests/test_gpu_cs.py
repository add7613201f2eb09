"""GPU tests of the compressed-sensing driver (the
reference spec's cs_solve / QCBP): Chambolle-Pock on the CUDA
operator, checked against the spec's examples and the optimality conditions of
  min ||x||_1  s.t.  ||A x - y||^2 <= eta."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cw():
    import paper_2106_00554_b200 as cw
    return cw


def _op(cw, nu=2, j=6, q=1, mask=None):
    spec = cw.WaveletSpec(cw.Family.Daubechies, nu, cw.Boundary.Vmp)
    return cw.ComposedOp(cw.FastOp(spec, j, q, 1), None if mask is None else cw.SamplingMask(mask), True)


def test_huge_eta_gives_zero(orc, cuda):
    """Spec example: eta huge -> x = 0 (zero is feasible and l1-minimal)."""
    import torch
    cw = _cw()
    A = _op(cw)
    y = torch.as_tensor(orc.normals(3, A.rows()), device="cuda")
    x, iters, res = cw.cs_solve(A, y, eta=1e6)
    assert iters <= 20 and float(x.abs().max()) == 0.0
    assert abs(res[0] - float((y * y).sum())) <= 1e-12 * res[0]


@pytest.mark.parametrize("k", [0, 17, 40])
def test_one_sparse_recovery(orc, cuda, k):
    """Spec example: x 1-sparse, full mask, tiny eta -> exact recovery to 1e-6."""
    import torch
    cw = _cw()
    A = _op(cw)
    xt = torch.zeros(A.cols(), dtype=torch.float64, device="cuda")
    xt[k] = 1.0
    y = A.forward(xt)
    x, iters, res = cw.cs_solve(A, y, eta=1e-14, tol=1e-9, max_iters=50000)
    err = float((x - xt).norm() / xt.norm())
    assert err <= 1e-6, (err, iters)
    assert res[0] <= 1e-14 + 1e-9 * float((y * y).sum())


def test_optimality_conditions_masked(orc, cuda):
    """Subsampled (underdetermined) system with a sparse truth: the returned x is
    feasible, no larger in l1 than the truth, and satisfies the KKT conditions
    g = A*(y - A x) = c sign(x) on the support, |g| <= c off it."""
    import torch
    cw = _cw()
    j, q = 6, 1
    M, N = 1 << j, 1 << (j + q)
    rng = np.random.default_rng(11)
    mask = np.sort(rng.choice(N, 40, replace=False)).astype(np.uint64)
    A = _op(cw, 2, j, q, mask)
    xt = np.zeros(M)
    xt[rng.choice(M, 4, replace=False)] = rng.standard_normal(4)
    xt_d = torch.as_tensor(xt, device="cuda")
    y = A.forward(xt_d)
    eta = 1e-6 * float((y * y).sum())
    x, iters, res = cw.cs_solve(A, y, eta=eta, tol=1e-10, max_iters=200000)
    xs = x.cpu().numpy()
    assert res[0] <= eta * (1 + 1e-6) + 1e-10 * float((y * y).sum())
    assert np.abs(xs).sum() <= np.abs(xt).sum() * (1 + 1e-6)
    g = A.adjoint(y - A.forward(x)).cpu().numpy()
    sup = np.abs(xs) > 1e-6 * np.abs(xs).max()
    c = np.abs(g[sup]).mean()
    assert np.all(np.abs(g[sup] - c * np.sign(xs[sup])) <= 1e-4 * c)  # equal magnitude, matching signs
    assert np.all(np.abs(g[~sup]) <= c * (1 + 1e-2))                   # (Chambolle-Pock accuracy)


def test_infeasible_eta(orc, cuda):
    """Overdetermined masked system with inconsistent data: eta below the
    least-squares residual is reported as infeasible (status 10)."""
    import torch
    cw = _cw()
    j, q = 5, 2
    rng = np.random.default_rng(5)
    mask = np.sort(rng.choice(1 << (j + q), 3 << j, replace=False)).astype(np.uint64)
    A = _op(cw, 2, j, q, mask)
    y = torch.as_tensor(orc.normals(8, A.rows()), device="cuda")
    x_ls, _, _ = cw.gs_solve(A, y, residual_tol=1e-13, max_iters=1000)
    r_ls = float(((A.forward(x_ls) - y) ** 2).sum())
    with pytest.raises(cw.CwwError) as e:
        cw.cs_solve(A, y, eta=0.5 * r_ls, max_iters=200)
    assert e.value.status == 10


def test_batched_equals_single(orc, cuda):
    import torch
    cw = _cw()
    A = _op(cw, 3, 7, 1)
    xs = torch.as_tensor(np.stack([orc.normals(60 + b, A.cols()) for b in range(2)]), device="cuda")
    ys = A.forward(xs)  # consistent data: every eta >= 0 is feasible
    eta = 0.1 * float((ys[0] * ys[0]).sum())
    xb, _, _ = cw.cs_solve(A, ys, eta=eta, tol=1e-9, max_iters=4000, raise_on_fail=False)
    x0, _, _ = cw.cs_solve(A, ys[0].contiguous(), eta=eta, tol=1e-9, max_iters=4000, raise_on_fail=False)
    assert float((xb[0] - x0).abs().max()) <= 1e-6 * max(float(x0.abs().max()), 1e-30)
