"""Edge cases of the CUDA operator (empty and ragged
inputs, maximum sizes, determinism, concurrency):

* batch 0 is a no-op through every entry point;
* the largest 1D size the ABI accepts (M = 2^23, N = 2^25: pass tiles of 512
  rows) satisfies the size-independent properties: adjoint
  identity <U x, y> = <x, U* y>, linearity, and a norm bound (U has
  orthonormal columns up to the quadrature, so ||U x|| <= ||x||(1 + eps));
* results are bitwise reproducible (fixed-order reductions everywhere: the
  adjoint's edge partial sums, the fused analysis's chunk-boundary partials);
* one op used from several host threads on their own streams gives the
  single-thread results (the reference's const forward / adjoint).
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cw():
    import paper_2106_00554_b200 as cw
    return cw


def _op(cw, nu, bnd, j, q, dim=1, r0=None):
    spec = cw.WaveletSpec(cw.Family.Daubechies, nu, cw.Boundary(bnd))
    return cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, r0)


@pytest.mark.parametrize("case", [(3, 1, 8, 2, 1), (3, 1, 16, 2, 1), (4, 1, 10, 1, 2)])
def test_empty_batch(cuda, case):
    import torch
    cw = _cw()
    nu, bnd, j, q, dim = case
    A = _op(cw, nu, bnd, j, q, dim)
    x = torch.empty((0, A.cols()), dtype=torch.float64, device="cuda")
    y = torch.empty((0, A.rows()), dtype=torch.float64, device="cuda")
    assert A.forward(x).shape == (0, A.rows())
    assert A.adjoint(y).shape == (0, A.cols())
    assert A.forward(np.empty((0, A.cols()))).shape == (0, A.rows())


def test_largest_1d_size_properties(cuda):
    import torch
    cw = _cw()
    A = _op(cw, 3, 1, 23, 2, 1, 4)  # M = 2^23, N = 2^25: 64 MB in, 256 MB out
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(A.cols(), dtype=torch.float64, device="cuda", generator=g)
    x2 = torch.randn(A.cols(), dtype=torch.float64, device="cuda", generator=g)
    y = torch.randn(A.rows(), dtype=torch.float64, device="cuda", generator=g)
    ux, aty = A.forward(x), A.adjoint(y)
    lhs, rhs = float(torch.dot(ux, y)), float(torch.dot(x, aty))
    assert abs(lhs - rhs) <= 1e-12 * float(ux.norm() * y.norm())
    lin = A.forward(2.5 * x - 0.75 * x2) - (2.5 * ux - 0.75 * A.forward(x2))
    assert float(lin.norm()) <= 1e-12 * float(ux.norm())
    assert float(ux.norm()) <= float(x.norm()) * (1 + 1e-6)
    del ux, aty, lin
    torch.cuda.empty_cache()


@pytest.mark.parametrize("case", [(3, 1, 21, 2, 1, 4, 3), (4, 1, 16, 2, 1, 4, 64), (4, 1, 10, 1, 2, 4, 3)])
def test_bitwise_reproducible(cuda, case):
    import torch
    cw = _cw()
    nu, bnd, j, q, dim, r0, B = case
    A = _op(cw, nu, bnd, j, q, dim, r0)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((B, A.cols()), dtype=torch.float64, device="cuda", generator=g)
    y = torch.randn((B, A.rows()), dtype=torch.float64, device="cuda", generator=g)
    f1, a1 = A.forward(x), A.adjoint(y)
    f2, a2 = A.forward(x), A.adjoint(y)
    assert torch.equal(f1, f2) and torch.equal(a1, a2)


def test_concurrent_host_threads(cuda):
    import torch
    cw = _cw()
    A = _op(cw, 3, 1, 14, 2, 1, 4)
    g = torch.Generator(device="cuda").manual_seed(11)
    xs = [torch.randn((4, A.cols()), dtype=torch.float64, device="cuda", generator=g) for _ in range(4)]
    want = [A.adjoint(A.forward(x)) for x in xs]
    torch.cuda.synchronize()
    got = [None] * len(xs)
    errs = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    got[i] = A.adjoint(A.forward(xs[i]))
            s.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(xs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for a, b in zip(got, want):
        assert torch.equal(a, b)


def test_concurrent_threads_different_sizes(cuda):
    """Several host threads driving operators of different sizes through the
    same kernels at once (different shared-memory footprints per launch): a
    per-launch cudaFuncSetAttribute raced here ("invalid argument")."""
    import torch
    cw = _cw()
    ops = [_op(cw, 3, 1, j, 2, 1, 4) for j in (13, 14, 15, 16)]
    g = torch.Generator(device="cuda").manual_seed(12)
    xs = [torch.randn((3, A.cols()), dtype=torch.float64, device="cuda", generator=g) for A in ops]
    want = [A.adjoint(A.forward(x)) for A, x in zip(ops, xs)]
    torch.cuda.synchronize()
    got = [None] * len(ops)
    errs = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(6):
                    got[i] = ops[i].adjoint(ops[i].forward(xs[i]))
            s.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    for _ in range(3):
        th = [threading.Thread(target=work, args=(i,)) for i in range(len(ops))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        for a, b in zip(got, want):
            assert torch.equal(a, b)


def test_too_large_is_rejected_cleanly(cuda):
    cw = _cw()
    with pytest.raises(cw.CwwError) as e:
        _op(cw, 3, 1, 24, 1, 1, 4)
    assert e.value.status == 7 and "j must be <= 23" in str(e.value)


def test_j22_j23_against_oracle(orc, cuda):
    """The 512-row pass tiles (j = 23) and the first size past config 3 (j = 22)
    against the C oracle (one vector each)."""
    import torch
    cw = _cw()
    for j in (22, 23):
        ref = orc.op(0, 3, 1, j, 1, 1, 4)
        A = _op(cw, 3, 1, j, 1, 1, 4)
        x = orc.normals(31 + j, ref.nin)
        y = orc.normals(41 + j, ref.nout)
        fx = A.forward(torch.as_tensor(x, device="cuda")).cpu().numpy()
        ay = A.adjoint(torch.as_tensor(y, device="cuda")).cpu().numpy()
        fr, ar = ref.forward(x), ref.adjoint(y)
        assert np.linalg.norm(fx - fr) / np.linalg.norm(fr) <= 1e-12
        assert np.linalg.norm(ay - ar) / np.linalg.norm(ar) <= 1e-12
