"""Small invocations of every kernel family, for compute-sanitizer
(tests/test_gpu_sanitizer.py): small path (1D / 2D), large path (pyramids,
TMA-staged Hadamard passes), banded normal rows + transposes, the
distributed-transpose pack / unpack kernels, solver vector kernels."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch
    import paper_2106_00554_b200 as cw
    from paper_2106_00554_b200 import dist as cdist
    dev = torch.device("cuda:0")
    g = torch.Generator().manual_seed(1)
    for nu, bnd, j, q, dim, r0 in [(4, 1, 8, 2, 1, 4), (3, 0, 7, 1, 1, -1), (3, 1, 13, 2, 1, 4),
                                   (2, 1, 6, 1, 2, 3), (1, 0, 9, 1, 1, 1)]:
        spec = cw.WaveletSpec(cw.Family.Daubechies, nu, cw.Boundary(bnd))
        op = (cw.HaarFullRankOp(j, q, r0) if nu == 1 else
              cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, None if r0 < 0 else r0))
        x = torch.randn((2, op.cols()), dtype=torch.float64, generator=g).to(dev)
        y = torch.randn((2, op.rows()), dtype=torch.float64, generator=g).to(dev)
        op.forward(x)
        op.adjoint(y)
        if nu > 1 and j <= 12:
            op.normal(x.clone(), iters=1)
    spec = cw.WaveletSpec(cw.Family.Daubechies, 2, cw.Boundary.Vmp)
    d = cdist.NativeRowPartitioned2D(spec, 6, 1, 3, nranks=2, local=True)
    rows = [torch.randn((32, 64), dtype=torch.float64, generator=g).to(dev) for _ in range(2)]
    d.normal(rows, 1)
    A = cw.ComposedOp(cw.FastOp(spec, 6, 1, 1), None, True, 3)
    yv = A.forward(torch.randn(A.cols(), dtype=torch.float64, generator=g).to(dev))
    cw.gs_solve(A, yv, residual_tol=1e-10, max_iters=5, raise_on_fail=False)
    cw.cs_solve(A, yv, eta=1e-3, max_iters=40, raise_on_fail=False)
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
