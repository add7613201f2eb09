"""A few U*U iterations of config 5 through cww_normal (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2106_00554_b200 as cw  # noqa: E402

fam, nu, bnd, j, q, dim, r0, batch, kind, dens, name = bench.CONFIGS[5]
op = cw.ComposedOp(cw.FastOp(cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd)), j, q, dim), None, True, r0)
x = torch.randn((1, op.cols()), dtype=torch.float64, device="cuda")
w = torch.empty((1, op.rows()), dtype=torch.float64, device="cuda")
op.normal(x, iters=2, work=w)
torch.cuda.synchronize()
print("ok")
