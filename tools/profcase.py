"""Runs a few forward/adjoint calls of one benchmark config (for ncu / quick timing)."""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0)
    a = ap.parse_args()
    import torch
    import bench
    import paper_2106_00554_b200 as cw
    fam, nu, bnd, j, q, dim, r0, batch, kind, dens, name = bench.CONFIGS[a.config]
    batch = a.batch or batch
    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    op = cw.HaarFullRankOp(j, q, r0) if nu == 1 else cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, r0)
    x = torch.randn((batch, op.cols()), dtype=torch.float64, device="cuda")
    y = torch.randn((batch, op.rows()), dtype=torch.float64, device="cuda")
    fo = torch.empty_like(y)
    ao = torch.empty_like(x)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for _ in range(a.iters):
        ev[0].record()
        op.forward(x, fo)
        ev[1].record()
        op.adjoint(y, ao)
        ev[2].record()
    torch.cuda.synchronize()
    print(f"cfg{a.config}: fwd {ev[0].elapsed_time(ev[1]):.4f} ms  adj {ev[1].elapsed_time(ev[2]):.4f} ms")


if __name__ == "__main__":
    main()
