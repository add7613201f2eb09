"""Per-phase cycle breakdown of k_normal_rows (debug build with
-DCWW_PHASE_TIMING -DCWW_PHASE_NU=<nu>); config 5 by default."""
import ctypes as C
import os
import sys

os.environ["CWW_LIB_NAME"] = "libcww_b200_phase.so"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2106_00554_b200 as cw  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
fam, nu, bnd, j, q, dim, r0, batch, kind, dens, name = bench.CONFIGS[cfg]
spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
op = cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, r0)
x = torch.randn(op.cols(), dtype=torch.float64, device="cuda")
w = torch.empty(op.rows(), dtype=torch.float64, device="cuda")
for _ in range(2):
    op.normal(x, iters=1, work=w)
torch.cuda.synchronize()
L = cw._load()
L.cww_debug_phase_read.argtypes = [C.c_void_p, C.c_size_t]
buf = np.zeros(1 << 20, dtype=np.int64)
assert L.cww_debug_phase_read(buf.ctypes.data, buf.size) == 0
ph = buf.reshape(-1, 16)[:, :6]
ph = ph[ph[:, 5] > 0]
d = np.diff(ph, axis=1)
names = ["load", "synthesis", "band", "analysis", "coarse out"]
tot = (ph[:, 5] - ph[:, 0]).mean()
print(f"cfg{cfg}: {len(ph)} CTAs (last launch), mean CTA cycles {tot:.0f}")
for n_, c in zip(names, d.mean(axis=0)):
    print(f"  {n_:12s} {c:9.0f} cyc  {100*c/tot:5.1f}%")
