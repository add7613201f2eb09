"""Per-phase cycle breakdown of k_small_fwd / k_small_adj for config 1 (Haar;
debug build with -DCWW_PHASE_TIMING -DCWW_PHASE_NU=1)."""
import ctypes as C
import os
import sys

os.environ["CWW_LIB_NAME"] = "libcww_b200_phase1.so"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2106_00554_b200 as cw  # noqa: E402

op = cw.HaarFullRankOp(10, 1, 1)
x = torch.randn((1, op.cols()), dtype=torch.float64, device="cuda")
y = torch.randn((1, op.rows()), dtype=torch.float64, device="cuda")
L = cw._load()
L.cww_debug_phase_read.argtypes = [C.c_void_p, C.c_size_t]
for name, fn, arg, names in (("fwd", op.forward, x, ["load", "idwt levels", "final level", "halo+ES+sync", "-", "H_A", "row stage"]),
                             ("adj", op.adjoint, y, ["row stage", "H_A", "W + overlap-add", "DWT levels", "store"])):
    for _ in range(5):
        fn(arg)
    torch.cuda.synchronize()
    buf = np.zeros(1 << 20, dtype=np.int64)
    assert L.cww_debug_phase_read(buf.ctypes.data, buf.size) == 0
    ph = buf.reshape(-1, 16)[:1, :len(names) + 1]
    d = np.diff(ph, axis=1)[0]
    tot = ph[0, -1] - ph[0, 0]
    print(f"cfg1 {name}: CTA cycles {tot}")
    for n_, c in zip(names, d):
        print(f"  {n_:16s} {c:7d} cyc  {100 * c / tot:5.1f}%")
