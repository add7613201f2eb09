"""Repeats the concurrent-host-threads scenario and reports which results differ."""
import sys, threading, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_00554_b200 as cw

j = int(sys.argv[1]) if len(sys.argv) > 1 else 14
spec = cw.WaveletSpec(cw.Family.Daubechies, 3, cw.Boundary.Vmp)
A = cw.ComposedOp(cw.FastOp(spec, j, 2), None, True, 4)
g = torch.Generator(device="cuda").manual_seed(11)
xs = [torch.randn((4, A.cols()), dtype=torch.float64, device="cuda", generator=g) for _ in range(4)]
fw = [A.forward(x) for x in xs]
want = [A.adjoint(f) for f in fw]
torch.cuda.synchronize()
bad = 0
for rep in range(40):
    got = [None] * 4
    gotf = [None] * 4
    def work(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                gotf[i] = A.forward(xs[i])
                got[i] = A.adjoint(gotf[i])
        s.synchronize()
    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    [t.start() for t in th]; [t.join() for t in th]
    for i in range(4):
        ef = not torch.equal(gotf[i], fw[i]); ea = not torch.equal(got[i], want[i])
        if ef or ea:
            bad += 1
            df = (gotf[i] - fw[i]).abs(); da = (got[i] - want[i]).abs()
            print(f"rep {rep} thread {i}: fwd differs {ef} (n={int((df>0).sum())}, max {float(df.max()):.3e}, first idx {df.flatten().nonzero()[:3].flatten().tolist()}) adj differs {ea} (n={int((da>0).sum())}, max {float(da.max()):.3e}, idx {da.flatten().nonzero()[:3].flatten().tolist()})")
print("bad", bad)
