import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from oracle_py import Oracle
import paper_2106_00554_b200 as cw
o = Oracle()
for case in [(0,6,0,11,2,1,-1), (0,4,1,10,1,1,4)]:
    fam,nu,bnd,j,q,dim,r0 = case
    ref = o.op(*case)
    spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
    op = cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, None if r0 < 0 else r0)
    for B in (1, 2, 3, 4, 5):
        x = np.stack([o.normals(100 + b, ref.nin) for b in range(B)])
        fx = op.forward(torch.as_tensor(x, device="cuda")).cpu().numpy()
        errs = [np.linalg.norm(fx[b]-ref.forward(x[b], True))/np.linalg.norm(ref.forward(x[b], True)) for b in range(B)]
        print(case, B, ["%.1e" % e for e in errs])
