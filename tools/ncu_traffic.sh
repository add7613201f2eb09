#!/bin/bash
# DRAM bytes per launch of each config's dominant kernel (bench.py roofline.traffic)
set -e
cat > /tmp/dom.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch, bench, paper_2106_00554_b200 as cw
c = int(sys.argv[1])
fam, nu, bnd, j, q, dim, r0, batch, kind, dens, name = bench.CONFIGS[c]
spec = cw.WaveletSpec(cw.Family(fam), nu, cw.Boundary(bnd))
op = cw.HaarFullRankOp(j, q, r0) if nu == 1 else cw.ComposedOp(cw.FastOp(spec, j, q, dim), None, True, r0)
x = torch.randn((batch, op.cols()), dtype=torch.float64, device="cuda")
y = torch.randn((batch, op.rows()), dtype=torch.float64, device="cuda")
for _ in range(2):
    if c == 5:
        op.normal(x[:1].contiguous(), iters=1, work=torch.empty(op.rows(), dtype=torch.float64, device="cuda"))
    else:
        op.forward(x); op.adjoint(y)
torch.cuda.synchronize()
PY
# spec = config:kernel[:launches per call] -- the second call's launches are captured
for spec in "1:k_wv_fwd" "1:k_wv_adj" "2:large_adj2" "2:k_dwt_wpyr:2" "3:large_adj2" "3:large_fwd2" "3:large_adj1" "3:large_fwd1_fz" "4:k_wv_adj:2" "4:k_wv_fwd:2" "5:normal_rows"; do
  c=$(echo $spec | cut -d: -f1); k=$(echo $spec | cut -d: -f2); n=$(echo $spec | cut -d: -f3); n=${n:-1}
  python /tmp/dom.py $c
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      -k regex:"$k" -s $n -c $n python /tmp/dom.py $c 2>/dev/null | grep -E "dram__|gpu__" | sed "s/^/cfg$c,/"
done
