#!/bin/bash
# One GPU call that regenerates the round's profile artefacts into gpurun_out/prof/:
# bench lines for configs 1-5, reference-arm lines, the default command's ncu
# launch list, per-config dominant-kernel DRAM traffic and an ncu --set full
# capture of the config-2 Hadamard passes.  (Copied into profiles/ afterwards.)
set -x
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/smi.txt
for c in 1 2 3 4 5; do timeout 400 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
for c in 2 3; do timeout 400 python bench.py --impl reference --config $c > $O/reference_cfg$c.json 2> $O/reference_cfg$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 1 > $O/ncu_launch.log 2>&1
timeout 600 bash tools/ncu_traffic.sh > $O/ncu_traffic.csv 2> $O/ncu_traffic.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_large_fwd2|k_large_adj2" \
    --launch-skip 2 --launch-count 2 -o $O/cfg2_fwd2_adj2 python tools/profcase.py --config 2 --iters 2 > $O/ncu_full.log 2>&1
true
