#!/bin/bash
# One GPU call that regenerates the round's profile artefacts into gpurun_out/prof/:
# bench lines for configs 1-5 (the default command = config 3 with its CPU
# baseline), reference-arm lines, the default command's ncu launch list,
# per-config dominant-kernel DRAM traffic, an ncu --set full capture of the
# config-3 passes and pyramids, the config-4 warp kernels and the config-5
# normal rows, the GPU test suite and smoke().  (Summaries are
# copied into profiles/ afterwards.)
set -x
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 600 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for c in 1 2 4 5; do timeout 400 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
for c in 3 2; do timeout 600 python bench.py --impl reference --config $c > $O/reference_cfg$c.json 2> $O/reference_cfg$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_cfg3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 bash tools/ncu_traffic.sh > $O/ncu_traffic.csv 2> $O/ncu_traffic.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_large_fwd2|k_large_adj2" \
    --launch-skip 2 --launch-count 2 -o $O/cfg3_fwd2_adj2 python tools/profcase.py --config 3 --iters 2 > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_large_adj1|k_large_fwd1_fz|k_dwt_wpyr|k_idwt_wpyr" \
    --launch-skip 7 --launch-count 9 -o $O/cfg3_pass1_pyramids python tools/profcase.py --config 3 --iters 2 >> $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_wv_" \
    --launch-skip 4 --launch-count 4 -o $O/cfg4_warp_kernels python tools/profcase.py --config 4 --iters 2 >> $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_normal_rows" \
    --launch-skip 2 --launch-count 1 -o $O/cfg5_normal_rows python tools/profnormal.py >> $O/ncu_full.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
true
