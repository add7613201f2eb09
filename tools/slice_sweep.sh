#!/bin/bash
# Large-path slice pipeline sweep: CWW_LARGE_SLICE vectors per slice on CWW_LARGE_STREAMS side streams.
mkdir -p gpurun_out/sweep2
for cfg in "1 2" "1 3" "1 4" "2 2" "2 3" "4 2" "1 6" "32 1"; do
  set -- $cfg
  CWW_LARGE_SLICE=$1 CWW_LARGE_STREAMS=$2 timeout 300 python bench.py --config 3 --steps 10 --no-cpu-baseline > gpurun_out/sweep2/cfg3_s$1_k$2.json 2>&1
done
for cfg in "8 2" "8 4" "16 2" "4 4"; do
  set -- $cfg
  CWW_LARGE_SLICE=$1 CWW_LARGE_STREAMS=$2 timeout 300 python bench.py --config 2 --steps 10 --no-cpu-baseline > gpurun_out/sweep2/cfg2_s$1_k$2.json 2>&1
done
