#!/bin/bash
# One gpurun call: a GPU test selection, then bench lines for the listed configs.
#   tools/gpu_check.sh "<pytest -k expr or ''>" "<configs>" [tag]
K="$1"; CFGS="$2"; TAG="${3:-chk}"
mkdir -p gpurun_out/$TAG
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > gpurun_out/$TAG/tests.log 2>&1
  echo "rc=$?" >> gpurun_out/$TAG/tests.log
fi
for c in $CFGS; do
  timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/$TAG/bench_cfg$c.json 2> gpurun_out/$TAG/bench_cfg$c.err
done
