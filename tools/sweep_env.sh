#!/bin/bash
# One gpurun call: bench lines of one config under a list of env settings.
#   tools/sweep_env.sh <config> <tag> "A=1 B=2" "A=3" ...
C="$1"; TAG="$2"; shift 2
mkdir -p gpurun_out/$TAG
i=0
for e in "$@"; do
  env $e timeout 300 python bench.py --config $C --steps 10 --no-cpu-baseline > gpurun_out/$TAG/$i.json 2> gpurun_out/$TAG/$i.err
  echo "$i: $e" >> gpurun_out/$TAG/index.txt
  i=$((i+1))
done
python tools/show.py gpurun_out/$TAG/*.json
