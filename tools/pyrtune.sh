#!/bin/bash
# quick timing of the large-path kernels under several env knobs: KNOB="name=v1,v2" tools/pyrtune.sh
for c in ${CONFIGS:-2 3}; do
  name=${KNOB%%=*}; vals=${KNOB#*=}
  for val in ${vals//,/ }; do
    env $name=$val python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg$c $name=$val', d['ms_per_step'], d['path_frac'], {k: v[0] for k, v in d['kernels'].items()})"
  done
done
