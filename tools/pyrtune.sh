#!/bin/bash
# quick timing of the large-path kernels for several pyramid parameters
for c in ${CONFIGS:-2 3}; do
  for sl in ${SYN:-12}; do for al in ${ANA:-11}; do for sb in ${SBOT:-0}; do
    CWW_PYR_SYN_BOT=$sb CWW_PYR_SYN_LOG=$sl CWW_PYR_ANA_LOG=$al python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg$c syn$sl ana$al sbot$sb', d['ms_per_step'], d['path_frac'], {k: v[0] for k, v in d['kernels'].items()})"
  done; done; done
done
