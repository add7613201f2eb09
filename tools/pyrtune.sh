#!/bin/bash
# quick timing of the large-path kernels for several pyramid parameters (env knobs)
for c in ${CONFIGS:-2 3}; do
  for sb in ${SBOT:-10}; do for wv in ${WLEV:-0}; do for wa in ${WANA:-3}; do
    CWW_PYR_SYN_BOT=$sb CWW_WPYR_LEVELS=$wv CWW_WPYR_ANA_LEVELS=$wa python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg$c sbot$sb wlev$wv wana$wa', d['ms_per_step'], d['path_frac'], {k: v[0] for k, v in d['kernels'].items()})"
  done; done; done
done
