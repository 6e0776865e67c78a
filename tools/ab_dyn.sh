#!/bin/bash
# A/B: dynamic work units of k_fit_warp (SPEEDREC_DYN_UNITS=1, default) vs the static stride (0), C3 + C4 + C2.
cd "$(dirname "$0")/.."
for q in 0 1 0 1; do
  for cfg in "--config C3" "--config C2"; do
  SPEEDREC_DYN_UNITS=$q python bench.py $cfg --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('dyn=$q', '$cfg', round(d['ms_per_step'],3), 'ms/step', '%.4g' % d['value'], {n: round(v['ms']/d['steps'],3) for n, v in k.items() if v['ms'] > 0.05}, 'frac', round(d['roofline']['frac'],4))"
  done
done
