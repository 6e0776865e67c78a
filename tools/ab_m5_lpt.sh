#!/bin/bash
# A/B: M5P units largest-first on GROUPS splits (SPEEDREC_M5_LPT=1, default) vs batch order, C2 (Table-2) and BH6.
cd "$(dirname "$0")/.."
for q in 0 1 0 1; do
  for cfg in "--config C2" "--config BH6"; do
  SPEEDREC_M5_LPT=$q python bench.py $cfg --learner m5 --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('lpt=$q', '$cfg', round(d['ms_per_step'],3), 'ms/step', '%.4g' % d['value'], {n: round(v['ms']/d['steps'],3) for n, v in k.items() if v['ms'] > 0.05})"
  done
done
