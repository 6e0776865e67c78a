#!/bin/bash
# A/B: dynamic work units for M5P (teams draw from the launch-wide counter) vs the static stride.
cd "$(dirname "$0")/.."
for q in 0 1 0 1; do
  for cfg in "--config C2" "--config C1" "--config C3 --splits 65536"; do
  SPEEDREC_DYN_UNITS=$q python bench.py $cfg --learner m5 --steps 5 --warmup 3 --no-e2e --no-extra --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('dyn=$q', '$cfg', round(d['ms_per_step'],3), 'ms/step', '%.4g' % d['value'], {n: round(v['ms']/d['steps'],3) for n, v in k.items() if v['ms'] > 0.05})"
  done
done
