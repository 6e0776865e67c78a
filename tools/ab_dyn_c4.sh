#!/bin/bash
# A/B: dynamic fit queue of k_fit_big (SPEEDREC_DYN_UNITS=1, default) vs the static stride (0), C4 592 splits.
cd "$(dirname "$0")/.."
for q in 0 1 0 1; do
  SPEEDREC_DYN_UNITS=$q python bench.py --config C4 --splits 592 --steps 5 --warmup 3 --no-e2e --no-extra --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('dyn=$q C4', round(d['ms_per_step'],3), 'ms/step', '%.4g' % d['value'], {n: round(v['ms']/d['steps'],3) for n, v in k.items() if v['ms'] > 0.05}, 'frac', round(d['roofline']['frac'],4))"
done
