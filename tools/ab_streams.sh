#!/bin/bash
# A/B: fork-join launch groups of the prefix-shared mask path (SPEEDREC_GROUP_STREAMS=1 sequential,
# 2..4 side streams) on C5 (all 2^20 masks x 128 folds).  Run under gpurun.
cd "$(dirname "$0")/.."
for k in ${KS:-4 6 8 4 6 8}; do
  SPEEDREC_GROUP_STREAMS=$k python bench.py --config C5 --masks-k 20 --steps 10 --warmup 3 --no-e2e --no-extra --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('streams=$k', round(d['ms_per_step'],3), 'ms/step', '%.4g' % d['value'], {n: round(v['ms']/d['steps'],3) for n, v in k.items() if v['ms'] > 0}, 'frac', round(d['roofline']['frac'],4))"
done
