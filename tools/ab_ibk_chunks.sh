#!/bin/bash
# A/B: test-tile chunks per fit of k_ibk_dist (SPEEDREC_IBK_CHUNKS; default ~8 waves), C4 IBK 16 splits.
cd "$(dirname "$0")/.."
for ch in default 37 74 256 default 256; do
  if [ $ch = default ]; then unset SPEEDREC_IBK_CHUNKS; else export SPEEDREC_IBK_CHUNKS=$ch; fi
  python bench.py --config C4 --splits 16 --learner ibk --steps 3 --warmup 3 --no-e2e --no-extra --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('chunks=$ch C4-ibk', round(d['ms_per_step'],3), 'ms/step', {n: round(v['ms']/d['steps'],3) for n, v in k.items() if v['ms'] > 0.05}, 'frac', round(d['roofline']['frac'],4))"
done
