#!/bin/bash
# A/B: warps per CTA of the split LS fit kernel (SPEEDREC_WMAX_LS) on C3.
cd "$(dirname "$0")/.."
B="--steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline"
for w in 16 20; do
  SPEEDREC_WMAX_LS=$w python bench.py $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']; print('wmax_ls=$w', round(d['ms_per_step'],2), 'ms/step', {n: round(v['ms']/5,2) for n,v in k.items() if v['launches']})"
done
