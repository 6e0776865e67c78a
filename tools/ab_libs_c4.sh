#!/bin/bash
# A/B of library variants (SPEEDREC_LIB) on C4 (592 of 1e7 splits).
cd "$(dirname "$0")/.."
B="--config C4 --splits 592 --steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline"
for so in paper_1910_07776_b200/ab_*.so; do
  [ -f "$so" ] || continue
  SPEEDREC_LIB=$PWD/$so python bench.py $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']; print('$so', round(d['ms_per_step'],2), 'ms/step', {n: round(v['ms']/5,2) for n,v in k.items() if v['launches'] and v['ms']>0.5}, 'frac', round(d['roofline']['frac'],4))"
done
