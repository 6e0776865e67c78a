#!/bin/bash
# A/B: model-table chunk size (SPEEDREC_CHUNK_MB) on C3: L2-resident chunks vs 1 GB.
cd "$(dirname "$0")/.."
B="--steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline"
for mb in ${MBS:-48 96 192 1024}; do
  SPEEDREC_CHUNK_MB=$mb python bench.py $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']; print('chunk_mb=$mb', round(d['ms_per_step'],2), 'ms/step', {n: (v['launches']//5, round(v['ms']/5,2)) for n,v in k.items() if v['launches']})"
done
