#!/bin/bash
# A/B of library variants built with extra nvcc flags (under gpurun): each
# variant is a separate .so selected with SPEEDREC_LIB; C3 bench ms/step.
cd "$(dirname "$0")/.."
B="--steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline"
for so in gpurun_out/ab_*.so paper_1910_07776_b200/ab_*.so; do
  [ -f "$so" ] || continue
  SPEEDREC_LIB=$so python bench.py $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']; print('$so', round(d['ms_per_step'],2), 'ms/step', {n: round(v['ms']/5,2) for n,v in k.items() if v['launches']})"
done
