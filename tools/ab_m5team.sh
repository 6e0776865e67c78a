#!/bin/bash
# A/B: M5P team size (SPEEDREC_M5_TEAM) on C2 (all 240 Table-2 scenarios) and C3 65536 splits.
cd "$(dirname "$0")/.."
for t in ${TS:-1 2 4}; do
  for cfg in "--config C2" "--config C3 --splits 65536"; do
    SPEEDREC_M5_TEAM=$t python bench.py $cfg --learner m5 --steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('team=$t', '$cfg', round(d['ms_per_step'],3), 'ms/step', round(d['value'],1))"
  done
done
