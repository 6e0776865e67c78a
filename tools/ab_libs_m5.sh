#!/bin/bash
# A/B of library variants on the M5P configs (C2, C1, C3 65536 splits): tools/ab_libs_m5.sh lib1.so lib2.so ...
cd "$(dirname "$0")/.."
for rep in 1 2; do
for lib in "$@"; do
  for cfg in "--config C2" "--config C1" "--config C3 --splits 65536"; do
  SPEEDREC_LIB=$PWD/paper_1910_07776_b200/$lib python bench.py $cfg --learner m5 --steps 5 --warmup 3 --no-e2e --no-extra --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', '$cfg', round(d['ms_per_step'],3), 'ms/step')"
  done
done
done
