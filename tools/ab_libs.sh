#!/bin/bash
# Time the C3 bench step for library variants (run under gpurun): tools/ab_libs.sh lib1.so lib2.so ...
cd "$(dirname "$0")/.."
for lib in "$@"; do
  r=$(SPEEDREC_LIB=$PWD/paper_1910_07776_b200/$lib python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('%.2f fit %.2f' % (d['ms_per_step'], k['k_fit_warp']['ms']/d['steps']))")
  echo "$lib $r"
done
