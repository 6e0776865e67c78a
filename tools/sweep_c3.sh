#!/bin/bash
# C3 launch-shape sweep (run under gpurun): warps per CTA x EX-table chunk size.
cd "$(dirname "$0")/.."
for w in ${WL:-12 16}; do for mb in ${MBL:-32 64 128 256}; do
  r=$(SPEEDREC_WMAX=$w SPEEDREC_CHUNK_MB=$mb python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('%.2f fit %.2f rank %.2f' % (d['ms_per_step'], k['k_fit_warp']['ms']/d['steps'], k.get('k_rank_warp', {'ms': 0})['ms']/d['steps']))")
  echo "wmax=$w chunk_mb=$mb step/fit/rank ms: $r"
done; done
