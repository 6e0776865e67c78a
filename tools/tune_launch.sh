#!/bin/bash
# Launch-shape sweep of k_fit_warp on the bench workload (run under gpurun).
# Prints kernel ms per step for each (stage, wmax, smem cap) setting.
cd "$(dirname "$0")/.."
for cfg in "1 12 0" "1 16 0" "0 12 0" "0 16 0" "0 16 160" "0 12 120"; do
  set -- $cfg
  export SPEEDREC_STAGE=$1 SPEEDREC_WMAX=$2
  if [ "$3" != "0" ]; then export SPEEDREC_SMEM_KB=$3; else unset SPEEDREC_SMEM_KB; fi
  ms=$(python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f' % d['roofline']['kernel_ms'])")
  echo "stage=$1 wmax=$2 smem_kb=$3 kernel_ms=$ms"
done
