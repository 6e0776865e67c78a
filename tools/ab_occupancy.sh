#!/bin/bash
# A/B of k_fit_warp occupancy knobs on C3 (run under gpurun): warps per CTA
# (SPEEDREC_WMAX) x shared-memory factor cap (SPEEDREC_MCAP).
cd "$(dirname "$0")/.."
B="--steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline"
for cfg in "16 32" "16 24" "20 24" "20 32" "24 24" "24 20"; do
  set -- $cfg
  SPEEDREC_WMAX=$1 SPEEDREC_MCAP=$2 python bench.py $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']; print('wmax=$1 mcap=$2', round(d['ms_per_step'],2), 'ms/step', {n: round(v['ms']/v['launches'],2) for n,v in k.items() if v['launches']})"
done
