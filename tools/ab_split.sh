#!/bin/bash
# A/B: split LS path (k_fit_warp MODE 4 + k_pred_rank) vs the EX-table path on C3.
cd "$(dirname "$0")/.."
B="--steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline"
for v in 1 0; do
  SPEEDREC_SPLIT_LS=$v python bench.py $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']; print('split_ls=$v', round(d['ms_per_step'],2), 'ms/step', {n: (v['launches'], round(v['ms'],2)) for n,v in k.items() if v['launches']}, 'acc', d['accuracy']['pooled_sign_accuracy_pct'], d['accuracy']['recommendations'])"
done
