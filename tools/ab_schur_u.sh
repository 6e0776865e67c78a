#!/bin/bash
# A/B harness of the (not kept) SPEEDREC_SCHUR_U knob, profiles/r4c_ab_schur_u.txt; the knob is gone,
# so today every U runs the default split.
B="--config C5 --masks-k 20 --steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline"
for u in 10 9 8; do
  SPEEDREC_SCHUR_U=$u python -m pytest tests/test_gpu_parity.py -k c5 -x -q 2>&1 | tail -1
  SPEEDREC_SCHUR_U=$u python bench.py $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']; print('U=$u', round(d['ms_per_step'],2), 'ms/step', {n: round(v['ms']/5,2) for n,v in k.items() if v['launches']}, d['accuracy']['pooled_sign_accuracy_pct'], d['accuracy']['recommendations'])"
done
