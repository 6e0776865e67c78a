#!/bin/bash
# C5 full step: per-kernel ms (k_mask_sfit launches summed).
cd "$(dirname "$0")/.."
B="--config C5 --masks-k 20 --steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline"
python bench.py $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']; print('C5', round(d['ms_per_step'],2), 'ms/step', {n: round(v['ms']/5,2) for n,v in k.items() if v['launches']}, d['roofline']['frac'], d['top_masks_head'])"
