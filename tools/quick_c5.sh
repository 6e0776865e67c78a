#!/bin/bash
# C5 quick check (run under gpurun): mask-path parity tests + full-C5 bench lines for library variants.
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -x -q -k "c5 or C5 or mask" 2>&1 | tail -1
for lib in "$@"; do
  SPEEDREC_LIB=$PWD/paper_1910_07776_b200/$lib python bench.py --config C5 --masks-k 20 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$lib step %.2f ms  %.3g evals/s  ' % (d['ms_per_step'], d['value']) + ' '.join('%s %.2f' % (n, v['ms']/d['steps']) for n, v in k.items() if v['ms'] > 0.1), d['accuracy']['cases'], d['top_masks_head'][:3])"
done
