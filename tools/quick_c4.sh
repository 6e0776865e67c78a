#!/bin/bash
# C4 quick check (run under gpurun): C4 parity tests + one 592-split bench line.
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -x -q -k "c4 or C4 or big" 2>&1 | tail -2
python bench.py --config C4 --splits 592 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; r=d['roofline']
print('step %.2f ms fit %.2f rank %.2f  %.2f TF frac %.3f' % (d['ms_per_step'], k['k_fit_big']['ms']/d['steps'], k['k_rank_big']['ms']/d['steps'], r['achieved'], r['frac']))"
