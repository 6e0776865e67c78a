#!/bin/bash
# Build kernel A/B variants into build/ (git-ignored) and time each on the
# bench workload under gpurun:   ./tools/ab_variants.sh build ; ./tools/ab_variants.sh run
cd "$(dirname "$0")/.."
NVCC="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC"
declare -A V=( [base]="" [noinline]="-DSPEEDREC_NOINLINE_FAST=1" [chol_rl]="-DSPEEDREC_CHOL_RL=1" )
if [ "$1" = "build" ]; then
  mkdir -p build
  for k in "${!V[@]}"; do $NVCC ${V[$k]} -o build/libspeedrec_$k.so paper_1910_07776_b200/csrc/speedrec.cu || exit 1; done
  exit 0
fi
for k in "${!V[@]}"; do
  for w in 12 16; do
    ms=$(SPEEDREC_LIB=$PWD/build/libspeedrec_$k.so SPEEDREC_WMAX=$w python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f %.1f' % (d['roofline']['kernel_ms'], d['ms_per_step']))")
    echo "variant=$k wmax=$w kernel_ms/step_ms=$ms"
  done
done
