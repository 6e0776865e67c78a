#!/bin/bash
# Round evidence (run under gpurun): default bench line, ncu --set full of the
# dominant kernel of C3 / C4 / C5, and the launch list of the default bench.
# Usage: tools/profile_round.sh TAG   -> gpurun_out/TAG_*
cd "$(dirname "$0")/.."
T=${1:-prof}
mkdir -p gpurun_out
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
B="--steps 1 --warmup 1 --no-e2e --no-extra --no-cpu-baseline"
ncu --set full --import-source on --clock-control none -k regex:k_fit_warp -c 1 -o gpurun_out/${T}_c3_fit python bench.py $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fit_big -c 1 -o gpurun_out/${T}_c4_fit python bench.py --config C4 --splits 592 $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_mask_sfit -s 5 -c 1 -o gpurun_out/${T}_c5_sfit python bench.py --config C5 --masks-k 20 $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c3_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-extra --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv python bench.py --config C5 --masks-k 20 --steps 2 --warmup 1 --no-e2e --no-extra --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c4_launches.csv python bench.py --config C4 --splits 592 --steps 2 --warmup 1 --no-e2e --no-extra --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | grep $T
