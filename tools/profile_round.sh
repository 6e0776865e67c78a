#!/bin/bash
# Round evidence (run under gpurun): default bench line, ncu --set full of the
# dominant kernels of C3 (fit + pred/rank) / C4 / C5 / C4-IBK, and the launch
# lists of the default bench.  Usage: tools/profile_round.sh TAG -> gpurun_out/TAG_*
cd "$(dirname "$0")/.."
T=${1:-prof}
mkdir -p gpurun_out
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
B="--steps 1 --warmup 1 --no-e2e --no-extra --no-cpu-baseline"
ncu --set full --import-source on --clock-control none -k regex:"k_fit_warp|k_pred_rank" -c 2 -o gpurun_out/${T}_c3 python bench.py $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fit_big -c 1 -o gpurun_out/${T}_c4_fit python bench.py --config C4 --splits 592 $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_mask_sfit<.int.5>" -c 1 -o gpurun_out/${T}_c5_sfit python bench.py --config C5 --masks-k 20 $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_ibk_dist -c 1 -o gpurun_out/${T}_ibk_dist python bench.py --config C4 --splits 16 --learner ibk $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_c3_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-extra --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv python bench.py --config C5 --masks-k 20 --steps 2 --warmup 1 --no-e2e --no-extra --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_c4_launches.csv python bench.py --config C4 --splits 592 --steps 2 --warmup 1 --no-e2e --no-extra --no-cpu-baseline > /dev/null 2>&1
# text summaries here; keep only the C3 report (gpurun brings back <= 64 MiB)
for r in c3 c4_fit c5_sfit ibk_dist; do
  python tools/ncu_summary.py gpurun_out/${T}_${r}.ncu-rep > gpurun_out/${T}_${r}_ncu.txt 2>&1
  ncu -i gpurun_out/${T}_${r}.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,local_load_requests > gpurun_out/${T}_${r}_raw.csv 2>&1
done
rm -f gpurun_out/${T}_c4_fit.ncu-rep gpurun_out/${T}_c5_sfit.ncu-rep gpurun_out/${T}_ibk_dist.ncu-rep
ls -la gpurun_out | grep $T
