cd /root/repo
for v in 0 1 0 1; do
SPEEDREC_L2_PERSIST=$v python bench.py --config C4 --splits 592 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; r=d['roofline']
print('persist=$v step %.2f ms fit %.2f rank %.2f %.2f TF' % (d['ms_per_step'], k['k_fit_big']['ms']/d['steps'], k['k_rank_big']['ms']/d['steps'], r['achieved']))"
done
SPEEDREC_L2_PERSIST=1 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_fit_big -c 1 python bench.py --config C4 --splits 592 --steps 1 --warmup 0 --no-e2e --no-extra --no-cpu-baseline 2>&1 | grep -E "dram__bytes|duration"
