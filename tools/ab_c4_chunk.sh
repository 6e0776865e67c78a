cd /root/repo
python -m pytest tests -m gpu -q -x -k "c4 or C4" 2>&1 | tail -1
for lib in libspeedrec.so libspeedrec_g32.so libspeedrec_g40.so libspeedrec.so; do
  SPEEDREC_LIB=$PWD/paper_1910_07776_b200/$lib python bench.py --config C4 --splits 592 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; r=d['roofline']
print('$lib step %.2f ms fit %.2f  %.2f TF frac %.3f' % (d['ms_per_step'], k['k_fit_big']['ms']/d['steps'], r['achieved'], r['frac']))"
done
