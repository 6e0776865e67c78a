cd $GRAFT_REPO_ROOT
for case in c3 c4 sweep; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py $case > gpurun_out/r2w_sanitize_racecheck_${case}.txt 2>&1
  echo "racecheck $case rc=$? $(grep -E 'RACECHECK SUMMARY' gpurun_out/r2w_sanitize_racecheck_${case}.txt | tail -1)"
done
PYTHONPATH=. python tools/c4_refine_probe.py > gpurun_out/r2w_c4_refine.txt 2>&1
