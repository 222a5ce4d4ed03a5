# compute-sanitizer over the small cases of tools/sanitize_cases.py (run on the GPU box):
#   bash tools/sanitize.sh  -> gpurun_out/sanitize_<tool>_<case>.log and a summary
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for c in tma l1 cluster ensemble host csr; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
        python tools/sanitize_cases.py $c > gpurun_out/sanitize_${tool}_${c}.log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/sanitize_${tool}_${c}.log | tail -1)
    echo "$tool $c rc=$rc $summ"
  done
done
