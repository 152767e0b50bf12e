# compute-sanitizer over tests/tools/sanitize_cases.py: memcheck, racecheck, synccheck, initcheck
mkdir -p gpurun_out
for t in memcheck synccheck racecheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 50 python tests/tools/sanitize_cases.py \
    > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok " gpurun_out/sanitize_$t.log | tail -12
done
