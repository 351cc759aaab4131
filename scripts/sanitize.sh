# compute-sanitizer over the small workloads (memcheck, racecheck, synccheck)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_driver.py "$@" > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc $?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/sanitize_$tool.log | head -8
done
