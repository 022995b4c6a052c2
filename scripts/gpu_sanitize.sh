# compute-sanitizer over scripts/sanitize_workload.py: $1 = tag
T=${1:-san}
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 200 python scripts/sanitize_workload.py > gpurun_out/${T}_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/${T}_sanitize_$tool.log | tail -2
done
