set -x
for tool in memcheck racecheck synccheck; do
  timeout 1700 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2s_sanitize_$tool.log 2>&1; echo "$tool rc=$?"
  tail -4 gpurun_out/r2s_sanitize_$tool.log
done
