set -x
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "workspace or phase_entry or contract" > gpurun_out/r2l_ws.log 2>&1; echo "ws rc=$?"
tail -3 gpurun_out/r2l_ws.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2l_sanitize_$tool.log 2>&1; echo "$tool rc=$?"
  tail -6 gpurun_out/r2l_sanitize_$tool.log
done
