# diff-max-min GPU parity + compute-sanitizer on small configs (C1-C3 reduced)
python -m pytest tests/test_gpu_dmaxmin.py -x -q > gpurun_out/dmaxmin.log 2>&1; tail -3 gpurun_out/dmaxmin.log
mkdir -p gpurun_out/sanitizer
for tool in memcheck initcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_configs.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer/$tool.log
done
