# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over scripts/sanitize_configs.py
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_configs.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool exit $?"; tail -2 gpurun_out/sanitizer/$tool.log
done
