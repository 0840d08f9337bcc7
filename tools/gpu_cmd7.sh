set -o pipefail
mkdir -p gpurun_out/san
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -x > gpurun_out/gt7.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gt7.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_smoke.py > gpurun_out/san/$tool.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/san/$tool.log
done
