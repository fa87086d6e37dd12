set -u
mkdir -p gpurun_out
T=${T:-san1}
timeout 300 python tools/sanitize_cases.py > gpurun_out/sanitize_plain_$T.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/sanitize_plain_$T.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_$T.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_${tool}_$T.log
done
