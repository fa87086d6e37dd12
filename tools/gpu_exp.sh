set -u
mkdir -p gpurun_out/sanitizer_r1b
D=gpurun_out/sanitizer_r1b
timeout 600 python tools/sanitize_cases.py > $D/plain.log 2>&1; echo "plain rc=$?"; tail -1 $D/plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > $D/$tool.log 2>&1; echo "$tool rc=$?"; tail -2 $D/$tool.log
done
