# compute-sanitizer over every kernel shape: default library, then the A/B library.
mkdir -p gpurun_out
T=${1:-r2k}
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}_$T.log
  HETOC_B200_LIB=libhetoc_b200_ab.so timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_ab_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}_ab_$T.log
done
tail -n 3 gpurun_out/sanitize_*_$T.log
