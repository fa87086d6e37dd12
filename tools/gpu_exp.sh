set -u
mkdir -p gpurun_out
T=${T:-exp73}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "pairs or width or geometry or pdl" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$T.log
A='{"default": {}, "nopair": {"HB_SMALL_PAIR": "0"}}'
for c in "md5 16777216 16 20" "md5 16777216 48 20" "md5 16777216 64 20"; do
  AB_ARMS="$A" timeout 600 python tools/ab_env.py $c 2>&1 | tail -2
done
