set -u
mkdir -p gpurun_out
T=${T:-exp42}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "decimal" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
AB_ARMS=v1_fma_digits,v1_run,v3_run timeout 900 python tools/ab_decimal.py md5 sha1 sm3 > gpurun_out/ab_decimal_$T.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_decimal_$T.txt
