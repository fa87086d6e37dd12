set -u
mkdir -p gpurun_out
T=${T:-exp61}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "pdl" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
HB_PDL=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "pdl" 2>&1 | tail -1
