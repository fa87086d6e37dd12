set -u
mkdir -p gpurun_out
T=${T:-exp25}
timeout 900 python -m pytest tests/test_multiproc.py tests/test_abi.py -q -m gpu --timeout 600 > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_$T.log
