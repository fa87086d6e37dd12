set -u
mkdir -p gpurun_out
T=${T:-exp34}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$T.log
