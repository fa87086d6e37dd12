set -u
mkdir -p gpurun_out
T=${T:-final2}
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$T.log
timeout 300 python __graft_entry__.py 2>&1 | tail -1
