set -u
mkdir -p gpurun_out
T=${T:-exp48}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "pipelined" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
AB_ARMS=1,4 timeout 900 python tools/ab_pipe.py > gpurun_out/ab_pipe_$T.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_pipe_$T.txt
