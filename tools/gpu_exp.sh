set -u
mkdir -p gpurun_out
T=${T:-exp59}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "geometry or tile or width" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$T.log
timeout 1800 python tools/bench_configs.py gpurun_out/sweep_$T.jsonl --sweep-only > /dev/null 2> gpurun_out/sweep_$T.err; echo "sweep rc=$?"; wc -l gpurun_out/sweep_$T.jsonl
