set -u
mkdir -p gpurun_out
T=${T:-exp3}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
timeout 600 python tools/bench_configs.py gpurun_out/configs_$T.jsonl --quick > /dev/null 2>gpurun_out/configs_$T.err; echo "configs rc=$?"; cat gpurun_out/configs_$T.jsonl
timeout 900 python tools/ab_small.py > gpurun_out/ab_small_$T.txt 2>&1; echo "ab rc=$?"
