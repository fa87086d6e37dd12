set -u
mkdir -p gpurun_out
T=${T:-exp4}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_$T.log
timeout 600 python tools/bench_configs.py gpurun_out/configs_$T.jsonl --quick > /dev/null 2>gpurun_out/configs_$T.err; echo "configs rc=$?"; cut -c1-250 gpurun_out/configs_$T.jsonl
