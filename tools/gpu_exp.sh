set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/pytest_exp1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_exp1.log
SWEEP_CFGS=ws3,ws3x2,ws2x2 SWEEP_VARS=13 SWEEP_ROUNDS=3 timeout 600 python tools/variant_sweep.py md5 sha1 sm3 > gpurun_out/variant_exp1.txt 2>&1; echo "sweep rc=$?"; cat gpurun_out/variant_exp1.txt
timeout 600 python tools/bench_configs.py gpurun_out/configs_exp1.jsonl --quick > /dev/null 2>gpurun_out/configs_exp1.err; echo "configs rc=$?"; cat gpurun_out/configs_exp1.jsonl
timeout 900 python tools/bench_configs.py gpurun_out/sweep_exp1.jsonl --sweep-only > /dev/null 2>gpurun_out/sweep_exp1.err; echo "sweep rc=$?"; wc -l gpurun_out/sweep_exp1.jsonl
