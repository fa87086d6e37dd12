set -u
mkdir -p gpurun_out
T=${T:-final3}
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$T.log
timeout 300 python __graft_entry__.py 2>&1 | tail -1
timeout 2400 python tools/bench_configs.py gpurun_out/configs_$T.jsonl > /dev/null 2> gpurun_out/configs_$T.err; echo "configs rc=$?"; wc -l < gpurun_out/configs_$T.jsonl; grep -c '"bit_exact_sample": true' gpurun_out/configs_$T.jsonl
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['parity'])" gpurun_out/bench_$T.json
