set -u
mkdir -p gpurun_out
T=${T:-exp67}
timeout 600 python bench.py --workload sha1_64 > gpurun_out/bench_sha1_64_$T.json 2>gpurun_out/bench_sha1_64_$T.err; echo rc=$?
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['parity'], d['config']['l2'])" gpurun_out/bench_sha1_64_$T.json
timeout 900 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$T.log
