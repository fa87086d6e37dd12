set -u
mkdir -p gpurun_out
T=${T:-exp54}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "chunk or pinned or pipelined or concurrent or error" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$T.log
timeout 300 python tools/latency_probe.py 2>&1 | tee gpurun_out/latency_$T.txt
timeout 600 python bench.py --workload sha1_64 > gpurun_out/bench_sha1_64_$T.json 2>/dev/null; python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])" gpurun_out/bench_sha1_64_$T.json
