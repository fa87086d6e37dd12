set -u
mkdir -p gpurun_out
T=${T:-exp63}
timeout 900 python -m pytest tests/test_multiproc.py -x -q -m gpu -k "multirank" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$T.log
timeout 600 python bench.py --workload sha1_64 --steps 20 --warmup 3 2>/dev/null | tail -1 | cut -c1-400
timeout 600 python bench.py --workload md5_1k --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['clocks'], d['roofline']['peak_source'])"
