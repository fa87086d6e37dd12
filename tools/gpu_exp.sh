set -u
mkdir -p gpurun_out
T=${T:-exp70}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "decimal" 2>&1 | tail -2
timeout 600 python bench.py --workload paper_md5 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['mhash_per_s'], d['roofline']['frac'])"
