set -u
mkdir -p gpurun_out
T=${T:-exp68}
for r in 1 2; do for e in 0 1; do
HB_PDL_EARLY=$e timeout 600 python bench.py --workload sha1_64 --no-cpu --no-e2e > gpurun_out/b64_${e}_$T.json 2>/dev/null; echo "early=$e $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])" gpurun_out/b64_${e}_$T.json)"
done; done
HB_PDL_EARLY=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "pdl or width or geometry" 2>&1 | tail -1
