set -u
mkdir -p gpurun_out
T=${T:-exp66}
for r in 1 2; do timeout 600 python bench.py --workload sha1_64 --no-cpu > gpurun_out/b64_${r}_$T.json 2>gpurun_out/b64_${r}_$T.err; python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['gpu_launches'], d['parity'])" gpurun_out/b64_${r}_$T.json; grep "kernel-only" gpurun_out/b64_${r}_$T.err; done
