set -u
mkdir -p gpurun_out
T=${T:-exp71}
timeout 900 python bench.py --workload paper_md5 > gpurun_out/bench_paper_md5_$T.json 2>gpurun_out/bench_paper_md5_$T.err; echo rc=$?
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['mhash_per_s'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['mhash_per_s'], d['cpu_baseline']['mhash_per_s'], d['parity'], d['clocks'])" gpurun_out/bench_paper_md5_$T.json
