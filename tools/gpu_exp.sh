set -u
mkdir -p gpurun_out
T=${T:-exp32}
for w in sha1_64 md5_1k; do timeout 600 python bench.py --workload $w --no-cpu > gpurun_out/b_${w}_$T.json 2> gpurun_out/b_${w}_$T.err; echo "$w rc=$?"; python -c "import json,sys; d=json.load(open('gpurun_out/b_${w}_$T.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['config']['launch'])"; grep "kernel-only" gpurun_out/b_${w}_$T.err; done
timeout 600 python -m pytest tests -q -m gpu -k "graph or multirank" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$T.log
