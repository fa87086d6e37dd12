set -u
mkdir -p gpurun_out
T=${T:-exp58}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_runtime.py -x -q -m gpu > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$T.log
A='{"pdl": {}, "nopdl": {"HB_PDL": "0"}}'
for c in "md5 16384 1024 100" "md5 4096 16384 50" "sha1 65536 4096 20" "sm3 16384 1024 50" "md5 16777216 1024 10" "sha1 65536 64 200"; do
  AB_ARMS="$A" timeout 600 python tools/ab_env.py $c 2>&1 | tail -2
done | tee gpurun_out/ab_pdl_$T.txt
for r in 1 2; do for p in 1 0; do
  HB_PDL=$p timeout 600 python bench.py --workload sha1_64 --no-cpu --no-e2e > gpurun_out/b64_${p}_$T.json 2>/dev/null
  echo "sha1_64 PDL=$p $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])" gpurun_out/b64_${p}_$T.json)"
done; done | tee -a gpurun_out/ab_pdl_$T.txt
