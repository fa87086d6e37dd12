set -u
mkdir -p gpurun_out
T=${T:-exp19}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
for w in md5_1k sm3_1k varlen_md5 paper_md5 sha1_64; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_${w}_$T.json 2> gpurun_out/bench_${w}_$T.err; echo "bench $w rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_${w}_$T.json')); r=d['roofline']; e=d['e2e'] or {}; print('$w', d['value'], d['mhash_per_s'], d['scaling'], r['bound'], r['frac'], 'e2e', e.get('value'), e.get('h2d_bytes_per_step'), e.get('d2h_bytes_per_step'), (e.get('roofline') or {}).get('frac'), d['parity'], d['gpu_launches'])"
done
