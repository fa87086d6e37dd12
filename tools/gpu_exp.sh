set -u
mkdir -p gpurun_out
T=${T:-exp10}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
for w in paper_sha1 paper_md5 paper_sm3 varlen_md5 md5_1k; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_${w}_$T.json 2> gpurun_out/bench_${w}_$T.err; echo "bench $w rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_${w}_$T.json')); r=d['roofline']; e=d['e2e'] or {}; print('$w', d['value'], d['unit'], d['mhash_per_s'], 'Mhash/s', r['bound'], r['frac'], 'e2e', e.get('value'), (e.get('roofline') or {}).get('frac'), d['parity'])"
done
timeout 300 python bench.py --impl reference --workload paper_sha1 --steps 3 --warmup 1 > gpurun_out/bench_ref_paper_sha1_$T.json 2>&1; echo "ref rc=$?"
