set -u
mkdir -p gpurun_out
T=${T:-exp11}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$T.log
for w in paper_md5 paper_sha1; do
  timeout 900 python bench.py --workload $w --no-e2e > gpurun_out/bench_${w}_$T.json 2> gpurun_out/bench_${w}_$T.err; echo "bench $w rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_${w}_$T.json')); r=d['roofline']; print('$w', d['value'], d['unit'], d['mhash_per_s'], 'Mhash/s', r['bound'], r['frac'], d['parity'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decimal -s 3 -c 1 \
  -o /tmp/prof_dec_$T python bench.py --workload paper_md5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_dec_$T.txt 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_dec_$T.ncu-rep --page raw --csv > gpurun_out/raw_paper_md5_$T.csv 2>/dev/null
ncu -i /tmp/prof_dec_$T.ncu-rep --page source --csv > gpurun_out/source_paper_md5_$T.csv 2>/dev/null
