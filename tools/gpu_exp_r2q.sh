# Round-2 (q): overlapped global sort for varlen SHA-1 / SM3 (HB_FLAG_INPUT_READY)
mkdir -p gpurun_out
T=r2ar
timeout 900 python -m pytest tests -q -m gpu -k "varlen" > gpurun_out/pytest_varlen_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_varlen_$T.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}_$T.log
done
for k in 1 2; do for a in sha1 sm3; do
timeout 600 python bench.py --workload varlen_$a --steps 20 --warmup 5 --configs none --no-e2e > gpurun_out/bench_vl_${a}_${T}_$k.json 2> gpurun_out/bench_vl_${a}_${T}_$k.err
HB_PDL=0 timeout 600 python bench.py --workload varlen_$a --steps 20 --warmup 5 --configs none --no-e2e > gpurun_out/bench_vl_${a}_nopdl_${T}_$k.json 2> gpurun_out/bench_vl_${a}_nopdl_${T}_$k.err
done; done
tail -n 2 gpurun_out/pytest_varlen_$T.log; tail -n 2 gpurun_out/sanitize_*_$T.log
grep -h headline gpurun_out/bench_vl_*_$T_*.err gpurun_out/bench_vl_*${T}*.err | sort | uniq
for f in gpurun_out/bench_vl_*${T}*.err; do echo "$f $(grep headline $f | cut -c1-80)"; done
