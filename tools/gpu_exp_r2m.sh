# Round-2 (m): the overlapped varlen sort (HB_FLAG_INPUT_READY on varlen):
# parity test, sanitizer, and the bench's varlen line with / without the flag.
mkdir -p gpurun_out
T=r2ac
timeout 600 python -m pytest tests -q -m gpu -k "varlen" > gpurun_out/pytest_varlen_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_varlen_$T.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck_$T.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck_$T.log
for k in 1 2; do
timeout 600 python bench.py --workload varlen_md5 --steps 20 --warmup 5 --configs none --no-e2e > gpurun_out/bench_vl_${T}_$k.json 2> gpurun_out/bench_vl_${T}_$k.err
HB_PDL=0 timeout 600 python bench.py --workload varlen_md5 --steps 20 --warmup 5 --configs none --no-e2e > gpurun_out/bench_vl_nopdl_${T}_$k.json 2> gpurun_out/bench_vl_nopdl_${T}_$k.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_varlen_$T.csv \
  python bench.py --workload varlen_md5 --steps 3 --warmup 3 --configs none --no-e2e > /dev/null 2>&1
tail -n 2 gpurun_out/pytest_varlen_$T.log; tail -n 3 gpurun_out/sanitize_*_$T.log; grep -h headline gpurun_out/bench_vl_*${T}*.err
