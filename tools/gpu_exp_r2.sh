# Round-2 validation pass: GPU tests (default + A/B), smoke, default bench +
# reference arm, paper workloads, ncu launch list of the headline command,
# compute-sanitizer over every kernel shape.
mkdir -p gpurun_out
T=${1:-r2j}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/smi_$T.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$T.log
HETOC_B200_LIB=libhetoc_b200_ab.so timeout 900 python -m pytest tests -q -m "gpu and ab" > gpurun_out/pytest_ab_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
SECONDS=0; timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench wall $SECONDS s" >> gpurun_out/bench_$T.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
for wl in paper_md5 paper_sha1 paper_sm3; do timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 > gpurun_out/bench_${wl}_$T.json 2> gpurun_out/bench_${wl}_$T.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 1 --configs none --no-e2e > gpurun_out/ncu_launch_bench_$T.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck_$T.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck_$T.log
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_synccheck_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_synccheck_$T.log
tail -n 3 gpurun_out/pytest_gpu_$T.log gpurun_out/pytest_ab_$T.log gpurun_out/smoke_$T.log gpurun_out/sanitize_*_$T.log
tail -n 2 gpurun_out/bench_$T.err
