# Round-2 validation pass of the final defaults: GPU tests on both libraries,
# smoke, default bench + reference arm, paper workloads, compute-sanitizer
# (memcheck / racecheck / synccheck on the shipped library, memcheck on the
# A/B library), launch list of the default bench command.
TAG=${1:-r2t}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/smi_$TAG.txt 2>&1
# ncu --set full of the headline kernel first (bench.py reads its traffic from profiles/ncu_summary.json;
# fold here with: python tools/ncu_configs.py fold $TAG gpurun_out/ncu_cfg_${TAG}_raw.csv gpurun_out/ncu_cfg_${TAG}_order.json)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fixed|k_varlen|k_generic|k_decimal" \
  -o /tmp/ncu_cfg_$TAG python tools/ncu_configs.py run gpurun_out/ncu_cfg_${TAG}_order.json ${NCU_CONFIGS:-md5_1k} > gpurun_out/ncu_cfg_$TAG.log 2>&1
ncu -i /tmp/ncu_cfg_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_cfg_${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/ncu_cfg_$TAG.ncu-rep --page source --csv > gpurun_out/ncu_cfg_${TAG}_source.csv 2>/dev/null
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
HETOC_B200_LIB=libhetoc_b200_ab.so timeout 900 python -m pytest tests -q -m "gpu and ab" > gpurun_out/pytest_ab_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
SECONDS=0; timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench wall $SECONDS s" >> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
for w in paper_md5 paper_sha1 paper_sm3; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --configs none > gpurun_out/bench_${w}_$TAG.json 2> gpurun_out/bench_${w}_$TAG.err
done
{ for a in md5 sha1 sm3; do python tools/digest_probe.py $a 0 55 1024 4096; done
  HB_SMALL_POLL=0 python tools/digest_probe.py md5 55 1024 | sed "s/^/HB_SMALL_POLL=0 /"; } > gpurun_out/digest_probe_$TAG.txt 2>&1
python tools/zero_copy_probe.py > gpurun_out/zero_copy_$TAG.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}_$TAG.log
done
HETOC_B200_LIB=libhetoc_b200_ab.so timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck_ab_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck_ab_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 5 --warmup 3 --configs none > gpurun_out/ncu_bench_stdout_$TAG.txt 2>&1
for f in gpurun_out/pytest_gpu_$TAG.log gpurun_out/pytest_ab_$TAG.log gpurun_out/smoke_$TAG.log gpurun_out/sanitize_*_$TAG.log; do echo "== $f"; tail -n 3 $f; done
tail -n 3 gpurun_out/bench_$TAG.err
