#!/bin/bash
# Full evidence pass on one GPU: GPU tests, smoke, default bench + reference
# arm, every bench workload, the BASELINE configs + configs[4] sweep, the
# launch list of the default bench command, and ncu --set full of the default
# kernel of each main workload (raw/source CSV exports; MD5 .ncu-rep kept).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
tail -2 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2>&1; echo "ref rc=$?"
for w in ${BENCH_WORKLOADS:-sha1_64 sm3_1k sha1_1k varlen_md5 varlen_sha1 varlen_sm3 paper_sha1 paper_md5 paper_sm3}; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_${w}_${TAG}.json 2> gpurun_out/bench_${w}_${TAG}.err; echo "bench $w rc=$?"
done
timeout 1200 python tools/bench_configs.py gpurun_out/configs_${TAG}.jsonl > /dev/null 2> gpurun_out/configs_${TAG}.err; echo "configs rc=$?"
if [ "${SKIP_NCU:-0}" = "0" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 5 --warmup 3 > gpurun_out/ncu_bench_stdout_${TAG}.txt 2>&1; echo "ncu launches rc=$?"
for w in ${NCU_WORKLOADS:-md5_1k sha1_1k sm3_1k varlen_md5 paper_md5}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fixed|k_varlen|k_decimal" -s 3 -c 1 \
    -o /tmp/prof_${w}_${TAG} python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_${w}_${TAG}.txt 2>&1
  echo "ncu $w rc=$?"
  ncu -i /tmp/prof_${w}_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_${w}_${TAG}.csv 2>/dev/null
  ncu -i /tmp/prof_${w}_${TAG}.ncu-rep --page source --csv > gpurun_out/source_${w}_${TAG}.csv 2>/dev/null
done
cp /tmp/prof_md5_1k_${TAG}.ncu-rep gpurun_out/ 2>/dev/null
fi
du -sh gpurun_out
