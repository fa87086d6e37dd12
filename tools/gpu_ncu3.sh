#!/bin/bash
# Launch list of the default bench command + ncu --set full of the default
# kernel per algorithm.  Keeps the MD5 .ncu-rep and raw/source CSV exports of
# all (gpurun_out is capped at 64 MiB).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 5 --warmup 3 > gpurun_out/ncu_bench_stdout_${TAG}.txt 2>&1; echo "ncu launches rc=$?"
for w in md5_1k sha1_1k sm3_1k; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fixed_tma -s 3 -c 1 \
    -o /tmp/prof_${w}_${TAG} python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_${w}_${TAG}.txt 2>&1
  echo "ncu $w rc=$?"
  ncu -i /tmp/prof_${w}_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_${w}_${TAG}.csv 2>/dev/null
  ncu -i /tmp/prof_${w}_${TAG}.ncu-rep --page details > gpurun_out/details_${w}_${TAG}.txt 2>/dev/null
done
cp /tmp/prof_md5_1k_${TAG}.ncu-rep gpurun_out/
ls -la gpurun_out; du -sh gpurun_out
