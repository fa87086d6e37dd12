#!/bin/bash
# GPU tests + ncu launch list + ncu full captures of the top kernels.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_md5.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_bench_stdout.txt 2>&1; echo "ncu launches rc=$?"
for w in md5_1k sha1_1k sm3_1k; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fixed_tma -s 3 -c 1 \
    -o gpurun_out/prof_$w python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_$w.txt 2>&1
  echo "ncu $w rc=$?"
done
ls -la gpurun_out
