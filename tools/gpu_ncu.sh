#!/bin/bash
# ncu --set full of k_fixed_tma for the given workloads (default variant unless HB_VARIANT set)
set -u
mkdir -p gpurun_out
TAG=${TAG:-x}
for w in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fixed_tma -s 3 -c 1 \
    -o gpurun_out/prof_${w}_${TAG} python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_${w}_${TAG}.txt 2>&1
  echo "ncu $w rc=$?"
done
