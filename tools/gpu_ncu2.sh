#!/bin/bash
# ncu captures of specific (workload, cfg, variant) points: args "wl:cfg:var ..."
set -u
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read w c v <<< "$spec"
  HB_TMA_CFG=$c HB_VARIANT=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fixed_tma -s 3 -c 1 \
    -o gpurun_out/prof_${w}_${c}_v${v} python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_${w}_${c}_v${v}.txt 2>&1
  echo "ncu $spec rc=$?"
done
