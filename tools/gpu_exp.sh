set -u
mkdir -p gpurun_out
T=${T:-exp50}
nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node" | head -8
for r in 1 2; do
for th in 8 12 16 4; do
  echo "threads=$th $(HB_MEMCPY_THREADS=$th timeout 600 python tools/e2e_pageable.py md5 4194304 1024 2>&1 | tail -1)"
done
done | tee gpurun_out/memcpy_threads_$T.txt
