set -u
mkdir -p gpurun_out
T=${T:-exp29}
timeout 600 python -m pytest tests -q -m gpu --timeout 300 -k "tile_configs or full_size" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$T.log
export AB_ARMS='{"l2_256": {}, "l2_128": {"HB_TMA_L2": "128"}, "l2_0": {"HB_TMA_L2": "0"}, "evict_first": {"HB_TMA_EVICT_FIRST": "1"}, "l2_128_ef": {"HB_TMA_L2": "128", "HB_TMA_EVICT_FIRST": "1"}}'
AB_ROUNDS=3 timeout 600 python tools/ab_env.py md5 16777216 1024 30 > gpurun_out/ab_tma_$T.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_tma_$T.txt
AB_ROUNDS=2 timeout 600 python tools/ab_env.py sha1 16777216 1024 10 >> gpurun_out/ab_tma_$T.txt 2>&1; tail -5 gpurun_out/ab_tma_$T.txt
