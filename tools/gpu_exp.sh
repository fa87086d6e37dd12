set -u
mkdir -p gpurun_out
T=${T:-exp76}
A='{"v1": {}, "v0": {"HB_VARIANT": "0"}, "v2": {"HB_VARIANT": "2"}, "v3": {"HB_VARIANT": "3"}}'
AB_ARMS="$A" AB_ROUNDS=3 timeout 900 python tools/ab_env.py md5 16777216 1024 150 2>&1 | tail -4 | tee gpurun_out/ab_md5var_$T.txt
nvidia-smi --query-gpu=power.limit,power.draw,clocks.sm --format=csv
