set -u
mkdir -p gpurun_out
T=${T:-exp74}
A='{"ws3": {}, "ws3x2": {"HB_TMA_CFG": "ws3x2"}, "ws2x2": {"HB_TMA_CFG": "ws2x2"}, "ws3u": {"HB_TMA_CFG": "ws3u"}}'
AB_ARMS="$A" AB_ROUNDS=3 timeout 900 python tools/ab_env.py md5 16777216 1024 50 2>&1 | tail -4 | tee gpurun_out/ab_md5cfg_$T.txt
