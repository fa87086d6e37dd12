# Round-2 (f): headline-style interleaved A/B at configs[1] (cool-down, 5 warm-ups,
# 20 timed, HB_FLAG_INPUT_READY), varlen uniform-finish / L2-policy arms.
mkdir -p gpurun_out
HETOC_B200_LIB=libhetoc_b200_ab.so timeout 900 python -m pytest tests -q -m "gpu and ab" -k "varlen_every_length or tile_configs" > gpurun_out/pytest_ab_r2q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab_r2q.log
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=4 AB_COOL=3 AB_ARMS='{"dflt": {}, "w1v4": {"HB_TMA_CFG": "w1x2p", "HB_VARIANT": "4"}, "old": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}, "w1s4": {"HB_TMA_CFG": "w1x2s4", "HB_VARIANT": "4"}}' timeout 900 python tools/ab_headline.py md5 > gpurun_out/ab_headline_r2q.txt 2>&1
AB_ROUNDS=3 AB_COOL=3 AB_FLAGS=none AB_ARMS='{"dflt": {}, "old": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}}' timeout 600 python tools/ab_headline.py md5 > gpurun_out/ab_headline_noflag_r2q.txt 2>&1
AB_ROUNDS=5 AB_COOL=2 AB_ARMS='{"dflt": {}, "uni48": {"HB_VARLEN_KERNEL": "48"}, "hint47": {"HB_VARLEN_KERNEL": "47"}, "old21": {"HB_VARLEN_KERNEL": "21"}}' timeout 900 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2q.txt 2>&1
AB_ROUNDS=3 AB_COOL=2 AB_ARMS='{"dflt": {}, "uni48": {"HB_VARLEN_KERNEL": "48"}}' timeout 900 python tools/ab_varlen.py sha1 sm3 >> gpurun_out/ab_varlen_r2q.txt 2>&1
tail -n 2 gpurun_out/pytest_ab_r2q.log
cat gpurun_out/ab_headline_r2q.txt gpurun_out/ab_headline_noflag_r2q.txt gpurun_out/ab_varlen_r2q.txt | cut -c1-260
