# Round-2 A/B: MD5 round variants 4 / 5 (variant 3's short chain with IADD3 off-chain sums).
mkdir -p gpurun_out
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=3 AB_ARMS='{"base": {}, "v1": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}, "v3": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "3"}, "v4": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "4"}, "v5": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "5"}}' AB_POINTS='md5:65536:256,md5:65536:1024,md5:65536:4096,md5:16384:1024,md5:131072:1024,md5:262144:1024,md5:1048576:1024,md5:4736:65536' timeout 1500 python tools/ab_mid.py > gpurun_out/ab_v45_r2m.txt 2>&1
AB_ROUNDS=3 AB_STEPS=60 AB_ARMS='{"v1": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}, "v4": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "4"}, "v5": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "5"}}' timeout 900 python tools/ab_power.py md5 > gpurun_out/ab_power_v45_r2m.txt 2>&1
cat gpurun_out/ab_v45_r2m.txt gpurun_out/ab_power_v45_r2m.txt
