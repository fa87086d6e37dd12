# Round-2 A/B: configs[1] arms under sustained load (power limit).
mkdir -p gpurun_out
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE > gpurun_out/smi_power_r2h.txt 2>&1
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=3 AB_STEPS=60 AB_ARMS='{"base": {}, "v0": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "0"}, "v2": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "2"}, "v3": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "3"}, "ws2": {"HB_TMA_CFG": "ws2"}, "ws3n": {"HB_TMA_CFG": "ws3n"}, "ws3x2": {"HB_TMA_CFG": "ws3x2"}, "direct": {"HB_DIRECT_MAX_L": "2048"}}' timeout 1200 python tools/ab_power.py md5 > gpurun_out/ab_power_r2h.txt 2>&1
cat gpurun_out/ab_power_r2h.txt
grep -i -A12 "Power Readings\|Power Limit" gpurun_out/smi_power_r2h.txt | head -40
