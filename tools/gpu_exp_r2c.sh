# Round-2 A/B (c): single-warp CTAs with NB = 1 / 2 / 4 messages per thread for
# mid-size MD5 batches, MD5 round variants 4 / 5, default-library GPU tests.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/smi_r2n.txt 2>&1
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r2n.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r2n.log
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=3 AB_ARMS='{"base": {}, "ws3v3": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "3"}, "w1x1v3": {"HB_TMA_CFG": "w1x1", "HB_VARIANT": "3"}, "w1x2v3": {"HB_TMA_CFG": "w1x2", "HB_VARIANT": "3"}, "w1x2v1": {"HB_TMA_CFG": "w1x2", "HB_VARIANT": "1"}, "w1x4v1": {"HB_TMA_CFG": "w1x4", "HB_VARIANT": "1"}, "w1x4v3": {"HB_TMA_CFG": "w1x4", "HB_VARIANT": "3"}, "w1x4v5": {"HB_TMA_CFG": "w1x4", "HB_VARIANT": "5"}, "w1x4s2": {"HB_TMA_CFG": "w1x4s2", "HB_VARIANT": "1"}}' AB_POINTS='md5:65536:1024,md5:65536:256,md5:65536:4096,md5:65536:16384,md5:16384:1024,md5:32768:1024,md5:131072:1024,sha1:65536:1024,sm3:65536:1024' timeout 1200 python tools/ab_mid.py > gpurun_out/ab_w1_r2n.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"base": {}, "v1": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}, "v3": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "3"}, "v4": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "4"}, "v5": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "5"}}' AB_POINTS='md5:65536:1024,md5:65536:4096,md5:262144:1024,md5:1048576:1024,md5:4736:65536' timeout 900 python tools/ab_mid.py > gpurun_out/ab_v45_r2n.txt 2>&1
AB_ROUNDS=2 AB_STEPS=40 AB_ARMS='{"v1": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}, "v4": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "4"}, "v5": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "5"}}' timeout 600 python tools/ab_power.py md5 > gpurun_out/ab_power_v45_r2n.txt 2>&1
tail -n 2 gpurun_out/pytest_gpu_r2n.log; cat gpurun_out/ab_w1_r2n.txt gpurun_out/ab_v45_r2n.txt gpurun_out/ab_power_v45_r2n.txt | cut -c1-220
