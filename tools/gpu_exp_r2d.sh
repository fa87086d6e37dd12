# Round-2 A/B (d): MD5 round variants 4 / 6 / 7 on every MD5 kernel family
# (TMA tiles, single-warp NB=2 tiles, compile-time-width, runs-of-ten decimal)
# and the lean varlen block loop (k_varlen16l) against the default varlen kernel.
mkdir -p gpurun_out
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=3 AB_ARMS='{"dflt": {}, "l40": {"HB_VARLEN_KERNEL": "40"}, "l41": {"HB_VARLEN_KERNEL": "41"}, "l42v4": {"HB_VARLEN_KERNEL": "42"}, "l43v4": {"HB_VARLEN_KERNEL": "43"}, "l44v6": {"HB_VARLEN_KERNEL": "44"}, "l45v7": {"HB_VARLEN_KERNEL": "45"}}' timeout 900 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2o.txt 2>&1
AB_ROUNDS=2 AB_ARMS='{"dflt": {}, "l40": {"HB_VARLEN_KERNEL": "40"}, "l41": {"HB_VARLEN_KERNEL": "41"}}' timeout 600 python tools/ab_varlen.py sha1 sm3 >> gpurun_out/ab_varlen_r2o.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"base": {}, "v1": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}, "v4": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "4"}, "v6": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "6"}, "v7": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "7"}, "w1x2v4": {"HB_TMA_CFG": "w1x2", "HB_VARIANT": "4"}}' AB_POINTS='md5:65536:1024,md5:65536:4096,md5:262144:1024,md5:1048576:1024,md5:4194304:1024,md5:4736:65536,md5:1048576:256' timeout 900 python tools/ab_mid.py > gpurun_out/ab_v467_r2o.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"default": {}, "cv4": {"HB_CONST_VARIANT": "4"}}' AB_POINTS='16777216:64,16777216:128,65536:64,1048576:128,16777216:48' timeout 600 python tools/ab_small.py md5 > gpurun_out/ab_small_v4_r2o.txt 2>&1
AB_N=1000000000 AB_ARMS=v1_run,v4_run timeout 600 python tools/ab_decimal.py md5 > gpurun_out/ab_decimal_v4_r2o.txt 2>&1
AB_ROUNDS=2 AB_STEPS=40 AB_ARMS='{"v1": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}, "v4": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "4"}, "v6": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "6"}}' timeout 600 python tools/ab_power.py md5 > gpurun_out/ab_power_v46_r2o.txt 2>&1
cat gpurun_out/ab_varlen_r2o.txt gpurun_out/ab_v467_r2o.txt gpurun_out/ab_small_v4_r2o.txt gpurun_out/ab_decimal_v4_r2o.txt gpurun_out/ab_power_v46_r2o.txt | cut -c1-200
