# Round-2 A/B batch (run under gpurun from the repo root): varlen carry arms,
# mid-size (n = 2^16) tile/variant arms, C1 arms, warps-per-scheduler scan,
# one ncu --set full launch per BASELINE config (roofline.traffic).
mkdir -p gpurun_out
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=5 AB_ARMS='{"v16": {"HB_VARLEN_KERNEL": "20"}, "carry": {"HB_VARLEN_KERNEL": "25"}, "carry_ld1": {"HB_VARLEN_KERNEL": "28"}, "pf": {"HB_VARLEN_KERNEL": "21"}, "ld1": {"HB_VARLEN_KERNEL": "23"}, "ld1pf": {"HB_VARLEN_KERNEL": "24"}, "u1": {"HB_VARLEN_KERNEL": "1"}, "c64": {"HB_VARLEN_KERNEL": "20", "HB_SMALL_CTA": "64"}}' timeout 900 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2c.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"v16": {"HB_VARLEN_KERNEL": "20"}, "carry": {"HB_VARLEN_KERNEL": "25"}, "carry_ld1": {"HB_VARLEN_KERNEL": "28"}}' timeout 900 python tools/ab_varlen.py sha1 sm3 >> gpurun_out/ab_varlen_r2c.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"base": {}, "ws3x2": {"HB_TMA_CFG": "ws3x2"}, "ws2x2": {"HB_TMA_CFG": "ws2x2"}, "v0": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "0"}, "v2": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "2"}, "v3": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "3"}, "nopdl": {"HB_PDL": "0"}}' AB_POINTS='md5:65536:256,md5:65536:1024,md5:65536:4096,sha1:65536:256,sha1:65536:1024,sha1:65536:4096,sm3:65536:256,sm3:65536:1024' timeout 1200 python tools/ab_mid.py > gpurun_out/ab_mid_r2b.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"base": {}, "pair": {"HB_SMALL_PAIR_ALL": "1"}, "cta64": {"HB_SMALL_CTA": "64"}, "cta32": {"HB_SMALL_CTA": "32"}, "plain": {"HB_CONST_VARIANT": "0"}, "nopdl": {"HB_PDL": "0"}}' AB_POINTS='sha1:65536:64,md5:65536:64,sm3:65536:64,sha1:65536:128' timeout 900 python tools/ab_mid.py > gpurun_out/ab_c1_r2b.txt 2>&1
unset HETOC_B200_LIB
SCAN='md5:1024,sha1:1024,sm3:1024,md5:256,sha1:64' timeout 900 python tools/ab_scan.py > gpurun_out/scan_r2a.txt 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_fixed|k_varlen|k_generic|k_decimal" \
  -o gpurun_out/ncu_cfg_r2a python tools/ncu_configs.py run gpurun_out/ncu_cfg_r2a_order.json > gpurun_out/ncu_cfg_r2a.log 2>&1
ncu -i gpurun_out/ncu_cfg_r2a.ncu-rep --page raw --csv > gpurun_out/ncu_cfg_r2a_raw.csv 2>/dev/null
tail -n 40 gpurun_out/ab_varlen_r2c.txt gpurun_out/ab_mid_r2b.txt gpurun_out/ab_c1_r2b.txt gpurun_out/scan_r2a.txt
tail -n 5 gpurun_out/ncu_cfg_r2a.log
