# Round-2 A/B batch (run under gpurun from the repo root).  ncu reports stay
# in /tmp on the box (only CSV exports come back: gpurun_out/ <= 64 MiB).
mkdir -p gpurun_out
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=5 AB_ARMS='{"v16": {"HB_VARLEN_KERNEL": "20"}, "pf": {"HB_VARLEN_KERNEL": "21"}, "v16_qm": {"HB_VARLEN_KERNEL": "20", "HB_SORT_QMAJOR": "1"}, "pf_qm": {"HB_VARLEN_KERNEL": "21", "HB_SORT_QMAJOR": "1"}, "v16_qm16k": {"HB_VARLEN_KERNEL": "20", "HB_SORT_QMAJOR": "1", "HB_SORT_WINDOW": "16384"}, "pf_qm16k": {"HB_VARLEN_KERNEL": "21", "HB_SORT_QMAJOR": "1", "HB_SORT_WINDOW": "16384"}, "u1_qm": {"HB_VARLEN_KERNEL": "1", "HB_SORT_QMAJOR": "1"}}' timeout 900 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2d.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"base": {}, "v3": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "3"}, "v0": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "0"}, "v1nopdl": {"HB_PDL": "0"}, "v3nopdl": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "3", "HB_PDL": "0"}}' AB_POINTS='md5:65536:256,md5:65536:512,md5:65536:1024,md5:65536:2048,md5:65536:4096,md5:65536:16384,md5:16384:1024,md5:16384:16384,md5:131072:1024,md5:262144:1024,md5:524288:1024,md5:4096:65536' timeout 1500 python tools/ab_mid.py > gpurun_out/ab_mid_r2c.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"base": {}, "c3": {"HB_CONST_VARIANT": "3"}}' AB_POINTS='md5:65536:64,md5:65536:128,md5:1048576:64,md5:65536:16,sha1:65536:64,sha1:1048576:64,sm3:65536:64' timeout 900 python tools/ab_mid.py > gpurun_out/ab_c1_r2c.txt 2>&1
unset HETOC_B200_LIB
SCAN='md5:1024' timeout 900 python tools/ab_scan.py > gpurun_out/scan_r2b.txt 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_fixed|k_varlen|k_generic|k_decimal" \
  -o /tmp/ncu_cfg_r2a python tools/ncu_configs.py run gpurun_out/ncu_cfg_r2a_order.json > gpurun_out/ncu_cfg_r2a.log 2>&1
ncu -i /tmp/ncu_cfg_r2a.ncu-rep --page raw --csv > gpurun_out/ncu_cfg_r2a_raw.csv 2>/dev/null
ls -la gpurun_out
cat gpurun_out/ab_varlen_r2d.txt gpurun_out/ab_mid_r2c.txt gpurun_out/ab_c1_r2c.txt gpurun_out/scan_r2b.txt
tail -n 3 gpurun_out/ncu_cfg_r2a.log
