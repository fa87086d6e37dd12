export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=5 AB_ARMS='{"v16": {"HB_VARLEN_KERNEL": "0"}, "u1": {"HB_VARLEN_KERNEL": "1"}, "u2": {"HB_VARLEN_KERNEL": "2"}, "u1_win16k": {"HB_VARLEN_KERNEL": "1", "HB_SORT_WINDOW": "16384"}}' timeout 600 python tools/ab_varlen.py md5 sha1 sm3 > gpurun_out/ab_varlen_r2a.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"base": {}, "nopdl": {"HB_PDL": "0"}}' AB_POINTS='md5:65536:256,md5:65536:1024,md5:65536:4096,sha1:65536:256,sha1:65536:1024,sm3:65536:256,sm3:65536:1024,sha1:65536:64,md5:131072:1024,md5:262144:1024' timeout 900 python tools/ab_mid.py > gpurun_out/ab_mid_r2a.txt 2>&1
cat gpurun_out/ab_varlen_r2a.txt gpurun_out/ab_mid_r2a.txt
