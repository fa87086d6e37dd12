# Round-2 A/B: register caps of the varlen kernels (MD5 configs[3]).
mkdir -p gpurun_out
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=5 AB_ARMS='{"dflt": {}, "pf_minb8": {"HB_VARLEN_KERNEL": "29"}, "pf_minb9": {"HB_VARLEN_KERNEL": "30"}, "plain_minb10": {"HB_VARLEN_KERNEL": "31"}, "pfl1": {"HB_VARLEN_KERNEL": "32"}, "plain": {"HB_VARLEN_KERNEL": "20"}}' timeout 900 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2g.txt 2>&1
cat gpurun_out/ab_varlen_r2g.txt
