# Round variants 3/4/5/6 in the shipping varlen MD5 loop (arms 53-56) vs the default (variant 1), configs[3].
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=5 AB_ARMS='{"dflt": {}, "h47": {"HB_VARLEN_KERNEL": "47"}, "v3": {"HB_VARLEN_KERNEL": "53"}, "v4": {"HB_VARLEN_KERNEL": "54"}, "v5": {"HB_VARLEN_KERNEL": "55"}, "v6": {"HB_VARLEN_KERNEL": "56"}}' \
  timeout 1200 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2ba.txt 2>&1
# second pass: idle 2 s before every arm (same power state), 8 rounds
AB_COOL=2 AB_ROUNDS=8 AB_ARMS='{"dflt": {}, "v4": {"HB_VARLEN_KERNEL": "54"}, "v6": {"HB_VARLEN_KERNEL": "56"}}' \
  timeout 1200 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2bb.txt 2>&1
cat gpurun_out/ab_varlen_r2bb.txt
