# Round-2 A/B: two messages per thread in the varlen kernel.
mkdir -p gpurun_out
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=5 AB_ARMS='{"dflt": {}, "x2": {"HB_VARLEN_KERNEL": "33"}, "x2_nb": {"HB_VARLEN_KERNEL": "33", "HB_SORT_QMAJOR": "0"}, "x2_16k": {"HB_VARLEN_KERNEL": "33", "HB_SORT_WINDOW": "16384"}}' timeout 900 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2i.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"dflt": {}, "x2": {"HB_VARLEN_KERNEL": "33"}}' timeout 900 python tools/ab_varlen.py sha1 sm3 >> gpurun_out/ab_varlen_r2i.txt 2>&1
cat gpurun_out/ab_varlen_r2i.txt
