# Round-2 (h): varlen MD5 uniform-finish arms (49, 50 = + L2 policies) against
# the lean default (l40) and the L2-policy lean loop (47); parity of the arms.
mkdir -p gpurun_out
HETOC_B200_LIB=libhetoc_b200_ab.so timeout 900 python -m pytest tests -q -m "gpu and ab" -k "varlen_every_length" > gpurun_out/pytest_ab_r2s.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab_r2s.log
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=6 AB_COOL=2 AB_ARMS='{"dflt": {}, "u49": {"HB_VARLEN_KERNEL": "49"}, "u50hint": {"HB_VARLEN_KERNEL": "50"}, "h47": {"HB_VARLEN_KERNEL": "47"}}' timeout 900 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2s.txt 2>&1
AB_ROUNDS=3 AB_COOL=2 AB_ARMS='{"dflt": {}, "u49": {"HB_VARLEN_KERNEL": "49"}}' timeout 900 python tools/ab_varlen.py sha1 sm3 >> gpurun_out/ab_varlen_r2s.txt 2>&1
for k in 49 50; do HB_VARLEN_KERNEL=$k timeout 600 ncu --set full --clock-control none -k regex:"k_varlen" -s 1 -c 1 -o /tmp/ncu_vl${k} python tools/ncu_one.py md5 varlen > gpurun_out/ncu_vl${k}_r2s.log 2>&1
ncu -i /tmp/ncu_vl${k}.ncu-rep --page raw --csv > gpurun_out/raw_vl${k}_r2s.csv 2>/dev/null; done
tail -n 2 gpurun_out/pytest_ab_r2s.log; cut -c1-200 gpurun_out/ab_varlen_r2s.txt
