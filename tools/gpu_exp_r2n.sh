# Round-2 (n): varlen realignment on the FMA pipe (arm 52: IMAD.HI + IMAD
# instead of funnel shifts, sort keyed on a-1) for the ALU-bound SHA-1 / SM3.
mkdir -p gpurun_out
export HETOC_B200_LIB=libhetoc_b200_ab.so
timeout 900 python -m pytest tests -q -m "gpu and ab" -k "varlen_every_length" > gpurun_out/pytest_ab_r2ae.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab_r2ae.log
AB_ROUNDS=4 AB_COOL=2 AB_ARMS='{"dflt": {}, "fma52": {"HB_VARLEN_KERNEL": "52"}, "plain20": {"HB_VARLEN_KERNEL": "20"}}' timeout 1200 python tools/ab_varlen.py sha1 sm3 > gpurun_out/ab_varlen_r2ae.txt 2>&1
AB_ROUNDS=3 AB_COOL=2 AB_ARMS='{"dflt": {}, "fma52": {"HB_VARLEN_KERNEL": "52"}}' timeout 600 python tools/ab_varlen.py md5 >> gpurun_out/ab_varlen_r2ae.txt 2>&1
for alg in sha1 sm3; do HB_VARLEN_KERNEL=52 timeout 300 ncu --set full --clock-control none -k regex:"k_varlen" -s 1 -c 1 -o /tmp/ncu_vl52_$alg python tools/ncu_one.py $alg varlen > /dev/null 2>&1
ncu -i /tmp/ncu_vl52_$alg.ncu-rep --page raw --csv > gpurun_out/raw_vl52_${alg}_r2ae.csv 2>/dev/null; done
tail -n 2 gpurun_out/pytest_ab_r2ae.log; cat gpurun_out/ab_varlen_r2ae.txt
