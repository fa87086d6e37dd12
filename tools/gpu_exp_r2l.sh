# Round-2 (l): varlen MD5 lean loop unrolled by two with the fifth granule
# carried (arm 51) against the shipped lean loop; parity of the arm; launch
# list of the varlen workload (sort vs hash kernel time).
mkdir -p gpurun_out
export HETOC_B200_LIB=libhetoc_b200_ab.so
timeout 900 python -m pytest tests -q -m "gpu and ab" -k "varlen_every_length" > gpurun_out/pytest_ab_r2ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab_r2ab.log
AB_ROUNDS=6 AB_COOL=2 AB_ARMS='{"dflt": {}, "c51": {"HB_VARLEN_KERNEL": "51"}}' timeout 900 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2ab.txt 2>&1
AB_ROUNDS=3 AB_COOL=2 AB_ARMS='{"dflt": {}, "c51": {"HB_VARLEN_KERNEL": "51"}}' timeout 900 python tools/ab_varlen.py sha1 sm3 >> gpurun_out/ab_varlen_r2ab.txt 2>&1
HB_VARLEN_KERNEL=51 timeout 300 ncu --set full --clock-control none -k regex:"k_varlen" -s 1 -c 1 -o /tmp/ncu_vl51 python tools/ncu_one.py md5 varlen > gpurun_out/ncu_vl51_r2ab.log 2>&1
ncu -i /tmp/ncu_vl51.ncu-rep --page raw --csv > gpurun_out/raw_vl51_r2ab.csv 2>/dev/null
unset HETOC_B200_LIB
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_varlen_r2ab.csv \
  python bench.py --workload varlen_md5 --steps 3 --warmup 3 --configs none --no-e2e > /dev/null 2>&1
tail -n 2 gpurun_out/pytest_ab_r2ab.log; cat gpurun_out/ab_varlen_r2ab.txt
grep -E "k_sort|k_varlen" gpurun_out/launches_varlen_r2ab.csv | awk -F'","' '{print $5, $(NF)}' | sort | uniq -c | head; grep -c k_varlen gpurun_out/launches_varlen_r2ab.csv
