# Round-2 (j): bench vs A/B timing of configs[3] MD5 in one session; SHA-1 /
# SM3 varlen with the windowed sort and L2 policies (DRAM traffic of the
# ALU-bound varlen kernels).
mkdir -p gpurun_out
T=r2w
timeout 600 python bench.py --workload varlen_md5 --steps 20 --warmup 5 --configs none --no-e2e > gpurun_out/bench_varlen_md5_$T.json 2> gpurun_out/bench_varlen_md5_$T.err
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=3 AB_COOL=2 AB_ARMS='{"dflt": {}}' timeout 300 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_$T.txt 2>&1
AB_ROUNDS=3 AB_COOL=2 AB_ARMS='{"dflt": {}, "win": {"HB_VARLEN_SORT": "window"}, "win_hint47": {"HB_VARLEN_SORT": "window", "HB_VARLEN_KERNEL": "47"}, "glob_hint47": {"HB_VARLEN_KERNEL": "47"}, "win_u50": {"HB_VARLEN_SORT": "window", "HB_VARLEN_KERNEL": "50"}, "glob_u50": {"HB_VARLEN_KERNEL": "50"}}' timeout 900 python tools/ab_varlen.py sha1 sm3 >> gpurun_out/ab_varlen_$T.txt 2>&1
for alg in sha1 sm3; do
for arm in "dflt:" "win:HB_VARLEN_SORT=window" "win47:HB_VARLEN_SORT=window HB_VARLEN_KERNEL=47" "glob47:HB_VARLEN_KERNEL=47" "win50:HB_VARLEN_SORT=window HB_VARLEN_KERNEL=50" "glob50:HB_VARLEN_KERNEL=50"; do
  name=${arm%%:*}; envs=${arm#*:}
  env $envs timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_varlen" -s 1 -c 1 --csv python tools/ncu_one.py $alg varlen > gpurun_out/ncu_${alg}_${name}_$T.csv 2>&1
done; done
head -c 500 gpurun_out/bench_varlen_md5_$T.json; echo; cat gpurun_out/ab_varlen_$T.txt
for f in gpurun_out/ncu_*_$T.csv; do echo "== $f"; grep -E "dram__bytes|gpu__time" $f | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'; done
