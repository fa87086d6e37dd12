# Round-2 (g): ncu evidence for the new MD5 defaults -- one --set full capture
# per BASELINE config (folded into profiles/ncu_summary.json here), source-level
# stall captures of the single-warp MD5 tile and the lean varlen loop, the
# varlen L2-policy arm's DRAM bytes, and the launch list of the default bench.
mkdir -p gpurun_out
T=${1:-r2r}
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:"k_fixed|k_varlen|k_generic|k_decimal" \
  -o /tmp/ncu_cfg_$T python tools/ncu_configs.py run gpurun_out/ncu_cfg_${T}_order.json > gpurun_out/ncu_cfg_$T.log 2>&1
ncu -i /tmp/ncu_cfg_$T.ncu-rep --page raw --csv > gpurun_out/ncu_cfg_${T}_raw.csv 2>/dev/null
for spec in "md5 1048576 1024" "md5 65536 1024" "md5 varlen"; do
  tag=$(echo $spec | tr ' ' '_')
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_fixed|k_varlen" -s 1 -c 1 \
    -o /tmp/ncu_${tag}_$T python tools/ncu_one.py $spec > gpurun_out/ncu_${tag}_$T.log 2>&1
  ncu -i /tmp/ncu_${tag}_$T.ncu-rep --page raw --csv > gpurun_out/raw_${tag}_$T.csv 2>/dev/null
  ncu -i /tmp/ncu_${tag}_$T.ncu-rep --page source --csv > gpurun_out/source_${tag}_$T.csv 2>/dev/null
done
HETOC_B200_LIB=libhetoc_b200_ab.so HB_VARLEN_KERNEL=47 timeout 600 ncu --set full --clock-control none -k regex:"k_varlen" \
  -s 1 -c 1 -o /tmp/ncu_vl47_$T python tools/ncu_one.py md5 varlen > gpurun_out/ncu_vl47_$T.log 2>&1
ncu -i /tmp/ncu_vl47_$T.ncu-rep --page raw --csv > gpurun_out/raw_vl47_$T.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$T.csv \
  python bench.py --steps 5 --warmup 3 --configs none > gpurun_out/ncu_bench_stdout_$T.txt 2>&1
cp /tmp/ncu_md5_1048576_1024_$T.ncu-rep gpurun_out/ 2>/dev/null
tail -n 3 gpurun_out/ncu_cfg_$T.log; du -sh gpurun_out
