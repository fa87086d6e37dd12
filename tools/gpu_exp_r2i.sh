# Round-2 (i): per-block varlen cost against message length; ncu of the new
# varlen defaults (C4 MD5 / SM3) folded into profiles/ncu_summary.json; the
# varlen_md5 workload alone.
mkdir -p gpurun_out
T=r2u
timeout 600 python tools/varlen_scan.py md5 > gpurun_out/varlen_scan_$T.txt 2>&1
timeout 600 python tools/varlen_scan.py sm3 1023 16383 >> gpurun_out/varlen_scan_$T.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fixed|k_varlen|k_generic|k_decimal" \
  -o /tmp/ncu_cfg_$T python tools/ncu_configs.py run gpurun_out/ncu_cfg_${T}_order.json C4_varlen_md5 C4_varlen_sm3 > gpurun_out/ncu_cfg_$T.log 2>&1
ncu -i /tmp/ncu_cfg_$T.ncu-rep --page raw --csv > gpurun_out/ncu_cfg_${T}_raw.csv 2>/dev/null
ncu -i /tmp/ncu_cfg_$T.ncu-rep --page source --csv > gpurun_out/ncu_cfg_${T}_source.csv 2>/dev/null
timeout 600 python bench.py --workload varlen_md5 --steps 20 --warmup 5 --configs none --no-cpu > gpurun_out/bench_varlen_md5_$T.json 2> gpurun_out/bench_varlen_md5_$T.err
cat gpurun_out/varlen_scan_$T.txt; tail -n 2 gpurun_out/ncu_cfg_$T.log; head -c 400 gpurun_out/bench_varlen_md5_$T.json
