set -u
mkdir -p gpurun_out
T=${T:-exp44}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_decimal" -s 3 -c 1 \
    -o /tmp/prof_dec_$T python bench.py --workload paper_md5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_dec_$T.txt 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_dec_$T.ncu-rep --page raw --csv > gpurun_out/raw_dec_$T.csv 2>/dev/null
ncu -i /tmp/prof_dec_$T.ncu-rep --page source --csv > gpurun_out/source_dec_$T.csv 2>/dev/null
ncu -i /tmp/prof_dec_$T.ncu-rep --page details > gpurun_out/details_dec_$T.txt 2>/dev/null
ls -la gpurun_out/*dec_$T*
