SCAN='md5:1024,sha1:1024,sm3:1024,md5:256,sha1:64' timeout 900 python tools/ab_scan.py > gpurun_out/scan_r2a.txt 2>&1
K='regex:k_fixed|k_varlen'
for spec in "md5 65536 1024" "sha1 65536 64" "md5 varlen"; do
  tag=$(echo $spec | tr ' ' '_')
  timeout 600 ncu --set full --import-source on --clock-control none -k "$K" -s 1 -c 1 -o gpurun_out/prof_$tag python tools/ncu_one.py $spec > gpurun_out/ncu_$tag.log 2>&1
  ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>/dev/null
  ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv > gpurun_out/source_$tag.csv 2>/dev/null
done
cat gpurun_out/scan_r2a.txt
