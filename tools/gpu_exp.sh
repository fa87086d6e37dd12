set -u
mkdir -p gpurun_out
T=${T:-exp17}
timeout 600 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_$T.txt 2>&1; echo "abv rc=$?"; cat gpurun_out/ab_varlen_$T.txt
