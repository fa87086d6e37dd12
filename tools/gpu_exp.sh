set -u
mkdir -p gpurun_out
T=${T:-exp45}
AB_ARMS=default,minb12,minb16 AB_ROUNDS=5 timeout 900 python tools/ab_varlen.py md5 sha1 sm3 > gpurun_out/ab_varlen_$T.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_varlen_$T.txt
