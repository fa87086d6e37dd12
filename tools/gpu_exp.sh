set -u
mkdir -p gpurun_out
T=${T:-exp38}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -k "varlen_every" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$T.log
AB_ROUNDS=7 timeout 900 python tools/ab_varlen.py md5 sha1 > gpurun_out/ab_varlen_$T.txt 2>&1; echo "abv rc=$?"; grep -E '"default"|prefetch' gpurun_out/ab_varlen_$T.txt
