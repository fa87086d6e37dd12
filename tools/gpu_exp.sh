set -u
mkdir -p gpurun_out
T=${T:-exp22}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -k "varlen" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
timeout 600 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_$T.txt 2>&1; echo "abv rc=$?"; cat gpurun_out/ab_varlen_$T.txt
