set -u
mkdir -p gpurun_out
T=${T:-exp15}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -k "tile_configs or geometry" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
SWEEP_CFGS=ws3,ws3u,ws3x2,ws3x2u SWEEP_VARS=1 SWEEP_ROUNDS=4 timeout 900 python tools/variant_sweep.py md5 sha1 sm3 > gpurun_out/variant_$T.txt 2>&1; echo "sweep rc=$?"; cat gpurun_out/variant_$T.txt
