set -u
mkdir -p gpurun_out
T=${T:-exp20}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -k "tile_configs" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
SWEEP_CFGS=ws3 SWEEP_VARS=0123 SWEEP_STEPS=50 SWEEP_ROUNDS=3 timeout 900 python tools/variant_sweep.py md5 > gpurun_out/variant_$T.txt 2>&1; echo "sweep rc=$?"; cat gpurun_out/variant_$T.txt
