set -u
mkdir -p gpurun_out
T=${T:-exp23}
timeout 600 python -m pytest tests -q -m gpu --timeout 300 -k "tile_configs and ws3n" > gpurun_out/pytest_$T.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -3 gpurun_out/pytest_$T.log
if [ $rc = 0 ]; then
SWEEP_CFGS=ws3,ws3n SWEEP_VARS=1 SWEEP_STEPS=50 SWEEP_ROUNDS=3 timeout 900 python tools/variant_sweep.py md5 sha1 > gpurun_out/variant_$T.txt 2>&1; echo "sweep rc=$?"; cat gpurun_out/variant_$T.txt
SWEEP_CFGS=ws3,ws3n SWEEP_VARS=1 SWEEP_STEPS=10 SWEEP_ROUNDS=3 timeout 900 python tools/variant_sweep.py md5 > gpurun_out/variant10_$T.txt 2>&1; echo "sweep10 rc=$?"; cat gpurun_out/variant10_$T.txt
fi
