set -u
mkdir -p gpurun_out
T=${T:-exp36}
timeout 900 python tools/runtime_bench.py sha1 20000000 > gpurun_out/runtime_bench_$T.txt 2>&1; echo "rc=$?"; cat gpurun_out/runtime_bench_$T.txt | tail -5
