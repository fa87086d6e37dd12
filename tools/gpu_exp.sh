set -u
mkdir -p gpurun_out
T=${T:-exp39}
timeout 1800 python tools/bench_configs.py gpurun_out/sweep_$T.jsonl --sweep-only > /dev/null 2> gpurun_out/sweep_$T.err; echo "sweep rc=$?"; wc -l gpurun_out/sweep_$T.jsonl; grep -c '"bit_exact_sample": true' gpurun_out/sweep_$T.jsonl
