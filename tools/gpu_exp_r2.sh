# Round-2 A/B batch (run under gpurun from the repo root).
mkdir -p gpurun_out
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=5 AB_ARMS='{"dflt": {}, "v16": {"HB_VARLEN_KERNEL": "20"}, "w32": {"HB_VARLEN_LD": "32", "HB_SORT_QMAJOR": "0"}, "w32_qm": {"HB_VARLEN_LD": "32"}, "w32pf_qm": {"HB_VARLEN_LD": "32", "HB_VARLEN_PREFETCH": "1"}, "w32pf_qm16k": {"HB_VARLEN_LD": "32", "HB_VARLEN_PREFETCH": "1", "HB_SORT_WINDOW": "16384"}, "pf_qm16k": {"HB_VARLEN_KERNEL": "21", "HB_SORT_WINDOW": "16384"}}' timeout 900 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2e.txt 2>&1
unset HETOC_B200_LIB
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err
cat gpurun_out/ab_varlen_r2e.txt
tail -n 2 gpurun_out/bench_r2e.err
