# N>1 regression of bench.py on the one-GPU box: two ranks sharing GPU 0
# through the gloo test hook (numbers are one GPU's; the path is what is checked).
mkdir -p gpurun_out
T=${1:-r2l}
export HB_BENCH_BACKEND=gloo
timeout 1500 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2_$T.json 2> gpurun_out/bench_n2_$T.err; echo "rc=$?" >> gpurun_out/bench_n2_$T.err
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --configs none --gather p2p > gpurun_out/bench_n2_p2p_$T.json 2> gpurun_out/bench_n2_p2p_$T.err; echo "rc=$?" >> gpurun_out/bench_n2_p2p_$T.err
timeout 600 python bench.py --gpus 2 --workload sm3_1k --steps 10 --warmup 3 > gpurun_out/bench_n2_sm3_$T.json 2> gpurun_out/bench_n2_sm3_$T.err; echo "rc=$?" >> gpurun_out/bench_n2_sm3_$T.err
timeout 600 python bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/bench_n2_ref_$T.json 2> gpurun_out/bench_n2_ref_$T.err; echo "rc=$?" >> gpurun_out/bench_n2_ref_$T.err
unset HB_BENCH_BACKEND
timeout 120 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_nccl_$T.json 2> gpurun_out/bench_n2_nccl_$T.err; echo "rc=$?" >> gpurun_out/bench_n2_nccl_$T.err
tail -n 3 gpurun_out/bench_n2_*_$T.err gpurun_out/bench_n2_$T.err
for f in gpurun_out/bench_n2_*$T.json gpurun_out/bench_n2_$T.json; do echo "== $f"; head -c 600 $f; echo; done
