set -u
mkdir -p gpurun_out
T=${T:-exp26}
export HB_BENCH_BACKEND=gloo
for g in none p2p; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --workload md5_1k --msgs 2097152 --steps 5 --warmup 3 --gather $g > gpurun_out/bench2_${g}_$T.json 2> gpurun_out/bench2_${g}_$T.err
  echo "bench2 $g rc=$?"; cut -c1-900 gpurun_out/bench2_${g}_$T.json; tail -3 gpurun_out/bench2_${g}_$T.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 2 --workload sm3_1k --msgs 1048576 --steps 3 --warmup 3 > gpurun_out/bench2_sm3_$T.json 2> gpurun_out/bench2_sm3_$T.err
echo "bench2 sm3 rc=$?"; cut -c1-600 gpurun_out/bench2_sm3_$T.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/bench2_ref_$T.json 2> gpurun_out/bench2_ref_$T.err
echo "bench2 ref rc=$?"; cut -c1-300 gpurun_out/bench2_ref_$T.json
