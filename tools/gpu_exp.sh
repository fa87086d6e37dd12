set -u
mkdir -p gpurun_out
T=${T:-exp60}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multiproc.py -x -q -m gpu -k "bind or multirank or p2p" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
python -c "import sys; sys.path.insert(0,'.'); from paper_2407_09333_b200.device import bind_host_to_gpu; print(bind_host_to_gpu(0))"
HB_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 2 --workload sha1_64 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'].get('host_affinity'), d['n_gpus'], d['value'])"
