set -u
mkdir -p gpurun_out/multirank
D=gpurun_out/multirank
run2() { HB_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 "${@:2}" 2>/dev/null | grep '^{' | tail -1; }
run2 29541 --steps 20 --warmup 3 > $D/bench2_none_final.json; echo "none rc=$?"
run2 29542 --steps 20 --warmup 3 --gather p2p > $D/bench2_p2p_final.json; echo "p2p rc=$?"
run2 29543 --steps 10 --warmup 3 --workload sm3_1k > $D/bench2_sm3_final.json; echo "sm3 rc=$?"
run2 29544 --steps 3 --warmup 3 --impl reference > $D/bench2_ref_final.json; echo "ref rc=$?"
for f in $D/*_final.json; do python -c "import json,sys; d=json.loads(open(sys.argv[1]).read()); print(sys.argv[1].split('/')[-1], d.get('impl','ours'), d['n_gpus'], d['value'], d.get('scaling'), d['config'].get('host_affinity'), d['config'].get('gather'), (d.get('e2e') or {}).get('matches_device_run'))" $f; done
