# Round-2 (p): early-release threshold for INPUT_READY launches with the late
# wait: half (default) vs a full wave of resident CTAs, through the bench.
mkdir -p gpurun_out
T=r2al
timeout 900 python -m pytest tests -q -m gpu -k "input_ready or pdl or geometry or last_kernel" > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$T.log
for k in a b; do
HB_TRIGGER_WAVE_PCT=50 timeout 1500 python bench.py --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_w50${k}_$T.json 2> gpurun_out/bench_w50${k}_$T.err
HB_TRIGGER_WAVE_PCT=100 timeout 1500 python bench.py --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_w100${k}_$T.json 2> gpurun_out/bench_w100${k}_$T.err
done
tail -n 2 gpurun_out/pytest_gpu_$T.log
python - <<'PY'
import json
keys=None
for f in ['w50a','w100a','w50b','w100b']:
    d=json.loads(open(f'gpurun_out/bench_{f}_r2al.json').read().strip().splitlines()[-1])
    c=d['configs']
    keys=keys or [k for k in c if 'max_bound' in c[k].get('roofline',{})]
    print(f, round(d['roofline']['frac'],3), ' '.join(f"{k.replace('C5_','')}={c[k]['roofline']['max_bound']['frac']:.3f}" for k in keys))
PY
