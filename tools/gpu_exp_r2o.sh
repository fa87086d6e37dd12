# Round-2 (o): late griddepcontrol.wait for HB_FLAG_INPUT_READY launches --
# GPU tests, sanitizers, and the bench line with HB_LATE_WAIT=1 (default) / 0.
mkdir -p gpurun_out
T=r2ak
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$T.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}_$T.log
done
HB_LATE_WAIT=0 timeout 1500 python bench.py --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_late0_$T.json 2> gpurun_out/bench_late0_$T.err
timeout 1500 python bench.py --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_late1_$T.json 2> gpurun_out/bench_late1_$T.err
HB_LATE_WAIT=0 timeout 1500 python bench.py --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_late0b_$T.json 2> gpurun_out/bench_late0b_$T.err
timeout 1500 python bench.py --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_late1b_$T.json 2> gpurun_out/bench_late1b_$T.err
tail -n 2 gpurun_out/pytest_gpu_$T.log; tail -n 3 gpurun_out/sanitize_*_$T.log
for f in gpurun_out/bench_late*_$T.err; do echo "== $f"; grep -E "headline|C1_sha1_64:|C5_md5_1024x65536:|C5_md5_16x65536:|C5_sha1_1024x65536:|C5_sm3_1024x65536:|C5_md5_65536x4096:" $f | cut -c1-110; done
