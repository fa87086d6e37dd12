# GPU-box check used during round 2: GPU test suite (default library, then the
# A/B arms against the -DHB_AB library), smoke, default bench + reference arm.
# Usage (from the repo root, under gpurun): bash tools/gpu_check_r2.sh TAG [tests|bench|all]
TAG=${1:-r2}
WHAT=${2:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
free -g >> gpurun_out/smi_$TAG.txt; nproc >> gpurun_out/smi_$TAG.txt
if [ "$WHAT" = tests ] || [ "$WHAT" = all ]; then
  timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "default rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
  HETOC_B200_LIB=libhetoc_b200_ab.so timeout 900 python -m pytest tests -q -m "gpu and ab" > gpurun_out/pytest_ab_$TAG.log 2>&1; echo "ab rc=$?" >> gpurun_out/pytest_ab_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
fi
if [ "$WHAT" = bench ] || [ "$WHAT" = all ]; then
  SECONDS=0; timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
  echo "bench wall $SECONDS s" >> gpurun_out/bench_$TAG.err
  timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
fi
tail -n 3 gpurun_out/*_$TAG.log 2>/dev/null
tail -n 2 gpurun_out/bench_$TAG.err
