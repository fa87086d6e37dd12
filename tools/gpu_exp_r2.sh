# Round-2 A/B batch (run under gpurun from the repo root).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r2d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r2d.log
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=3 AB_ARMS='{"base": {}, "ready": {"HB_INPUT_READY": "1"}}' AB_POINTS='sha1:65536:64,md5:65536:64,sm3:65536:64,md5:65536:16,sha1:65536:128,md5:65536:256,md5:65536:1024,sha1:65536:256,sha1:65536:1024,sm3:65536:256,sm3:65536:1024,md5:1048576:64,md5:262144:1024,md5:4096:4096,sha1:4096:4096' timeout 1500 python tools/ab_mid.py > gpurun_out/ab_ready_r2d.txt 2>&1
AB_ROUNDS=2 AB_ARMS='{"base": {}, "v1": {"HB_CHAIN_N": "0"}, "v0": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "0"}, "v2": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "2"}, "v3": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "3"}}' AB_POINTS='md5:4736:65536,sha1:4736:65536,sm3:4736:65536,md5:4736:4096' timeout 900 python tools/ab_mid.py > gpurun_out/ab_chain_r2d.txt 2>&1
unset HETOC_B200_LIB
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err
tail -n 3 gpurun_out/pytest_gpu_r2d.log
cat gpurun_out/ab_ready_r2d.txt gpurun_out/ab_chain_r2d.txt
tail -n 2 gpurun_out/bench_r2d.err
