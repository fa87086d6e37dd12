# Round-2 (e): new MD5 defaults (single-warp NB=2 tiles with variant 4 from 2^16
# messages, variant 6 in the 4+1-warp tile below; lean varlen loop) -- GPU
# tests on both libraries, A/B against the previous defaults, L2-policy varlen
# arms, and the default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/smi_r2p.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_r2p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r2p.log
HETOC_B200_LIB=libhetoc_b200_ab.so timeout 1200 python -m pytest tests -q -m "gpu and ab" > gpurun_out/pytest_ab_r2p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab_r2p.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2p.log 2>&1
export HETOC_B200_LIB=libhetoc_b200_ab.so
AB_ROUNDS=4 AB_ARMS='{"dflt": {}, "old": {"HB_VARLEN_KERNEL": "21"}, "l47hint": {"HB_VARLEN_KERNEL": "47"}, "l46": {"HB_VARLEN_KERNEL": "46"}}' timeout 900 python tools/ab_varlen.py md5 > gpurun_out/ab_varlen_r2p.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"dflt": {}, "old": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}, "oldv3": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "3"}, "w1x2p_v6": {"HB_TMA_CFG": "w1x2p", "HB_VARIANT": "6"}, "w1x2_nopdl": {"HB_TMA_CFG": "w1x2", "HB_VARIANT": "4"}}' AB_POINTS='md5:65536:1024,md5:65536:256,md5:49152:1024,md5:65536:16384,md5:262144:1024,md5:1048576:1024,md5:4194304:1024,md5:16384:1024,md5:4736:65536' timeout 900 python tools/ab_mid.py > gpurun_out/ab_mid_r2p.txt 2>&1
AB_ROUNDS=4 AB_STEPS=8 AB_ARMS='{"dflt": {}, "old": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}}' timeout 600 python tools/ab_power.py md5 > gpurun_out/ab_c2short_r2p.txt 2>&1
AB_ROUNDS=2 AB_STEPS=60 AB_ARMS='{"dflt": {}, "old": {"HB_TMA_CFG": "ws3", "HB_VARIANT": "1"}}' timeout 600 python tools/ab_power.py md5 > gpurun_out/ab_c2long_r2p.txt 2>&1
unset HETOC_B200_LIB
SECONDS=0; timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2p.json 2> gpurun_out/bench_r2p.err; echo "bench wall $SECONDS s" >> gpurun_out/bench_r2p.err
tail -n 2 gpurun_out/pytest_gpu_r2p.log gpurun_out/pytest_ab_r2p.log gpurun_out/smoke_r2p.log
cat gpurun_out/ab_varlen_r2p.txt gpurun_out/ab_mid_r2p.txt gpurun_out/ab_c2short_r2p.txt gpurun_out/ab_c2long_r2p.txt | cut -c1-180
tail -n 3 gpurun_out/bench_r2p.err
