# Round-2 (k): single-warp MD5 tile shapes -- 2 stages (more CTAs per SM) and
# 3 messages per thread -- against the shipped 3-stage two-message tile.
mkdir -p gpurun_out
export HETOC_B200_LIB=libhetoc_b200_ab.so
timeout 600 python -m pytest tests -q -m "gpu and ab" -k tile_configs > gpurun_out/pytest_ab_r2y.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab_r2y.log
AB_ROUNDS=4 AB_COOL=3 AB_ARMS='{"dflt": {}, "s2": {"HB_TMA_CFG": "w1x2s2"}, "nb3": {"HB_TMA_CFG": "w1x3"}}' timeout 900 python tools/ab_headline.py md5 > gpurun_out/ab_headline_r2y.txt 2>&1
AB_ROUNDS=3 AB_ARMS='{"dflt": {}, "s2": {"HB_TMA_CFG": "w1x2s2"}, "nb3": {"HB_TMA_CFG": "w1x3"}}' AB_POINTS='md5:65536:1024,md5:65536:16384,md5:262144:1024,md5:1048576:1024,md5:4194304:1024,md5:98304:1024' timeout 900 python tools/ab_mid.py > gpurun_out/ab_mid_r2y.txt 2>&1
tail -n 2 gpurun_out/pytest_ab_r2y.log; cut -c1-230 gpurun_out/ab_headline_r2y.txt gpurun_out/ab_mid_r2y.txt
