set -u
mkdir -p gpurun_out
T=${T:-exp55}
AB_CASES=small AB_ARMS=1,2@0.5,2@1,4@0.5,4@1,8@0.25 timeout 900 python tools/ab_pipe.py 2>&1 | tee gpurun_out/ab_pipe_$T.txt
