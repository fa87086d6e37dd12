set -u
mkdir -p gpurun_out
T=${T:-exp52}
{ timeout 300 ./tools/gather4_probe 32 4194304 8192; timeout 300 ./tools/gather4_probe 32 4194304 1; timeout 300 ./tools/gather4_probe 8 4194304 8192; } 2>&1 | tee gpurun_out/gather4_$T.txt
