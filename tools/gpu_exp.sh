set -u
mkdir -p gpurun_out
T=${T:-exp35}
timeout 900 python tools/e2e_pageable.py md5 4194304 1024 > gpurun_out/e2e_pageable_$T.txt 2>&1; echo "rc=$?"; cat gpurun_out/e2e_pageable_$T.txt
