set -u
mkdir -p gpurun_out
T=${T:-exp27}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -k "varlen or multirank or p2p" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$T.log
timeout 600 python tools/ab_varlen.py > gpurun_out/ab_varlen_$T.txt 2>&1; echo "abv rc=$?"; grep -E '"default"|ld16_global' gpurun_out/ab_varlen_$T.txt
timeout 900 compute-sanitizer --tool initcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_initcheck_$T.log 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/sanitize_initcheck_$T.log
grep "Device Frame" gpurun_out/sanitize_initcheck_$T.log | sed -E 's/\+0x[0-9a-f]+//' | sort | uniq -c
