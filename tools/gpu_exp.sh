set -u
mkdir -p gpurun_out
T=${T:-exp62}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "numa or bind or sharding or uneven or concurrent or engine" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$T.log
python - <<'PY'
import subprocess
bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
print("nvidia-smi bus id", bus)
import glob
for p in glob.glob("/sys/bus/pci/devices/*/local_cpulist")[:0]: pass
b = bus.lower()
if b.startswith("00000000:"): b = b[4:]
try:
    print("local_cpulist", open(f"/sys/bus/pci/devices/{b}/local_cpulist").read().strip())
except Exception as e:
    print("sysfs", e)
PY
