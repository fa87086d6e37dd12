"""CPU checks of bench.py's launch contract: `--gpus N` is authoritative --
without WORLD_SIZE it relaunches itself under torch.distributed.run with N
ranks (gloo test hook: ranks may share GPUs / run without one), and it refuses
to run N ranks on fewer than N visible GPUs."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=300, env=env, cwd=ROOT)


def test_gpus_2_spawns_two_ranks():
    r = _run(["--gpus", "2", "--dry-run"], {"HB_BENCH_BACKEND": "gloo"})
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert sorted(x["rank"] for x in line["ranks"]) == [0, 1]
    assert len({x["pid"] for x in line["ranks"]}) == 2


def test_gpus_more_than_visible_fails_loudly():
    try:
        import torch

        if torch.cuda.device_count() >= 3:
            pytest.skip("enough GPUs: the launch would proceed")
    except Exception:
        pass
    r = _run(["--gpus", "3"], {"HB_BENCH_BACKEND": "nccl"})
    assert r.returncode == 2
    assert "needs 3 visible CUDA devices" in r.stderr


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "4", "--dry-run"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr
