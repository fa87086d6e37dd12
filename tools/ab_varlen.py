"""A/B of the varlen kernels on configs[3] (2^22 messages, uniform 1-4096 B),
interleaved rounds, digests cross-checked.  One JSON line per arm.
Arms: $AB_ARMS (JSON {name: {env}}), default per-thread kernel vs prefetch;
run against the A/B library (HETOC_B200_LIB=libhetoc_b200_ab.so)."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09333_b200 import _native, device  # noqa: E402

DLEN = {"md5": 16, "sha1": 20, "sm3": 32}
n, maxlen = 1 << 22, 4096
lens = np.random.default_rng(4).integers(1, maxlen + 1, n).astype(np.int64)
off = np.zeros(n + 1, np.int64)
off[1:] = np.cumsum(lens)
data = torch.empty(int(off[-1]), dtype=torch.uint8, device="cuda:0")
device.fill_random(data, 4)
d_off = torch.from_numpy(off).cuda()
scratch = torch.empty(int(_native.lib().hb_varlen_scratch_bytes(n)), dtype=torch.uint8, device="cuda:0")
C = _native.HB_FLAG_VARLEN_COOP
P = _native.HB_FLAG_VARLEN_COOP_OFF
ARMS = {k: (v, 0) for k, v in json.loads(os.environ.get("AB_ARMS", '{"default": {}, "prefetch": {"HB_VARLEN_PREFETCH": "1"}}')).items()}
KEYS = sorted({k for env, _ in ARMS.values() for k in env} | {"HB_VC_STAGES", "HB_VC_PF", "HB_VARLEN_SORT",
                                                          "HB_SORT_WINDOW", "HB_VARLEN_PREFETCH", "HB_VARLEN_BULK",
                                                          "HB_VARLEN_LD", "HB_VARLEN_Q"})
for alg in sys.argv[1:] or ["md5", "sha1", "sm3"]:
    ref, times = None, {}
    for _ in range(int(os.environ.get("AB_ROUNDS", 3))):
        for arm, (env, flags) in ARMS.items():
            for k in KEYS:
                os.environ.pop(k, None)
            os.environ.update(env)
            _native.reload_tuning()
            if float(os.environ.get("AB_COOL", 0)) > 0:  # idle first: every arm starts from the same power state
                torch.cuda.synchronize()
                time.sleep(float(os.environ["AB_COOL"]))
            out = torch.empty((n, DLEN[alg]), dtype=torch.uint8, device="cuda:0")
            f = lambda: device.hash_varlen(alg, data, d_off, out=out, scratch=scratch, flags=flags,  # noqa: E731
                                           offset_base=0)
            f()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(5):
                f()
            e.record()
            torch.cuda.synchronize()
            if ref is None:
                ref = out.clone()
            assert torch.equal(out, ref), (alg, arm)
            times.setdefault(arm, []).append(s.elapsed_time(e) / 5)
    for arm, ts in times.items():
        ms = statistics.median(ts)
        alg_bytes = int(off[-1]) + 8 * (n + 1) + n * DLEN[alg]
        print(json.dumps({"alg": alg, "arm": arm, "ms": round(ms, 4), "ms_min": round(min(ts), 4),
                          "GBps": round(int(off[-1]) / ms / 1e6, 1),
                          "frac_of_6459": round(alg_bytes / ms / 1e6 / 6459.3, 4)}), flush=True)
