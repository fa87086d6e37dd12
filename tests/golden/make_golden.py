"""Generate the golden fixtures in this directory by running the REFERENCE itself.

Run in the authoring container, where the read-only reference lives at
/root/reference:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The outputs (``*.json``) are committed; nothing at test time reads
/root/reference.  Message bytes for the batch fixtures come from the
counter-based generator in ``oracle.fill_random`` (identical to the engine's
``hb_fill_random_dev``); each fixture also stores a SHA-256 of its input bytes
so the generator itself is pinned.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

import oracle  # noqa: E402  (only for the shared synthetic-byte generator)
from hetoc.crypto import batch_digest, digest, gen_messages, hash_batch  # noqa: E402
from hetoc.passes.partition import partition_range  # noqa: E402

ALGS = ("sha1", "md5", "sm3")


def kats():
    # SPEC.md:255-257, SPEC.md:266 plus the standard FIPS 180 / RFC 1321 / GB/T 32905 vectors
    msgs = [b"", b"abc", b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq",
            b"message digest", b"abcd" * 16, b"a" * 1000]
    out = []
    for alg in ALGS:
        for m in msgs:
            out.append({"alg": alg, "msg_hex": m.hex(), "digest": digest(alg, m).hex()})
    return out


BOUNDARY = [0, 1, 3, 4, 9, 15, 16, 17, 31, 32, 55, 56, 57, 63, 64, 65, 119, 120, 121, 127,
            128, 129, 191, 255, 256, 1000, 1024, 4096]


def boundary():
    rng = np.random.default_rng(20240709)
    out = []
    for L in BOUNDARY:
        m = rng.integers(0, 256, L, dtype=np.uint8).tobytes()
        row = {"len": L, "msg_hex": m.hex()}
        for alg in ALGS:
            row[alg] = digest(alg, m).hex()  # scalar reference (batch.py:102-109)
        out.append(row)
    return out


FIXED = [(5, 0), (1, 64), (8, 9), (33, 16), (65, 55), (40, 56), (40, 63), (129, 64), (31, 100),
         (17, 128), (12, 1000), (257, 1024), (3, 4096)]


def fixed_batches():
    out = []
    for k, (n, L) in enumerate(FIXED):
        seed = 1000 + k
        data = oracle.fill_random(n * L, seed).reshape(n, L)
        row = {"n": n, "msg_len": L, "seed": seed,
               "input_sha256": hashlib.sha256(data.tobytes()).hexdigest()}
        for alg in ALGS:
            ref = batch_digest(alg, data)  # the reference vectorized path, batch.py:274-290
            row[alg] = hashlib.sha256(ref.tobytes()).hexdigest()
            row[alg + "_first"] = ref[0].tobytes().hex()
            row[alg + "_last"] = ref[-1].tobytes().hex()
        out.append(row)
    return out


def varlen_batches():
    out = []
    rng = np.random.default_rng(7)
    for k, (n, maxlen) in enumerate([(50, 200), (40, 1100), (9, 70)]):
        lens = rng.integers(0, maxlen + 1, n)
        offsets = np.zeros(n + 1, np.uint64)
        offsets[1:] = np.cumsum(lens)
        seed = 2000 + k
        data = oracle.fill_random(int(offsets[-1]), seed)
        row = {"seed": seed, "lens": [int(x) for x in lens],
               "input_sha256": hashlib.sha256(data.tobytes()).hexdigest()}
        for alg in ALGS:
            digs = [digest(alg, data[int(offsets[i]):int(offsets[i + 1])].tobytes()).data
                    for i in range(n)]
            row[alg] = hashlib.sha256(b"".join(digs)).hexdigest()
        out.append(row)
    return out


def decimal_batches():
    out = []
    for start, count in [(0, 1000), (123456789, 3), (999999000, 1000)]:
        b = gen_messages(start, count)
        row = {"start": start, "count": count, "width": 9,
               "input_sha256": hashlib.sha256(b.data).hexdigest()}
        for alg in ALGS:
            digs = hash_batch(alg, b, threads=1)  # batch.py:293-316
            row[alg] = hashlib.sha256(b"".join(d.data for d in digs)).hexdigest()
        out.append(row)
    return out


def partitions():
    rnd = random.Random(5)
    cases = [(0, 10, [0.5, 0.5]), (0, 1000, [0.3, 0.7]), (0, 7, [0.33, 0.33, 0.34]),
             (0, 1 << 24, [0.25] * 4), (0, 1 << 24, [0.125] * 8), (0, 1 << 24, [1 / 3] * 3)]
    for _ in range(200):
        k = rnd.randint(1, 8)
        w = [rnd.random() for _ in range(k)]
        s = sum(w)
        lb = rnd.randint(0, 1000)
        cases.append((lb, lb + rnd.randint(0, 1 << 26), [x / s for x in w]))
    for k in (1, 2, 3, 4, 5, 6, 7, 8):
        for n in (0, 1, 7, 65536, 1 << 22, (1 << 24) + 3):
            cases.append((0, n, [1.0 / k] * k))
    return [{"lb": lb, "ub": ub, "ratios": r, "ranges": partition_range(lb, ub, r)} for lb, ub, r in cases]


def scheduler_models():
    """The reference's calibration (hetoc.scheduler.model.fit_model) and its
    predictions on deterministic sample sets, incl. ones that clamp."""
    from hetoc.scheduler.model import PerfModel, fit_model, predict_opt_ratio, t_opt

    rnd = random.Random(11)
    cases = []
    sets = [([(1000, 0.01), (2000, 0.021), (4000, 0.039)], [(1000, 0.002), (2000, 0.0031), (8000, 0.0105)], 8),
            ([(10, 1.0), (20, 2.0)], [(10, 5.0), (20, 1.0)], 1),  # negative device slope -> clamped
            ([(100, 1.0), (300, 2.9)], [(100, 0.1), (300, 0.5)], 16)]  # negative intercept -> clamped
    for _ in range(20):
        k = rnd.randint(2, 6)
        cpu = [(rnd.randint(1, 10**7), rnd.uniform(0.001, 50.0)) for _ in range(k)]
        dev = [(rnd.randint(1, 10**7), rnd.uniform(0.0001, 5.0)) for _ in range(rnd.randint(2, 6))]
        sets.append((cpu, dev, rnd.randint(1, 256)))
    for cpu, dev, cores in sets:
        m = fit_model(cpu, dev, cores)
        row = {"cpu": cpu, "dev": dev, "n_core": cores,
               "model": {k: getattr(m, k) for k in ("p_cpu", "n_core", "p_gpu_over_nthread", "t_alloc",
                                                     "t_memcpy", "o_gpu")}}
        try:
            row["opt_ratio"] = {str(n): predict_opt_ratio(m, n) for n in (1, 1000, 10**6, 10**9)}
        except ValueError:
            row["opt_ratio"] = None
        row["t_opt"] = {f"{n}:{x}": t_opt(m, n, x) for n in (1000, 10**6) for x in (0.0, 0.1, 0.5, 1.0)}
        cases.append(row)
    extra = PerfModel(p_cpu=2e-6, n_core=12, p_gpu_over_nthread=1e-8, t_alloc=2e-9, t_memcpy=3e-8, o_gpu=1e-3)
    cases.append({"model": {k: getattr(extra, k) for k in ("p_cpu", "n_core", "p_gpu_over_nthread", "t_alloc",
                                                           "t_memcpy", "o_gpu")},
                  "opt_ratio": {str(n): predict_opt_ratio(extra, n) for n in (1, 1000, 10**6, 10**9)},
                  "t_opt": {f"{n}:{x}": t_opt(extra, n, x) for n in (1000, 10**6) for x in (0.0, 0.1, 0.5, 1.0)}})
    return cases


def main():
    fixtures = {
        "kats.json": kats,
        "boundary.json": boundary,
        "fixed_batches.json": fixed_batches,
        "varlen_batches.json": varlen_batches,
        "decimal_batches.json": decimal_batches,
        "partition.json": partitions,
        "scheduler_model.json": scheduler_models,
    }
    only = sys.argv[1:]
    for name, obj in fixtures.items():
        if only and name not in only:
            continue
        obj = obj() if callable(obj) else obj
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(obj, f, indent=0 if name != "partition.json" else None)
            f.write("\n")
        print(name, len(obj))


if __name__ == "__main__":
    main()
