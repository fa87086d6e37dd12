"""CPU oracle for the batched-hash hot path -- TEST INFRASTRUCTURE ONLY.

This package restates the reference algorithm (``hetoc.crypto``, see
``hetoc_oracle.c`` for the file:line of every function) in plain C so that
tests, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg can check
and time the B200 engine.  The product package ``paper_2407_09333_b200`` never
imports it.

Pinning: ``tests/test_oracle.py`` checks this oracle against
``tests/golden/*.json``, which ``tests/golden/make_golden.py`` produced by
running the reference package itself (``/root/reference/pkg/src``), and
against the KATs of SPEC.md:255-257 / SPEC.md:266.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
ALG_ID = {"sha1": 0, "md5": 1, "sm3": 2}
DIGEST_LEN = {"sha1": 20, "md5": 16, "sm3": 32}

_lib = None


def build() -> str:
    """Compile liboracle.so in place (gcc via the committed Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        L.orc_digest.argtypes = [ctypes.c_int, u8p, ctypes.c_uint64, u8p]
        L.orc_batch_fixed.argtypes = [ctypes.c_int, u8p, ctypes.c_uint64, ctypes.c_uint64, u8p, ctypes.c_int]
        L.orc_batch_varlen.argtypes = [ctypes.c_int, u8p, u64p, ctypes.c_uint64, u8p, ctypes.c_int]
        L.orc_fill_random.argtypes = [u8p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        L.orc_fill_random.restype = None
        L.orc_gen_decimal.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, u8p]
        _lib = L
    return _lib


def _u8(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def digest(alg: str, msg: bytes) -> bytes:
    out = np.empty(DIGEST_LEN[alg], np.uint8)
    buf = np.frombuffer(bytes(msg) + b"\0", np.uint8)  # never a NULL pointer
    rc = lib().orc_digest(ALG_ID[alg], _u8(buf), len(msg), _u8(out))
    assert rc == 0
    return out.tobytes()


def batch_fixed(alg: str, data: np.ndarray, threads: int = 1) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.uint8)
    n, L = data.shape
    out = np.empty((n, DIGEST_LEN[alg]), np.uint8)
    if n:
        src = data if data.size else np.zeros(1, np.uint8)
        rc = lib().orc_batch_fixed(ALG_ID[alg], _u8(src), n, L, _u8(out), int(threads))
        assert rc == 0, rc
    return out


def batch_varlen(alg: str, data: np.ndarray, offsets: np.ndarray, threads: int = 1) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = offsets.shape[0] - 1
    out = np.empty((n, DIGEST_LEN[alg]), np.uint8)
    if n > 0:
        src = data if data.size else np.zeros(1, np.uint8)
        rc = lib().orc_batch_varlen(
            ALG_ID[alg], _u8(src), offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n, _u8(out), int(threads)
        )
        assert rc == 0, rc
    return out


def fill_random(nbytes: int, seed: int, byte_offset: int = 0) -> np.ndarray:
    """Same bytes as hb_fill_random_dev(seed, byte_offset) writes on the GPU."""
    assert byte_offset % 8 == 0
    out = np.empty(nbytes, np.uint8)
    if nbytes:
        lib().orc_fill_random(_u8(out), nbytes, seed, byte_offset)
    return out


def gen_decimal(start: int, count: int, width: int = 9) -> np.ndarray:
    out = np.empty((count, width), np.uint8)
    if count:
        assert lib().orc_gen_decimal(start, count, width, _u8(out)) == 0
    return out


def round_half_up(x: float) -> int:
    """pkg/src/hetoc/passes/partition.py:13-14."""
    import math

    return math.floor(x + 0.5)


def partition_range(lb: int, ub: int, ratios: list[float]) -> list[tuple[int, int]]:
    """Restatement of pkg/src/hetoc/passes/partition.py:17-31 (cumulative
    round-half-up split, last endpoint forced to ub)."""
    if lb > ub:
        raise ValueError("inverted range")
    if not ratios:
        raise ValueError("need at least one ratio")
    n = ub - lb
    bounds = [lb]
    cum = 0.0
    for r in ratios[:-1]:
        cum += r
        b = lb + round_half_up(n * cum)
        bounds.append(min(max(b, bounds[-1]), ub))
    bounds.append(ub)
    return list(zip(bounds, bounds[1:]))
