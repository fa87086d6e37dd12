"""Host-side checker for the tools/ scripts: per-row digests from Python's
hashlib (OpenSSL's SHA-1 / MD5 / SM3 -- an implementation independent of both
the CUDA kernels and oracle/, which only tests/, smoke() and bench.py's CPU
legs use), random host bytes, and the paper's decimal messages."""
import hashlib

import numpy as np


def digests(alg, rows):
    """(n, dlen) uint8 digests of the rows of a 2-D uint8 array."""
    rows = np.ascontiguousarray(rows, dtype=np.uint8)
    return np.stack([np.frombuffer(hashlib.new(alg, r.tobytes()).digest(), np.uint8) for r in rows]) \
        if len(rows) else np.zeros((0, {"sha1": 20, "md5": 16, "sm3": 32}[alg]), np.uint8)


def digests_varlen(alg, data, offsets):
    data = np.asarray(data, np.uint8)
    off = [int(x) for x in offsets]
    return np.stack([np.frombuffer(hashlib.new(alg, data[off[i]:off[i + 1]].tobytes()).digest(), np.uint8)
                     for i in range(len(off) - 1)])


def random_bytes(nbytes, seed):
    return np.random.default_rng(seed).integers(0, 256, nbytes, dtype=np.uint8)


def decimal_messages(start, count, width):
    """gen_messages(start, count, width) (pkg/src/hetoc/crypto/batch.py:86-99) as a (count, width) array."""
    return np.frombuffer("".join(f"{v:0{width}d}"[-width:] for v in range(start, start + count)).encode(),
                         np.uint8).reshape(count, width)
