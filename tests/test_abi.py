"""The C-ABI library loads and exports every symbol include/hetoc_b200.h
declares, and its host-only logic (partition, digest lengths, argument
validation, error mapping) behaves like the reference.  No compute calls
that need a GPU (CPU suite)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2407_09333_b200 as hb
from paper_2407_09333_b200 import _native
from paper_2407_09333_b200.crypto import (
    ALGORITHMS,
    DIGEST_LEN,
    Digest,
    MessageBatch,
    UnknownAlgorithmError,
    batch_digest,
    batch_digest_varlen,
    digest,
    gen_messages,
    hash_batch,
)
from paper_2407_09333_b200.passes import partition_range

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hetoc_b200.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTS)


def test_library_is_sm100a():
    # the cubin inside the .so is sm_100a (checked without a GPU)
    import subprocess

    out = subprocess.run(["cuobjdump", "-lelf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_header_flags_match_python_constants():
    """Every HB_FLAG_* the header defines has the same value in _native."""
    flags = dict(re.findall(r"#define\s+(HB_FLAG_[A-Z0-9_]+)\s+(0x[0-9a-fA-F]+)u?", open(HEADER).read()))
    assert "HB_FLAG_INPUT_READY" in flags and len(flags) >= 7
    for name, val in flags.items():
        assert getattr(_native, name) == int(val, 16), name
    assert len(set(flags.values())) == len(flags)  # distinct bits


def test_abi_basics():
    lib = _native.lib()
    assert lib.hb_abi_version() == 3
    assert [lib.hb_digest_len(i) for i in range(3)] == [20, 16, 32]
    assert lib.hb_digest_len(7) == -1
    assert hb.launch_count() >= 0


def test_partition_matches_reference_golden(golden):
    for row in golden("partition.json"):
        assert [list(x) for x in partition_range(row["lb"], row["ub"], row["ratios"])] == row["ranges"]


def test_partition_spec_examples():
    # SPEC.md:188-190
    assert partition_range(0, 10, [0.5, 0.5]) == [(0, 5), (5, 10)]
    assert partition_range(0, 1000, [0.3, 0.7]) == [(0, 300), (300, 1000)]
    assert partition_range(0, 7, [0.33, 0.33, 0.34]) == [(0, 2), (2, 5), (5, 7)]
    with pytest.raises(ValueError):
        partition_range(5, 1, [1.0])
    with pytest.raises(ValueError):
        partition_range(0, 1, [])


def test_partition_totality_random():
    # SPEC.md:506 partition totality
    rng = np.random.default_rng(11)
    for _ in range(2000):
        k = int(rng.integers(1, 9))
        w = rng.random(k)
        r = list(w / w.sum())
        lb = int(rng.integers(0, 100))
        ub = lb + int(rng.integers(0, 10**7))
        got = partition_range(lb, ub, r)
        assert got[0][0] == lb and got[-1][1] == ub
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
        assert all(lo <= hi for lo, hi in got)


def test_api_constants_and_types():
    assert ALGORITHMS == ("md5", "sha1", "sm3")
    assert DIGEST_LEN == {"sha1": 20, "md5": 16, "sm3": 32}
    assert issubclass(UnknownAlgorithmError, ValueError)
    with pytest.raises(ValueError):
        Digest("md5", b"\0" * 15)
    with pytest.raises(UnknownAlgorithmError):
        Digest("sha256", b"")
    with pytest.raises(ValueError):
        MessageBatch(1, 0, b"")
    with pytest.raises(ValueError):
        MessageBatch(2, 3, b"12345")
    b = MessageBatch(2, 3, b"abcdef")
    assert b.message(1) == b"def"
    assert b.as_array().shape == (2, 3)


def test_gen_messages(golden):
    import hashlib

    for row in golden("decimal_batches.json"):
        b = gen_messages(row["start"], row["count"], row["width"])
        assert hashlib.sha256(b.data).hexdigest() == row["input_sha256"]
    assert gen_messages(0, 1).data == b"000000000"
    assert gen_messages(999999999, 1).data == b"999999999"
    with pytest.raises(ValueError):
        gen_messages(999999999, 2)
    with pytest.raises(ValueError):
        gen_messages(0, 1, 0)


def test_validation_before_device():
    # argument errors surface before any device work (and identically with or without a GPU)
    with pytest.raises(UnknownAlgorithmError):
        batch_digest("sha256", np.zeros((1, 4), np.uint8))
    with pytest.raises(ValueError):
        batch_digest("md5", np.zeros(4, np.uint8))
    with pytest.raises(ValueError):
        hash_batch("md5", MessageBatch(1, 1, b"a"), threads=0)
    assert hash_batch("md5", MessageBatch(0, 1, b"")) == []
    assert batch_digest("sm3", np.zeros((0, 7), np.uint8)).shape == (0, 32)
    with pytest.raises(ValueError):
        batch_digest_varlen("md5", np.zeros(4, np.uint8), np.array([0, 5], np.uint64))


def test_bad_alg_id_maps_to_unknown_algorithm():
    lib = _native.lib()
    rc = lib.hb_hash_fixed(9, None, 1, 1, None, None, 0, 0, None)
    assert rc == _native.HB_ERR_ALG
    with pytest.raises(UnknownAlgorithmError):
        _native.check(rc)


def test_no_cpu_fallback_without_gpu():
    # with no CUDA device the product path raises instead of computing on the CPU
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        batch_digest("md5", np.zeros((4, 16), np.uint8))
    lib = _native.lib()
    assert lib.hb_hash_fixed_dev(1, 0, ctypes.c_void_p(16), 1, 16, ctypes.c_void_p(16), None, 0) == _native.HB_ERR_NODEV
    with pytest.raises(RuntimeError, match="no CUDA device"):
        digest("md5", b"abc")


def test_digest_small_validation():
    """hb_digest_small rejects a bad alg, an over-long message and null
    buffers before touching a device; the header's limit matches _native."""
    hdr = open(HEADER).read()
    assert int(re.search(r"#define\s+HB_DIGEST_SMALL_MAX\s+(\d+)u", hdr).group(1)) == _native.HB_DIGEST_SMALL_MAX
    lib = _native.lib()
    out = ctypes.create_string_buffer(32)
    assert lib.hb_digest_small(9, b"a", 1, out, -1) == _native.HB_ERR_ALG
    big = b"x" * (_native.HB_DIGEST_SMALL_MAX + 1)
    assert lib.hb_digest_small(1, big, len(big), out, -1) == _native.HB_ERR_INVAL
    assert "HB_DIGEST_SMALL_MAX" in _native.last_error()
    assert lib.hb_digest_small(1, None, 4, out, -1) == _native.HB_ERR_INVAL
    assert lib.hb_digest_small(1, b"abcd", 4, None, -1) == _native.HB_ERR_INVAL


def test_ratio_validation_matches_reference_verifier():
    # pkg/src/hetoc/hir/verify.py:245-260: ratios in [0,1], sum within 1e-9 (checked before any device work)
    from paper_2407_09333_b200.crypto import batch_digest as bd

    rows = np.zeros((4, 8), np.uint8)
    with pytest.raises(ValueError, match="outside"):
        bd("md5", rows, gpus=[0, 0], ratios=[1.5, -0.5])
    with pytest.raises(ValueError, match="sum"):
        bd("md5", rows, gpus=[0, 0], ratios=[0.5, 0.4])
    with pytest.raises(ValueError):
        bd("md5", rows, gpus=[0], ratios=[0.5, 0.5])


def test_var_message_batch_layout():
    from paper_2407_09333_b200.crypto import VarMessageBatch

    b = VarMessageBatch.from_messages([b"", b"abc", b"x" * 70])
    assert b.count == 3 and b.message(0) == b"" and b.message(1) == b"abc" and b.message(2) == b"x" * 70
    assert list(b.offsets_array()) == [0, 0, 3, 73]
    with pytest.raises(ValueError):
        VarMessageBatch(b"abc", (0, 2, 1))
    with pytest.raises(ValueError):
        VarMessageBatch(b"abc", (0, 4))
    with pytest.raises(IndexError):
        b.message(3)


def test_out_argument_validation():
    """``out=`` (keyword-only extension) is checked before any device work."""
    from paper_2407_09333_b200.crypto import batch_digest, batch_digest_varlen, hash_decimal

    data = np.zeros((4, 8), np.uint8)
    for bad in (np.zeros((4, 20), np.uint8), np.zeros((4, 16), np.int32), np.zeros((16, 4), np.uint8).T,
                [[0] * 16] * 4):
        with pytest.raises(ValueError):
            batch_digest("md5", data, out=bad)
    with pytest.raises(ValueError):
        batch_digest_varlen("sha1", np.zeros(8, np.uint8), np.array([0, 8], np.uint64), out=np.zeros((2, 20), np.uint8))
    with pytest.raises(ValueError):
        hash_decimal("sm3", 0, 3, out=np.zeros((3, 20), np.uint8))


def test_digest_list_matches_constructor():
    """hash_batch's fast Digest construction leaves the same objects the
    validating dataclass __init__ does (equality, hash, repr, frozenness)."""
    import dataclasses

    from paper_2407_09333_b200.crypto import Digest, batch
    from paper_2407_09333_b200.crypto.batch import _digest_list

    assert batch._hb_pyobj is not None, "csrc/hb_pyobj.c not built"
    helper = batch._hb_pyobj
    for alg, dlen in (("md5", 16), ("sha1", 20), ("sm3", 32)):
        raw = bytes(range(256)) * 2
        n = len(raw) // dlen
        fast = _digest_list(alg, raw, n)
        batch._hb_pyobj = None  # the pure-Python reference loop
        try:
            assert _digest_list(alg, raw, n) == fast
        finally:
            batch._hb_pyobj = helper
        assert helper.digest_list(Digest, alg, memoryview(raw), dlen, n) == fast
        arr = np.frombuffer(raw, np.uint8)[: n * dlen].reshape(n, dlen)  # the digest-array form hash_batch passes
        assert _digest_list(alg, arr, n) == fast
        ref = [Digest(alg, raw[i * dlen:(i + 1) * dlen]) for i in range(n)]
        assert fast == ref
        assert [hash(d) for d in fast] == [hash(d) for d in ref]
        assert repr(fast[1]) == repr(ref[1]) and fast[1].hex() == ref[1].hex()
        with pytest.raises(dataclasses.FrozenInstanceError):
            fast[0].data = b""
    assert _digest_list("md5", b"", 0) == []
    with pytest.raises(ValueError):
        helper.digest_list(Digest, "md5", b"x" * 31, 16, 2)  # buffer shorter than count * dlen
    with pytest.raises(TypeError):
        helper.digest_list(int, "md5", b"x" * 32, 16, 2)  # not a Python class


def test_buffer_address_helper():
    """crypto's _addr (the C helper) returns what ndarray.ctypes.data does,
    for writable, read-only, empty and offset views; non-contiguous buffers
    are rejected rather than passed as a wrong address."""
    from paper_2407_09333_b200.crypto import batch

    assert batch._hb_pyobj is not None, "csrc/hb_pyobj.c not built"
    base = np.arange(512, dtype=np.uint8).reshape(8, 64)
    for a in (base, base[3:], np.frombuffer(b"abcdef", np.uint8), np.zeros((0, 16), np.uint8),
              np.zeros(9, np.uint64)):
        assert batch._addr(a) == a.ctypes.data
    with pytest.raises((BufferError, ValueError)):
        batch._hb_pyobj.addr(base[:, ::2])
