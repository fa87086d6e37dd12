"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.json,
produced by tests/golden/make_golden.py from /root/reference) and against
hashlib as an independent implementation.  CPU only."""

import hashlib

import numpy as np
import pytest

import oracle

ALGS = ("sha1", "md5", "sm3")


def _hashlib_has_sm3():
    try:
        hashlib.new("sm3")
        return True
    except ValueError:
        return False


def test_kats(golden):
    # SPEC.md:255-257, SPEC.md:266 + FIPS 180 / RFC 1321 / GB/T 32905
    for row in golden("kats.json"):
        assert oracle.digest(row["alg"], bytes.fromhex(row["msg_hex"])).hex() == row["digest"]


def test_spec_vectors_literal():
    assert oracle.digest("sha1", b"abc").hex() == "a9993e364706816aba3e25717850c26c9cd0d89d"
    assert oracle.digest("md5", b"").hex() == "d41d8cd98f00b204e9800998ecf8427e"
    assert oracle.digest("sm3", b"abc").hex() == "66c7f0f462eeedd9d1f2d46bdc10e4e24167c4875cf2f7a2297da02b8f4ba8e0"
    assert oracle.digest("sha1", b"").hex() == "da39a3ee5e6b4b0d3255bfef95601890afd80709"


def test_boundary_lengths(golden):
    # MD padding boundaries and more, against the reference scalar digest()
    for row in golden("boundary.json"):
        m = bytes.fromhex(row["msg_hex"])
        assert len(m) == row["len"]
        for alg in ALGS:
            assert oracle.digest(alg, m).hex() == row[alg], (alg, row["len"])


def test_fixed_batches(golden):
    # reference batch_digest (batch.py:274-290) on counter-generated inputs
    for row in golden("fixed_batches.json"):
        n, L = row["n"], row["msg_len"]
        data = oracle.fill_random(n * L, row["seed"]).reshape(n, L)
        assert hashlib.sha256(data.tobytes()).hexdigest() == row["input_sha256"]  # pins the generator
        for alg in ALGS:
            out = oracle.batch_fixed(alg, data, threads=3)
            assert hashlib.sha256(out.tobytes()).hexdigest() == row[alg], (alg, n, L)
            assert out[0].tobytes().hex() == row[alg + "_first"]
            assert out[-1].tobytes().hex() == row[alg + "_last"]


def test_varlen_batches(golden):
    for row in golden("varlen_batches.json"):
        lens = np.array(row["lens"], np.uint64)
        off = np.zeros(len(lens) + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        data = oracle.fill_random(int(off[-1]), row["seed"])
        assert hashlib.sha256(data.tobytes()).hexdigest() == row["input_sha256"]
        for alg in ALGS:
            out = oracle.batch_varlen(alg, data, off, threads=2)
            assert hashlib.sha256(out.tobytes()).hexdigest() == row[alg]


def test_decimal_batches(golden):
    # gen_messages + hash_batch (batch.py:86-99, :293-316)
    for row in golden("decimal_batches.json"):
        msgs = oracle.gen_decimal(row["start"], row["count"], row["width"])
        assert hashlib.sha256(msgs.tobytes()).hexdigest() == row["input_sha256"]
        for alg in ALGS:
            out = oracle.batch_fixed(alg, msgs)
            assert hashlib.sha256(out.tobytes()).hexdigest() == row[alg]


def test_against_hashlib_random():
    rng = np.random.default_rng(3)
    algs = ALGS if _hashlib_has_sm3() else ("sha1", "md5")
    for L in list(range(0, 130)) + [255, 256, 1023, 1024, 4096, 65536]:
        data = rng.integers(0, 256, (3, L), dtype=np.uint8)
        for alg in algs:
            out = oracle.batch_fixed(alg, data)
            for i in range(3):
                assert out[i].tobytes() == hashlib.new(alg, data[i].tobytes()).digest(), (alg, L)


def test_thread_count_invariance():
    # output independent of thread count
    data = oracle.fill_random(257 * 65, 9).reshape(257, 65)
    for alg in ALGS:
        ref = oracle.batch_fixed(alg, data, 1)
        for t in (2, 4, 8, 300):
            assert np.array_equal(oracle.batch_fixed(alg, data, t), ref)


def test_partition_oracle(golden):
    for row in golden("partition.json"):
        got = oracle.partition_range(row["lb"], row["ub"], row["ratios"])
        assert [list(x) for x in got] == row["ranges"]


@pytest.mark.parametrize("nbytes,off", [(0, 0), (1, 0), (7, 8), (64, 16), (1001, 800)])
def test_fill_random_offset_consistency(nbytes, off):
    # bytes at a byte_offset equal the same slice of a longer stream (shard independence)
    full = oracle.fill_random(off + nbytes + 8, 42)
    part = oracle.fill_random(nbytes, 42, off)
    assert np.array_equal(full[off:off + nbytes], part)
