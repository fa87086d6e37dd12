"""Batch hashing over fixed-width and variable-length message buffers, on B200.

Drop-in for the reference module ``hetoc.crypto.batch``
(``pkg/src/hetoc/crypto/batch.py``): same names, argument meaning, layouts and
error behaviour.  The digests are computed by the sm_100a kernels of
``libhetoc_b200.so`` (one thread per message, padding generated in registers);
host buffers are staged, sharded across GPUs by message range and streamed in
chunks by the engine behind ``hb_hash_fixed`` / ``hb_hash_varlen``.  There is
no CPU fallback: without the library or a GPU these functions raise.

Deliberate differences from the reference (documented in DESIGN.md):
  * ``accel`` is accepted and validated but selects nothing -- every algorithm
    runs the same GPU kernels (the reference uses it to pick OpenSSL SHA-1,
    batch.py:266-271).
  * ``threads`` (hash_batch) is validated and otherwise ignored: the whole batch
    is one engine call (splitting it would only add launches).
  * keyword-only ``gpus=`` selects devices (default: all, or $HETOC_B200_GPUS).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .. import _native

try:  # host-object helper compiled next to the CUDA library (csrc/hb_pyobj.c)
    from .. import _hb_pyobj
except ImportError:  # an interpreter it was not built for: the pure-Python loop below
    _hb_pyobj = None

DIGEST_LEN = {"sha1": 20, "md5": 16, "sm3": 32}  # batch.py:23

ALGORITHMS = tuple(sorted(DIGEST_LEN))  # batch.py:25


class UnknownAlgorithmError(ValueError):  # batch.py:33-34
    pass


def _check_alg(alg: str) -> None:  # batch.py:37-39
    if alg not in DIGEST_LEN:
        raise UnknownAlgorithmError(f"unknown hash algorithm {alg!r}; expected one of {ALGORITHMS}")


@dataclass(frozen=True)
class Digest:
    """A single hash result; ``data`` length always matches the algorithm (batch.py:42-57)."""

    alg: str
    data: bytes

    def __post_init__(self):
        _check_alg(self.alg)
        if len(self.data) != DIGEST_LEN[self.alg]:
            raise ValueError(
                f"{self.alg} digest must be {DIGEST_LEN[self.alg]} bytes, got {len(self.data)}"
            )

    def hex(self) -> str:
        return self.data.hex()


@dataclass(frozen=True)
class MessageBatch:
    """Fixed-width message layout: message i lives at bytes [i*msg_len, (i+1)*msg_len) (batch.py:60-83)."""

    count: int
    msg_len: int
    data: bytes

    def __post_init__(self):
        if self.count < 0 or self.msg_len <= 0:
            raise ValueError("count must be >= 0 and msg_len > 0")
        if len(self.data) != self.count * self.msg_len:
            raise ValueError(
                f"data holds {len(self.data)} bytes, expected count*msg_len = "
                f"{self.count * self.msg_len}"
            )

    def message(self, i: int) -> bytes:
        if not 0 <= i < self.count:
            raise IndexError(i)
        return self.data[i * self.msg_len : (i + 1) * self.msg_len]

    def as_array(self) -> np.ndarray:
        return np.frombuffer(self.data, np.uint8).reshape(self.count, self.msg_len)


@dataclass(frozen=True)
class VarMessageBatch:
    """Variable-length layout (configs[3]): message i
    lives at bytes [offsets[i], offsets[i+1]) of ``data``.  The reference's
    ``MessageBatch`` is fixed-width by design and its only
    variable-length path is the scalar ``digest``; this type lets
    ``hash_batch`` take a whole mixed-length batch in one engine call.
    Zero-length messages are allowed (their digest is the empty-message one)."""

    data: bytes
    offsets: tuple

    def __post_init__(self):
        off = np.asarray(self.offsets, dtype=np.int64)
        if off.ndim != 1 or off.shape[0] < 1:
            raise ValueError("offsets must be a 1-D sequence of count+1 entries")
        if off[0] < 0 or np.any(np.diff(off) < 0):
            raise ValueError("offsets must be non-negative and non-decreasing")
        if int(off[-1]) > len(self.data):
            raise ValueError(f"offsets[-1]={int(off[-1])} exceeds the data length {len(self.data)}")
        object.__setattr__(self, "offsets", tuple(int(x) for x in off))

    @classmethod
    def from_messages(cls, messages) -> "VarMessageBatch":
        msgs = [bytes(m) for m in messages]
        off = np.zeros(len(msgs) + 1, np.int64)
        off[1:] = np.cumsum([len(m) for m in msgs])
        return cls(b"".join(msgs), tuple(int(x) for x in off))

    @property
    def count(self) -> int:
        return len(self.offsets) - 1

    def message(self, i: int) -> bytes:
        if not 0 <= i < self.count:
            raise IndexError(i)
        return self.data[self.offsets[i] : self.offsets[i + 1]]

    def offsets_array(self) -> np.ndarray:
        return np.asarray(self.offsets, dtype=np.uint64)


def gen_messages(start_index: int, count: int, width: int = 9) -> MessageBatch:
    """Zero-padded decimal messages for indices [start_index, start_index+count) (batch.py:86-99)."""
    if width <= 0:
        raise ValueError("width must be positive")
    if start_index < 0 or count < 0 or start_index + count > 10**width:
        raise ValueError(
            f"index range [{start_index}, {start_index + count}) does not fit in {width} digits"
        )
    idx = np.arange(start_index, start_index + count, dtype=np.uint64)
    digits = np.empty((count, width), np.uint8)
    for pos in range(width - 1, -1, -1):
        digits[:, pos] = (idx % 10).astype(np.uint8) + ord("0")
        idx //= 10
    return MessageBatch(count=count, msg_len=width, data=digits.tobytes())


def _as_rows(data) -> np.ndarray:
    """(n, width) uint8, C-contiguous.  Non-uint8 input is cast mod 256, as the
    reference's uint8 assignment does (batch.py:133)."""
    arr = np.asarray(data)
    if arr.ndim != 2:
        raise ValueError(f"expected a 2-D (count, width) array, got shape {arr.shape}")
    if arr.dtype != np.uint8:
        arr = arr.astype(np.uint8)
    return np.ascontiguousarray(arr)


def _addr(a: np.ndarray) -> int:
    """Address of a C-contiguous array (the C helper skips building the
    ``ndarray.ctypes`` object, ~1.4 us per buffer on a ~20 us small call)."""
    return _hb_pyobj.addr(a) if _hb_pyobj is not None else a.ctypes.data


def _ptr(a: np.ndarray) -> int | None:
    return _addr(a) if a.size else None


def _out_array(out, n: int, alg: str) -> np.ndarray:
    """The digest array: a new (n, dlen) uint8 array, or the caller's ``out=``
    (keyword-only extension: a reused -- e.g. page-locked -- buffer lets the
    engine DMA digests straight into it)."""
    shape = (n, DIGEST_LEN[alg])
    if out is None:
        return np.empty(shape, np.uint8)
    if not isinstance(out, np.ndarray) or out.dtype != np.uint8 or out.shape != shape or \
            not out.flags.c_contiguous or not out.flags.writeable:
        raise ValueError(f"out must be a writable C-contiguous uint8 array of shape {shape}")
    return out


def _timing_arg(t, timing):
    """hb_timing out-parameter: NULL unless the caller asked for timings (the
    engine then skips its per-stage events, a few driver calls per chunk)."""
    return ctypes.byref(t) if timing is not None else None


def batch_digest(alg: str, data, accel: bool = False, *, gpus=None, ratios=None, flags: int = 0,
                 timing: dict | None = None, out=None) -> np.ndarray:
    """Hash each row of an (n, width) uint8 array; returns a new (n, digest_len) uint8 array.

    Reference: batch.py:274-290.  ``accel`` is accepted for API compatibility.
    ``ratios`` (with ``gpus``) are hyper.for duty ratios: GPU i hashes the
    message range partition_range gives it (lower_hyper_for.py:207-254).
    If ``timing`` is a dict it receives the engine's hb_timing fields.
    """
    _check_alg(alg)
    rows = _as_rows(data)
    n, width = rows.shape
    out = _out_array(out, n, alg)
    if ratios is not None:
        if gpus is None or len(gpus) != len(ratios):
            raise ValueError("ratios need a gpus list of the same length")
    if n == 0 and ratios is None:
        return out
    garr, ng = _native.gpu_array(gpus)
    t = _native.HbTiming()
    if ratios is not None:
        r = (ctypes.c_double * len(ratios))(*[float(x) for x in ratios])
        rc = _native.lib().hb_hash_fixed_split(_native.ALG_ID[alg], _ptr(rows), n, width, _addr(out), garr,
                                               r, ng, int(flags), _timing_arg(t, timing))
    else:
        rc = _native.lib().hb_hash_fixed(_native.ALG_ID[alg], _ptr(rows), n, width, _addr(out), garr, ng,
                                         int(flags), _timing_arg(t, timing))
    _native.check(rc, "hb_hash_fixed")
    if timing is not None:
        timing.update(t.as_dict())
    return out


def batch_digest_varlen(alg: str, data, offsets, *, gpus=None, flags: int = 0,
                        timing: dict | None = None, out=None) -> np.ndarray:
    """Hash message i = data[offsets[i]:offsets[i+1]] for i < len(offsets)-1.

    The reference has no variable-length batch; this is
    ``digest(alg, m)`` (batch.py:102-109) mapped over an offsets array, the
    layout of BASELINE.json config 4.
    """
    _check_alg(alg)
    buf = np.ascontiguousarray(np.asarray(data, dtype=np.uint8).reshape(-1))
    off = np.ascontiguousarray(np.asarray(offsets), dtype=np.uint64)
    if off.ndim != 1 or off.shape[0] < 1:
        raise ValueError("offsets must be a 1-D array of n+1 entries")
    n = off.shape[0] - 1
    out = _out_array(out, n, alg)
    if n == 0:
        return out
    if int(off[-1]) > buf.shape[0]:
        raise ValueError(f"offsets[-1]={int(off[-1])} exceeds the data length {buf.shape[0]}")
    garr, ng = _native.gpu_array(gpus)
    t = _native.HbTiming()
    rc = _native.lib().hb_hash_varlen(_native.ALG_ID[alg], _ptr(buf), _addr(off), n, _addr(out), garr,
                                      ng, int(flags), _timing_arg(t, timing))
    _native.check(rc, "hb_hash_varlen")
    if timing is not None:
        timing.update(t.as_dict())
    return out


def hash_decimal(alg: str, start_index: int, count: int, width: int = 9, *, gpus=None,
                 timing: dict | None = None, out=None) -> np.ndarray:
    """Digests of ``gen_messages(start_index, count, width)`` with the messages
    generated in registers on the GPU (the paper's 10^9 x 9-digit workload,
    PAPER.md:206); returns (count, digest_len) uint8."""
    _check_alg(alg)
    if width <= 0:
        raise ValueError("width must be positive")
    if start_index < 0 or count < 0 or start_index + count > 10**width:
        raise ValueError(
            f"index range [{start_index}, {start_index + count}) does not fit in {width} digits"
        )
    out = _out_array(out, count, alg)
    if count == 0:
        return out
    if width > 20:  # leading zeros beyond 64-bit indices: hash the materialised bytes
        return batch_digest(alg, gen_messages(start_index, count, width).as_array(), gpus=gpus, timing=timing,
                            out=out)
    garr, ng = _native.gpu_array(gpus)
    t = _native.HbTiming()
    rc = _native.lib().hb_hash_decimal(_native.ALG_ID[alg], start_index, count, width, _addr(out), garr, ng,
                                       0, _timing_arg(t, timing))
    _native.check(rc, "hb_hash_decimal")
    if timing is not None:
        timing.update(t.as_dict())
    return out


def digest(alg: str, message: bytes) -> Digest:
    """Single-message digest (batch.py:102-109), computed on the GPU.  Up to
    HB_DIGEST_SMALL_MAX (4 KiB) bytes it is one launch with the message in the
    kernel's parameters (hb_digest_small); longer messages take the varlen path."""
    _check_alg(alg)
    message = bytes(message)
    if len(message) <= _native.HB_DIGEST_SMALL_MAX:
        garr, ng = _native.gpu_array(None)
        out = ctypes.create_string_buffer(DIGEST_LEN[alg])
        rc = _native.lib().hb_digest_small(_native.ALG_ID[alg], message, len(message), out, garr[0] if ng else -1)
        _native.check(rc, "hb_digest_small")
        return Digest(alg, out.raw)
    m = np.frombuffer(message, np.uint8)
    out = batch_digest_varlen(alg, m, np.array([0, m.shape[0]], np.uint64))
    return Digest(alg, out[0].tobytes())


def digest_sha1_accel(message: bytes) -> Digest:
    """SHA-1 of one message (batch.py:112-116); bit-identical to digest("sha1", ...)."""
    return digest("sha1", message)


def hash_batch(alg: str, batch, threads: int = 1, accel: bool = False, *,
               gpus=None) -> list[Digest]:
    """Digest every message of a batch; output is independent of ``threads`` (batch.py:293-316).
    ``batch`` is a ``MessageBatch`` (fixed width) or a ``VarMessageBatch``."""
    _check_alg(alg)
    if threads < 1:
        raise ValueError("threads must be >= 1")
    if batch.count == 0:
        return []
    if isinstance(batch, VarMessageBatch):
        out = batch_digest_varlen(alg, np.frombuffer(batch.data, np.uint8) if batch.data else np.zeros(0, np.uint8),
                                  batch.offsets_array(), gpus=gpus)
    else:
        out = batch_digest(alg, batch.as_array(), accel=accel, gpus=gpus)
    return _digest_list(alg, out, batch.count)


def _digest_list(alg: str, raw, count: int) -> list[Digest]:
    """``count`` Digest objects over consecutive ``DIGEST_LEN[alg]``-byte
    slices of ``raw`` (bytes or the C-contiguous digest array).

    Their fields are valid by construction (``alg`` checked by the caller,
    every slice exactly dlen bytes), so the per-object ``__post_init__`` is
    skipped: the fields go straight into each frozen instance's attribute
    storage, the state the dataclass ``__init__`` leaves.  Building the list
    dominates ``hash_batch`` at large n (reference: ~70 % of a 10^6 x 9 B
    batch).  The compiled helper ``_hb_pyobj`` (built with the
    CUDA library) does it in one C loop, ~6x faster than the dataclass
    constructor; the loop below is its reference implementation and covers an
    interpreter the helper was not built for.  Only Python objects are
    created here -- no hashing."""
    dlen = DIGEST_LEN[alg]
    if _hb_pyobj is not None:  # the same objects, built in one C loop (csrc/hb_pyobj.c)
        return _hb_pyobj.digest_list(Digest, alg, raw, dlen, count)
    raw = bytes(raw)
    new = object.__new__
    out = []
    append = out.append
    for i in range(0, count * dlen, dlen):
        d = new(Digest)
        d.__dict__.update(alg=alg, data=raw[i : i + dlen])
        append(d)
    return out


def sha1(msg: bytes) -> bytes:
    """20-byte SHA-1 of ``msg`` (sha1.py:40-46)."""
    return digest("sha1", msg).data


def md5(msg: bytes) -> bytes:
    """16-byte MD5 of ``msg`` (md5.py:57-63)."""
    return digest("md5", msg).data


def sm3(msg: bytes) -> bytes:
    """32-byte SM3 of ``msg`` (sm3.py:66-72)."""
    return digest("sm3", msg).data
