"""ctypes binding of ``libhetoc_b200.so`` (the C ABI in ``include/hetoc_b200.h``).

The shared library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2407_09333_b200/csrc``).  There is deliberately no fallback: if the
library is missing, or no CUDA device is visible, every hashing call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# $HETOC_B200_LIB selects another in-tree build (A/B tools use the -DHB_AB
# library, ``make -C paper_2407_09333_b200/csrc ab``); a bare name is looked
# up next to this file.
LIB_PATH = os.path.join(_HERE, os.environ.get("HETOC_B200_LIB", "libhetoc_b200.so"))

HB_OK, HB_ERR_ALG, HB_ERR_INVAL, HB_ERR_CUDA, HB_ERR_NOMEM, HB_ERR_NODEV = range(6)
HB_FLAG_NO_TMA, HB_FLAG_NO_SORT, HB_FLAG_SYNC_H2D, HB_FLAG_VARLEN_WORDS = 0x1, 0x2, 0x4, 0x8
HB_FLAG_VARLEN_COOP_OFF, HB_FLAG_VARLEN_COOP = 0x10, 0x20
HB_DIGEST_SMALL_MAX = 4096  # hb_digest_small: longest message passed inside the launch
HB_FLAG_INPUT_READY = 0x40  # fixed width, device-resident: messages not written by the preceding kernel
ALG_ID = {"sha1": 0, "md5": 1, "sm3": 2}

# Every symbol include/hetoc_b200.h declares (tests check the library exports all of them).
EXPORTS = (
    "hb_abi_version", "hb_last_error", "hb_digest_len", "hb_device_count", "hb_device_info", "hb_launch_count",
    "hb_hash_fixed", "hb_hash_fixed_split", "hb_hash_varlen", "hb_digest_small", "hb_hash_decimal", "hb_hash_fixed_dev", "hb_hash_varlen_dev",
    "hb_varlen_scratch_bytes", "hb_hash_decimal_dev", "hb_fill_random_dev", "hb_gen_decimal_dev",
    "hb_alloc_pinned", "hb_free_pinned", "hb_sync_device", "hb_shutdown", "hb_partition_range",
    "hb_ipc_handle", "hb_ipc_open", "hb_ipc_close",
    "hb_tuning_reload", "hb_built_with_ab", "hb_last_kernel_name", "hb_last_timeline", "hb_engine_budget",
)


class HbTiming(ctypes.Structure):
    _fields_ = [
        ("total_ms", ctypes.c_double),
        ("kernel_ms", ctypes.c_double),
        ("h2d_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64),
        ("chunks", ctypes.c_uint64),
        ("launches", ctypes.c_uint64),
        ("shards", ctypes.c_uint64),
        ("device_mask", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class HbSpan(ctypes.Structure):
    _fields_ = [
        ("dev", ctypes.c_int32),
        ("stage", ctypes.c_int32),
        ("chunk", ctypes.c_uint64),
        ("t0_ms", ctypes.c_double),
        ("t1_ms", ctypes.c_double),
    ]


class HbDeviceInfo(ctypes.Structure):
    _fields_ = [
        ("ordinal", ctypes.c_int),
        ("sm_count", ctypes.c_int),
        ("cc_major", ctypes.c_int),
        ("cc_minor", ctypes.c_int),
        ("total_mem", ctypes.c_uint64),
        ("free_mem", ctypes.c_uint64),
        ("pci_bus_id", ctypes.c_int),
        ("clock_khz", ctypes.c_int),
        ("name", ctypes.c_char * 96),
    ]


_lib = None
_lock = threading.Lock()

_u8p = ctypes.POINTER(ctypes.c_uint8)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_intp = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_int = ctypes.c_int

_SIGS = {
    "hb_abi_version": (_int, []),
    "hb_last_error": (ctypes.c_char_p, []),
    "hb_digest_len": (_int, [_int]),
    "hb_device_count": (_int, [_intp]),
    "hb_device_info": (_int, [_int, ctypes.POINTER(HbDeviceInfo)]),
    "hb_launch_count": (_u64, []),
    "hb_hash_fixed": (_int, [_int, _vp, _u64, _u64, _vp, _intp, _int, _u32, ctypes.POINTER(HbTiming)]),
    "hb_hash_fixed_split": (_int, [_int, _vp, _u64, _u64, _vp, _intp, ctypes.POINTER(ctypes.c_double), _int, _u32,
                                   ctypes.POINTER(HbTiming)]),
    "hb_hash_varlen": (_int, [_int, _vp, _vp, _u64, _vp, _intp, _int, _u32, ctypes.POINTER(HbTiming)]),
    "hb_digest_small": (_int, [_int, _vp, _u64, _vp, _int]),
    "hb_hash_decimal": (_int, [_int, _u64, _u64, _int, _vp, _intp, _int, _u32, ctypes.POINTER(HbTiming)]),
    "hb_hash_fixed_dev": (_int, [_int, _int, _vp, _u64, _u64, _vp, _vp, _u32]),
    "hb_hash_varlen_dev": (_int, [_int, _int, _vp, _u64, _vp, _u64, _u64, _vp, _vp, _vp, _u32]),
    "hb_varlen_scratch_bytes": (_u64, [_u64]),
    "hb_hash_decimal_dev": (_int, [_int, _int, _u64, _u64, _int, _vp, _vp]),
    "hb_fill_random_dev": (_int, [_int, _vp, _u64, _u64, _u64, _vp]),
    "hb_gen_decimal_dev": (_int, [_int, _u64, _u64, _int, _vp, _vp]),
    "hb_alloc_pinned": (_vp, [_u64]),
    "hb_free_pinned": (_int, [_vp]),
    "hb_sync_device": (_int, [_int]),
    "hb_shutdown": (_int, []),
    "hb_ipc_handle": (_int, [_vp, _u8p, _u64p]),
    "hb_ipc_open": (_int, [_int, _u8p, ctypes.POINTER(_vp)]),
    "hb_ipc_close": (_int, [_int, _vp]),
    "hb_partition_range": (_int, [ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_double), _int,
                                  ctypes.POINTER(ctypes.c_int64)]),
    "hb_tuning_reload": (_int, []),
    "hb_built_with_ab": (_int, []),
    "hb_last_kernel_name": (_int, [ctypes.c_char_p, _int]),
    "hb_last_timeline": (_int, [ctypes.POINTER(HbSpan), _int]),
    "hb_engine_budget": (_int, [_int, _u64p, _u64p]),
}


class NativeLibraryError(ImportError):
    pass


def lib() -> ctypes.CDLL:
    """Load (once) and return the engine library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "or `make -C paper_2407_09333_b200/csrc` (there is no CPU fallback)"
                )
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def last_error() -> str:
    msg = lib().hb_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map an hb_status to the reference's exception types (batch.py:33-39)."""
    if rc == HB_OK:
        return
    msg = last_error()
    where = f"{what}: " if what else ""
    if rc == HB_ERR_ALG:
        from .crypto.batch import UnknownAlgorithmError

        raise UnknownAlgorithmError(where + msg)
    if rc == HB_ERR_INVAL:
        raise ValueError(where + msg)
    if rc == HB_ERR_NOMEM:
        raise MemoryError(where + msg)
    raise RuntimeError(where + (msg or f"hb status {rc}"))


def device_count() -> int:
    n = ctypes.c_int(0)
    check(lib().hb_device_count(ctypes.byref(n)), "hb_device_count")
    return n.value


def device_info(ordinal: int) -> dict:
    info = HbDeviceInfo()
    check(lib().hb_device_info(ordinal, ctypes.byref(info)), "hb_device_info")
    d = {k: getattr(info, k) for k, _ in HbDeviceInfo._fields_}
    d["name"] = info.name.decode(errors="replace")
    return d


def launch_count() -> int:
    return int(lib().hb_launch_count())


def reload_tuning() -> None:
    """Re-read the $HB_* tuning environment (the library parses it once)."""
    check(lib().hb_tuning_reload(), "hb_tuning_reload")


def built_with_ab() -> bool:
    return bool(lib().hb_built_with_ab())


def last_kernel_name() -> str:
    """Demangled name of the last hash kernel this thread launched (directly
    or through the engine's last call) -- what ncu's launch list shows."""
    buf = ctypes.create_string_buffer(512)
    check(lib().hb_last_kernel_name(buf, 512), "hb_last_kernel_name")
    return buf.value.decode(errors="replace")


STAGES = ("h2d", "kernel", "d2h")


def last_timeline() -> list[dict]:
    """Per-chunk stage spans of this thread's last call made with timing."""
    n = lib().hb_last_timeline(None, 0)
    arr = (HbSpan * max(1, n))()
    n = lib().hb_last_timeline(arr, n)
    return [{"dev": s.dev, "stage": STAGES[s.stage], "chunk": s.chunk, "t0_ms": s.t0_ms, "t1_ms": s.t1_ms}
            for s in arr[:n]]


def engine_budget(gpu: int) -> dict:
    b, c = ctypes.c_uint64(0), ctypes.c_uint64(0)
    check(lib().hb_engine_budget(gpu, ctypes.byref(b), ctypes.byref(c)), "hb_engine_budget")
    return {"budget_bytes": b.value, "chunk_cap_bytes": c.value}


def gpu_array(gpus):
    """(ctypes int array or None, count) for an optional GPU list."""
    if gpus is None:
        env = os.environ.get("HETOC_B200_GPUS", "").strip()
        if env:
            gpus = [int(x) for x in env.split(",") if x.strip()]
    if gpus is None:
        return None, 0
    gpus = [int(g) for g in gpus]
    arr = (ctypes.c_int * max(1, len(gpus)))(*gpus)
    return arr, len(gpus)
