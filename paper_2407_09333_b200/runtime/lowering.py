"""Lowering of a hash batch onto per-device launch groups (the *hyper* task
splitting + data management contract), emitted as a :class:`Program`.

Restates, for ``crypto.hash_batch`` over a ``(count, msg_len)`` message buffer,
what the reference's ``lower-crypto`` + ``lower-hyper-for`` passes emit
(``pkg/src/hetoc/passes/lower_crypto.py:35-80``,
``pkg/src/hetoc/passes/lower_hyper_for.py:200-368``):

* ``partition_range(0, count, ratios)`` splits the messages
  (``passes/partition.py:17-31``); bindings whose range is empty are dropped;
* a host-mapped binding becomes a ``par.loop`` (``_emit_par_loop``);
* every other binding becomes launch group g: ``hyper.alloc`` of the message
  slice (``slice_stride = msg_len``) and copy-in from ``src_off = s*msg_len``,
  ``hyper.alloc`` of the digest slice (``slice_stride = dlen``), ``dev.launch``
  over ``[0, n)`` with ``offset(s)``, then ``hyper.dealloc`` of the message
  slice, copy-back to ``dst_off = s*dlen`` and ``hyper.dealloc`` of the digest
  slice (``_emit_dev_launch``, ``:279-368``);
* ``accel`` is set only for SHA-1 when the host reports the SHA extension and
  it is not disabled, then narrowed per device (``select_digest_accel``
  ``lower_crypto.py:29-32``, ``_refine_digest_accel`` ``lower_hyper_for.py:256-259``).

``tests/test_runtime.py`` checks the printed result against the reference
pipeline's own output for every golden program (``tests/golden/lowered.json``).
"""

from __future__ import annotations

import numpy as np

from ..crypto.batch import DIGEST_LEN, _check_alg
from ..passes import partition_range
from .devices import DeviceTable
from .program import BufType, DigestLoop, Op, Program, VarDigestLoop

RATIO_SUM_TOL = 1e-9  # hir/core.py RATIO_SUM_TOL


class LoweringError(ValueError):
    pass


def _check_bindings(bindings):
    bindings = [(str(d), float(r)) for d, r in bindings]
    total = sum(r for _, r in bindings)
    if abs(total - 1.0) > RATIO_SUM_TOL:
        raise LoweringError(f"duty ratios sum to {total!r}, expected 1")
    return bindings


def lower_hash_batch(alg: str, count: int, msg_len: int, bindings, devices: DeviceTable,
                     no_sha_accel: bool = False) -> Program:
    """``bindings``: sequence of ``(device_id, duty_ratio)``."""
    _check_alg(alg)
    if count < 0 or msg_len <= 0:
        raise LoweringError("count must be >= 0 and msg_len > 0")
    bindings = _check_bindings(bindings)
    dlen = DIGEST_LEN[alg]
    msgs, out = 0, 1
    prog = Program("main", [(msgs, BufType("i8", count * msg_len)), (out, BufType("i8", count * dlen))], [],
                   ["msgs", "out"])
    accel0 = alg == "sha1" and not no_sha_accel and devices.host.sha_accel
    ranges = partition_range(0, count, [r for _, r in bindings])
    nxt, group = 2, 0
    for (dev, _), (s, e) in zip(bindings, ranges):
        if s >= e:
            continue
        spec = devices.resolve(dev)
        accel = accel0 and spec.sha_accel
        if devices.is_host_mapped(dev):
            prog.ops.append(Op("par.loop", [], nxt, {"device": dev, "lb": s, "ub": e},
                               body=DigestLoop(msgs, out, alg, msg_len, accel)))
            nxt += 1
            continue
        n = e - s
        dm, do, iv = nxt, nxt + 1, nxt + 2
        nxt += 3
        prog.ops += [
            Op("hyper.alloc", [], dm, {"device": dev, "group": group, "slice_stride": msg_len},
               rtype=BufType("i8", n * msg_len, dev)),
            Op("hyper.memcpy", [msgs, dm], None, {"group": group, "src_off": s * msg_len, "dst_off": 0,
                                                  "count": n * msg_len}),
            Op("hyper.alloc", [], do, {"device": dev, "group": group, "slice_stride": dlen},
               rtype=BufType("i8", n * dlen, dev)),
            Op("dev.launch", [], iv, {"device": dev, "lb": 0, "ub": n, "offset": s, "group": group},
               body=DigestLoop(dm, do, alg, msg_len, accel)),
            Op("hyper.dealloc", [dm], None, {"group": group}),
            Op("hyper.memcpy", [do, out], None, {"group": group, "src_off": 0, "dst_off": s * dlen,
                                                 "count": n * dlen}),
            Op("hyper.dealloc", [do], None, {"group": group}),
        ]
        group += 1
    prog.ops.append(Op("return"))
    return prog


def lower_hash_batch_varlen(alg: str, offsets, bindings, devices: DeviceTable) -> Program:
    """The variable-length counterpart (the reference
    compiler has none: ``crypto.hash_batch`` requires ``msg_len``,
    ``pkg/src/hetoc/hir/verify.py:343-358``).  ``offsets``: n+1 non-decreasing
    byte offsets into the ``msgs`` parameter (``buf<i8, offsets[n]>``);
    message i = ``msgs[offsets[i], offsets[i+1])``.

    Same task splitting and data management as the fixed-width lowering
    (``_emit_dev_launch``, ``lower_hyper_for.py:279-368``), by message count:
    binding j gets messages ``[s, e)`` of ``partition_range(0, n, ratios)``;
    its group allocates and copies in the data slice ``[offsets[s],
    offsets[e])`` (``src_off = offsets[s]``; ``slice_offsets`` marks a buffer
    sliced by the offsets), the offsets slice ``[s, e]`` (n+1 entries, still
    global) and the digest slice (``slice_stride = dlen``), launches the varlen digest loop with
    ``offset_base = offsets[s]`` (the offsets re-based per shard), and copies
    the digests back to ``dst_off = s*dlen``.  Host bindings are refused (no
    CPU hash path)."""
    _check_alg(alg)
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64).reshape(-1))
    if off.shape[0] < 1 or off[0] < 0 or np.any(np.diff(off) < 0):
        raise LoweringError("offsets must be n+1 non-negative, non-decreasing byte offsets")
    n = off.shape[0] - 1
    bindings = _check_bindings(bindings)
    dlen = DIGEST_LEN[alg]
    msgs, offp, out = 0, 1, 2
    prog = Program("main", [(msgs, BufType("i8", int(off[-1]))), (offp, BufType("i64", n + 1)),
                            (out, BufType("i8", n * dlen))], [], ["msgs", "offsets", "out"])
    ranges = partition_range(0, n, [r for _, r in bindings])
    nxt, group = 3, 0
    for (dev, _), (s, e) in zip(bindings, ranges):
        if s >= e:
            continue
        if devices.is_host_mapped(dev):
            raise LoweringError(f"binding '{dev}' is host-mapped: the B200 runtime has no CPU hash path; "
                                "give the host a duty ratio of 0")
        devices.resolve(dev)
        cnt = e - s
        b0, b1 = int(off[s]), int(off[e])
        dm, doff, do, iv = nxt, nxt + 1, nxt + 2, nxt + 3
        nxt += 4
        prog.ops += [
            Op("hyper.alloc", [], dm, {"device": dev, "group": group, "slice_offsets": 1},
               rtype=BufType("i8", b1 - b0, dev)),
            Op("hyper.memcpy", [msgs, dm], None, {"group": group, "src_off": b0, "dst_off": 0, "count": b1 - b0}),
            Op("hyper.alloc", [], doff, {"device": dev, "group": group, "slice_stride": 1},
               rtype=BufType("i64", cnt + 1, dev)),
            Op("hyper.memcpy", [offp, doff], None, {"group": group, "src_off": s, "dst_off": 0, "count": cnt + 1}),
            Op("hyper.alloc", [], do, {"device": dev, "group": group, "slice_stride": dlen},
               rtype=BufType("i8", cnt * dlen, dev)),
            Op("dev.launch", [], iv, {"device": dev, "lb": 0, "ub": cnt, "offset": s, "group": group},
               body=VarDigestLoop(dm, doff, do, alg, b0)),
            Op("hyper.dealloc", [dm], None, {"group": group}),
            Op("hyper.dealloc", [doff], None, {"group": group}),
            Op("hyper.memcpy", [do, out], None, {"group": group, "src_off": 0, "dst_off": s * dlen,
                                                 "count": cnt * dlen}),
            Op("hyper.dealloc", [do], None, {"group": group}),
        ]
        group += 1
    prog.ops.append(Op("return"))
    return prog
