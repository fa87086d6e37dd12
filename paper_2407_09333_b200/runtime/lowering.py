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

from ..crypto.batch import DIGEST_LEN, _check_alg
from ..passes import partition_range
from .devices import DeviceTable
from .program import BufType, DigestLoop, Op, Program

RATIO_SUM_TOL = 1e-9  # hir/core.py RATIO_SUM_TOL


class LoweringError(ValueError):
    pass


def lower_hash_batch(alg: str, count: int, msg_len: int, bindings, devices: DeviceTable,
                     no_sha_accel: bool = False) -> Program:
    """``bindings``: sequence of ``(device_id, duty_ratio)``."""
    _check_alg(alg)
    if count < 0 or msg_len <= 0:
        raise LoweringError("count must be >= 0 and msg_len > 0")
    bindings = [(str(d), float(r)) for d, r in bindings]
    total = sum(r for _, r in bindings)
    if abs(total - 1.0) > RATIO_SUM_TOL:
        raise LoweringError(f"duty ratios sum to {total!r}, expected 1")
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
