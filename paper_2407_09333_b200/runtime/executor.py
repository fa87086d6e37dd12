"""Executor of lowered hash programs on B200 GPUs.

The reference interprets lowered modules against *simulated* accelerators
(``pkg/src/hetoc/runtime/executor.py``): ``hyper.alloc`` reserves bytes in a
per-device ``Arena``, ``hyper.memcpy`` copies between bytearrays and charges a
per-byte latency, ``dev.launch`` of the canonical digest loop calls
``batch_digest`` on the CPU (``_fast_digest``, ``:562-599``), and
``execute_batched`` re-runs an over-capacity launch group in sub-batches
(``_run_group``, ``:603-699``).  Here the same program drives real GPUs:

* ``hyper.alloc`` on a ``cuda`` device -> device memory (PyTorch's caching
  allocator is the pool; the arena check against ``DeviceSpec.mem_bytes``
  is the reference's, ``arena.py:40-44``);
* ``hyper.memcpy`` -> asynchronous H2D / D2H / D2D copies on the device's
  streams from page-locked host buffers, element offsets as ``_exec_copy``
  (``:492-522``);
* ``dev.launch`` of the digest loop -> ``hb_hash_fixed_dev`` on rows
  ``[lb + base, ub + base)`` of the device slice (the same row arithmetic as
  ``_fast_digest``), i.e. the sm_100a kernels;
* launch groups over capacity run as ``k`` sub-batches with the reference's
  ``k`` and chunk bounds (so ``batch_count`` matches), alternating between two
  streams per GPU so sub-batch c+1's copy-in overlaps sub-batch c's kernel;
* groups on different GPUs are issued asynchronously and run concurrently;
  the host synchronises once, at the end.

Time in the report is measured, not simulated: per device the CUDA-event span
of its work (``wall_time``), the summed kernel time (``compute_s``) and the
summed copy time (``charge_s``).  There is no CPU hash path: a digest loop
bound to the host (a non-zero host duty ratio) raises :class:`ExecError`.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from .. import _native
from ..crypto.batch import DIGEST_LEN
from .devices import DeviceTable
from .program import ELEM_BYTES, Op, Program, ProgramError, VarDigestLoop, parse


class ExecError(RuntimeError):
    pass


@dataclass
class ExecReport:
    """Same fields as the reference's ``ExecReport`` (executor.py:69-81)."""

    wall_time: dict[str, float] = field(default_factory=dict)
    batch_count: dict[str, int] = field(default_factory=dict)
    bytes_copied: dict[str, int] = field(default_factory=dict)
    outputs: dict[str, bytes] = field(default_factory=dict)
    returned: list = field(default_factory=list)
    elapsed_s: float = 0.0
    compute_s: dict[str, float] = field(default_factory=dict)
    charge_s: dict[str, float] = field(default_factory=dict)

    def max_wall(self) -> float:
        return max(self.wall_time.values(), default=0.0)


def _wrap(kind: str, v):  # executor.py:52-59
    if kind == "f64":
        return v
    bits = ELEM_BYTES[kind] * 8
    v &= (1 << bits) - 1
    return v - (1 << bits) if v >= 1 << (bits - 1) else v


class _Buf:
    __slots__ = ("device", "elem", "length", "nbytes", "host", "dev", "ordinal", "pending", "origin")

    def __init__(self, device, elem, length, host=None, dev=None, ordinal=-1):
        self.device, self.elem, self.length = device, elem, length
        self.nbytes = length * ELEM_BYTES[elem]
        self.host, self.dev, self.ordinal = host, dev, ordinal
        self.pending = []  # CUDA events of in-flight async writes into a host buffer
        self.origin = None  # (host buffer, element shift): dev[j] was copied from host[j + shift]


class _Executor:
    def __init__(self, program: Program, devices: DeviceTable, inputs: dict | None, batched: bool):
        import torch

        self.torch = torch
        self.prog = program
        self.devices = devices
        self.inputs = dict(inputs or {})
        self.batched = batched
        self.env: dict[int, object] = {}
        self.in_use = {d.id: 0 for d in devices.all_devices()}
        self.batches = {d.id: 0 for d in devices.all_devices()}
        self.copied = {d.id: 0 for d in devices.all_devices()}
        self.streams: dict[str, list] = {}
        self.cur: dict[str, int] = {}  # device -> index of the stream in use
        self.t_start: dict[str, object] = {}
        self.t_end: dict[str, list] = {}
        self.kernel_ev: dict[str, list] = {}
        self.copy_ev: dict[str, list] = {}
        self.returned: list = []

    # ---------------------------------------------------------------- helpers
    def _spec(self, dev: str):
        spec = self.devices.get(dev)
        if spec is None:
            raise ExecError(f"no arena for device '{dev}'")
        return spec

    def _stream(self, dev: str):
        torch = self.torch
        spec = self._spec(dev)
        if dev not in self.streams:
            self.streams[dev] = [torch.cuda.Stream(device=spec.ordinal), torch.cuda.Stream(device=spec.ordinal)]
            self.cur[dev] = 0
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(self.streams[dev][0])
            self.streams[dev][1].wait_event(ev)
            self.t_start[dev] = ev
            self.t_end[dev], self.kernel_ev[dev], self.copy_ev[dev] = [], [], []
        return self.streams[dev][self.cur[dev]]

    def _timed(self, dev: str, bucket: dict, fn):
        torch = self.torch
        s = self._stream(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            fn(s)
            b.record(s)
        bucket[dev].append((a, b))
        self.t_end[dev].append(b)
        return b

    def value(self, vid: int):
        try:
            return self.env[vid]
        except KeyError:
            raise ExecError(f"value %{vid} has no runtime binding") from None

    def _alloc(self, space: str, elem: str, length: int) -> _Buf:
        spec = self._spec(space)
        nbytes = length * ELEM_BYTES[elem]
        if self.in_use[space] + nbytes > spec.mem_bytes:  # arena.py:40-44
            raise ExecError(f"arena '{space}' over capacity: {self.in_use[space]} + {nbytes} > {spec.mem_bytes} bytes")
        self.in_use[space] += nbytes
        torch = self.torch
        if spec.kind == "host":
            return _Buf(space, elem, length, host=torch.zeros(nbytes, dtype=torch.uint8, pin_memory=True))
        s = self._stream(space)
        with torch.cuda.stream(s):
            t = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{spec.ordinal}")
        return _Buf(space, elem, length, dev=t, ordinal=spec.ordinal)

    def _dealloc(self, buf: _Buf, loc: str) -> None:
        if buf.nbytes > self.in_use[buf.device]:
            raise ExecError(f"{loc}: dealloc of unknown or already-freed buffer on '{buf.device}'")
        self.in_use[buf.device] -= buf.nbytes
        # The tensor is released when the last reference goes.  It may have been
        # used on either ping-pong stream of its device: mark it in use on both,
        # so the caching allocator does not hand its memory out again before
        # the work already enqueued on them has finished with it.
        if buf.dev is not None:
            for s in self.streams.get(buf.device, ()):
                buf.dev.record_stream(s)

    def _host_sync(self, buf: _Buf) -> None:
        for ev in buf.pending:
            ev.synchronize()
        buf.pending.clear()

    # ------------------------------------------------------------------ entry
    def run(self) -> ExecReport:
        t0 = time.perf_counter()
        self._bind_params()
        self._run_ops(self.prog.ops)
        for dev, ss in self.streams.items():
            for s in ss:
                s.synchronize()
        report = ExecReport(returned=self.returned, elapsed_s=time.perf_counter() - t0)
        for d in self.devices.all_devices():
            report.batch_count[d.id] = self.batches[d.id]
            report.bytes_copied[d.id] = self.copied[d.id]
            if d.id in self.t_start and self.t_end[d.id]:
                start = self.t_start[d.id]
                report.wall_time[d.id] = max(start.elapsed_time(e) for e in self.t_end[d.id]) * 1e-3
                report.compute_s[d.id] = sum(a.elapsed_time(b) for a, b in self.kernel_ev[d.id]) * 1e-3
                report.charge_s[d.id] = sum(a.elapsed_time(b) for a, b in self.copy_ev[d.id]) * 1e-3
            else:
                report.wall_time[d.id] = report.compute_s[d.id] = report.charge_s[d.id] = 0.0
        for (vid, _), name in zip(self.prog.params, self.prog.names()):
            buf = self.value(vid)
            self._host_sync(buf)
            report.outputs[name] = bytes(buf.host.numpy()) if buf.host is not None else bytes(buf.dev.cpu().numpy())
        return report

    def _bind_params(self) -> None:
        names = self.prog.names()
        known = set(names)
        for (vid, t), name in zip(self.prog.params, names):
            buf = self._alloc(t.space if t.space in self.in_use else "host", t.elem, t.length)
            data = self.inputs.get(name)
            if data is not None:
                raw = np.frombuffer(bytes(data) if not isinstance(data, (bytes, bytearray, memoryview, np.ndarray))
                                    else data, dtype=np.uint8).reshape(-1)
                if raw.size != buf.nbytes:
                    raise ExecError(f"input '{name}' holds {raw.size} bytes, expected {buf.nbytes}")
                if buf.host is not None:
                    buf.host.numpy()[:] = raw
                else:
                    buf.dev.copy_(self.torch.from_numpy(raw.copy()))
            self.env[vid] = buf
        unknown = set(self.inputs) - known
        if unknown:
            raise ExecError(f"inputs name unknown parameters: {sorted(unknown)}")

    # ------------------------------------------------------------ top level
    def _run_ops(self, ops: list[Op]) -> None:
        groups: dict[int, list[Op]] = {}
        if self.batched:
            for op in ops:
                if op.attrs.get("group") is not None:
                    groups.setdefault(op.attrs["group"], []).append(op)
        done: set[int] = set()
        for pos, op in enumerate(ops):
            if id(op) in done:
                continue
            gid = op.attrs.get("group")
            if self.batched and gid is not None and gid in groups:
                g = groups.pop(gid)
                done.update(id(o) for o in g)
                self._run_group(g, pos)
                continue
            if self._run_op(op, f"main#{pos}") == "return":
                return

    def _run_op(self, op: Op, loc: str, lb=None, ub=None, shift: int = 0) -> str | None:
        o = op.opcode
        if o == "const":
            v = op.attrs["value"]
            self.env[op.result] = v if op.rtype == "f64" else _wrap(op.rtype, int(v))
        elif o in ("addi", "muli"):
            a, b = (self.value(x) for x in op.operands)
            self.env[op.result] = _wrap(op.rtype, a + b if o == "addi" else a * b)
        elif o == "memref.alloc":
            self.env[op.result] = self._alloc(op.rtype.space, op.rtype.elem, op.rtype.length)
        elif o == "hyper.alloc":
            self.env[op.result] = self._alloc(op.attrs["device"], op.rtype.elem, op.rtype.length)
        elif o in ("memref.dealloc", "hyper.dealloc"):
            self._dealloc(self.value(op.operands[0]), loc)
        elif o in ("memref.copy", "hyper.memcpy"):
            self._copy(op, loc)
        elif o in ("par.loop", "dev.launch"):
            self._launch(op, loc, lb, ub, shift)
        elif o == "return":
            self.returned = [self.value(x) for x in op.operands]
            return "return"
        else:
            raise ExecError(f"{loc}: opcode '{o}' is not executable at top level")
        return None

    def _copy(self, op: Op, loc: str, src_off=None, dst_off=None, count=None) -> None:
        """Element-offset copy, bounds as executor.py:492-522, issued async."""
        torch = self.torch
        src, dst = self.value(op.operands[0]), self.value(op.operands[1])
        so = op.attrs.get("src_off", 0) if src_off is None else src_off
        do = op.attrs.get("dst_off", 0) if dst_off is None else dst_off
        cnt = op.attrs.get("count") if count is None else count
        if cnt is None:
            cnt = min(src.length - so, dst.length - do)
        if so < 0 or do < 0 or cnt < 0:
            raise ExecError(f"{loc}: negative copy range")
        if so + cnt > src.length or do + cnt > dst.length:
            raise ExecError(f"{loc}: copy range exceeds buffer bounds")
        es = ELEM_BYTES[src.elem]
        a0, a1, b0 = so * es, (so + cnt) * es, do * es
        nbytes = a1 - a0
        if nbytes == 0:
            return
        if src.host is not None and dst.host is not None:
            self._host_sync(src)
            self._host_sync(dst)
            dst.host.numpy()[b0:b0 + nbytes] = src.host.numpy()[a0:a1]
            return
        if src.host is not None:  # H2D
            dev = dst.device

            def h2d(s):
                for ev in src.pending:
                    s.wait_event(ev)
                dst.dev[b0:b0 + nbytes].copy_(src.host[a0:a1], non_blocking=True)
            self._timed(dev, self.copy_ev, h2d)
            if src.elem == dst.elem:  # where a varlen launch finds the offsets' host values
                dst.origin = (src, so - do)
            self.copied[dev] += nbytes
        elif dst.host is not None:  # D2H
            dev = src.device
            ev = self._timed(dev, self.copy_ev,
                             lambda s: dst.host[b0:b0 + nbytes].copy_(src.dev[a0:a1], non_blocking=True))
            dst.pending.append(ev)
            self.copied[dev] += nbytes
        else:  # device to device (same or peer GPU)
            dev = dst.device
            if src.device != dst.device:
                # the source may have been written on either ping-pong stream of its device
                self._stream(src.device)
                for ss in self.streams[src.device]:
                    ev = torch.cuda.Event()
                    ev.record(ss)
                    self._stream(dev).wait_event(ev)
            self._timed(dev, self.copy_ev, lambda s: dst.dev[b0:b0 + nbytes].copy_(src.dev[a0:a1], non_blocking=True))
            self.copied[dev] += nbytes
            if src.origin is not None and src.elem == dst.elem:
                dst.origin = (src.origin[0], src.origin[1] + so - do)

    def _launch(self, op: Op, loc: str, lb=None, ub=None, shift: int = 0) -> None:
        dev = op.attrs["device"]
        spec = self._spec(dev)
        lb = op.attrs["lb"] if lb is None else lb
        ub = op.attrs["ub"] if ub is None else ub
        if ub <= lb:
            return
        if spec.kind == "host" or spec.host_mapped:
            raise ExecError(f"{loc}: digest loop bound to host device '{dev}': the B200 runtime has no CPU hash "
                            "path (no CPU fallback); give the host a duty ratio of 0")
        self.batches[dev] += 1
        d = op.body
        if isinstance(d, VarDigestLoop):
            self._launch_varlen(d, spec, dev, loc, lb, ub)
            return
        base = d.base + (shift if d.from_const else 0)
        msgs, out = self.value(d.msgs), self.value(d.out)
        dlen = DIGEST_LEN[d.alg]
        lo, hi = lb + base, ub + base
        if msgs.elem != "i8" or out.elem != "i8":
            raise ExecError(f"{loc}: digest buffers must be i8")
        if msgs.length % d.msg_len or out.length % dlen:
            raise ExecError(f"{loc}: digest buffers are not whole rows")
        if lo < 0 or hi * d.msg_len > msgs.length or hi * dlen > out.length:
            raise ExecError(f"digest rows [{lo}, {hi}) out of bounds")
        if msgs.dev is None or out.dev is None or msgs.device != dev or out.device != dev:
            raise ExecError(f"{loc}: dev.launch on '{dev}' must address buffers resident on '{dev}'")
        lib = _native.lib()

        def k(s):
            rc = lib.hb_hash_fixed_dev(_native.ALG_ID[d.alg], spec.ordinal, msgs.dev.data_ptr() + lo * d.msg_len,
                                       hi - lo, d.msg_len, out.dev.data_ptr() + lo * dlen, s.cuda_stream, 0)
            _native.check(rc, "hb_hash_fixed_dev")
        self._timed(dev, self.kernel_ev, k)

    def _offset_at(self, offb: _Buf, j: int) -> int:
        """Global byte offset held in element j of an i64 offsets buffer: from
        the host buffer it was copied from (no device read), else read back."""
        if offb.origin is not None:
            src, shift = offb.origin
            self._host_sync(src)
            return int(src.host.numpy().view(np.int64)[j + shift])
        return int(offb.dev[8 * j:8 * j + 8].cpu().numpy().view(np.int64)[0])

    def _launch_varlen(self, d: VarDigestLoop, spec, dev: str, loc: str, lb: int, ub: int) -> None:
        """Rows [lb, ub) of the varlen digest loop: message t is
        msgs[offsets[t] - B, offsets[t+1] - B) with B the offset of the
        buffer's first message (offsets re-based per shard / sub-batch)."""
        msgs, offb, out = self.value(d.msgs), self.value(d.offsets), self.value(d.out)
        dlen = DIGEST_LEN[d.alg]
        if msgs.elem != "i8" or out.elem != "i8" or offb.elem not in ("i64", "index"):
            raise ExecError(f"{loc}: varlen digest needs i8 data/digests and i64 offsets")
        if lb < 0 or ub + 1 > offb.length or ub * dlen > out.length:
            raise ExecError(f"varlen digest rows [{lb}, {ub}) out of bounds")
        if any(b.dev is None or b.device != dev for b in (msgs, offb, out)):
            raise ExecError(f"{loc}: dev.launch on '{dev}' must address buffers resident on '{dev}'")
        base = self._offset_at(offb, 0)
        lo_b, hi_b = self._offset_at(offb, lb) - base, self._offset_at(offb, ub) - base
        if lo_b < 0 or hi_b > msgs.nbytes:
            raise ExecError(f"{loc}: offsets address bytes [{lo_b}, {hi_b}) outside the {msgs.nbytes}-byte data buffer")
        lib = _native.lib()
        n = ub - lb
        torch = self.torch

        def k(s):
            with torch.cuda.stream(s):
                scratch = torch.empty(int(lib.hb_varlen_scratch_bytes(n)), dtype=torch.uint8,
                                      device=f"cuda:{spec.ordinal}")
            rc = lib.hb_hash_varlen_dev(_native.ALG_ID[d.alg], spec.ordinal, msgs.dev.data_ptr(), msgs.nbytes,
                                        offb.dev.data_ptr() + 8 * lb, base, n, out.dev.data_ptr() + lb * dlen,
                                        scratch.data_ptr(), s.cuda_stream, 0)
            _native.check(rc, "hb_hash_varlen_dev")
        self._timed(dev, self.kernel_ev, k)

    # -------------------------------------------------------- batched groups
    def _run_group(self, ops: list[Op], pos: int) -> None:
        """executor.py:603-699, sub-batches alternating between two streams."""
        loc = f"main#{pos}(group)"
        launches = [o for o in ops if o.opcode == "dev.launch"]
        if len(launches) != 1:
            for o in ops:
                self._run_op(o, loc)
            return
        launch = launches[0]
        if isinstance(launch.body, VarDigestLoop):
            self._run_group_varlen(ops, launch, loc)
            return
        dev = launch.attrs["device"]
        spec = self._spec(dev)
        allocs = [o for o in ops if o.opcode == "hyper.alloc"]
        needed = sum(o.rtype.nbytes for o in allocs)
        cap = spec.mem_bytes
        if needed <= cap:
            for o in ops:
                self._run_op(o, loc)
            return
        n = launch.attrs["ub"] - launch.attrs["lb"]
        sliced = sum(o.rtype.nbytes for o in allocs if o.attrs.get("slice_stride") is not None)
        whole = needed - sliced
        if whole >= cap or n == 0:
            raise ExecError(f"{loc}: group needs {needed} bytes of which {whole} are unsplittable, over capacity {cap}")
        k = math.ceil(needed / cap)
        k = max(k, math.ceil(sliced / (cap - whole)))
        k = min(k, n)
        chunks = _chunk_ranges(n, k)
        while True:
            per_elem = sliced / n
            biggest = max(hi - lo for lo, hi in chunks)
            if whole + math.ceil(biggest * per_elem) <= cap or k >= n:
                break
            k += 1
            chunks = _chunk_ranges(n, k)
        if whole + math.ceil(max(hi - lo for lo, hi in chunks) * per_elem) > cap:
            raise ExecError(f"{loc}: a single element exceeds device capacity {cap}")
        alloc_ids = {o.result for o in allocs}
        stride_of = {o.result: o.attrs.get("slice_stride") for o in allocs}
        copies_in = [o for o in ops if o.opcode == "hyper.memcpy" and o.operands[1] in alloc_ids]
        copies_out = [o for o in ops if o.opcode == "hyper.memcpy" and o.operands[0] in alloc_ids]
        torch = self.torch
        s0, s1 = self._stream(dev), self.streams[dev][1]
        # stream 1 joins stream 0's order before the group (buffers written
        # earlier on stream 0 may be read by sub-batches on stream 1) ...
        ev = torch.cuda.Event()
        ev.record(s0)
        s1.wait_event(ev)
        for ci, (c0, c1) in enumerate(chunks):
            self.cur[dev] = ci % 2  # ping-pong: chunk c+1's copy-in overlaps chunk c's kernel
            cn = c1 - c0
            for a in allocs:
                stride = stride_of[a.result]
                length = a.rtype.length if stride is None else cn * stride
                self.env[a.result] = self._alloc(dev, a.rtype.elem, length)
            for cp in copies_in:
                stride = stride_of[cp.operands[1]]
                if stride is None:
                    self._copy(cp, loc)
                else:
                    self._copy(cp, loc, src_off=cp.attrs.get("src_off", 0) + c0 * stride, dst_off=0,
                               count=cn * stride)
            self._launch(launch, loc, lb=0, ub=cn, shift=c0)
            for cp in copies_out:
                stride = stride_of[cp.operands[0]]
                if stride is None:
                    self._copy(cp, loc)
                else:
                    self._copy(cp, loc, src_off=0, dst_off=cp.attrs.get("dst_off", 0) + c0 * stride,
                               count=cn * stride)
            for a in allocs:
                self._dealloc(self.value(a.result), loc)
        # ... and stream 0 waits for stream 1 after it, so later ops on stream 0
        # see every sub-batch's writes
        ev = torch.cuda.Event()
        ev.record(s1)
        s0.wait_event(ev)
        self.cur[dev] = 0


    def _run_group_varlen(self, ops: list[Op], launch: Op, loc: str) -> None:
        """The capacity sub-batching of _run_group (executor.py:603-699) for a
        varlen group: if the group's buffers exceed the device's ``mem_bytes``,
        its messages are cut into k equal-count chunks, k grown from the
        reference's starting estimate until the largest chunk's data +
        offsets + digests fit; each chunk copies in its own byte range and
        offsets slice and launches with its own offset base."""
        dev = launch.attrs["device"]
        spec = self._spec(dev)
        d = launch.body
        allocs = {o.result: o for o in ops if o.opcode == "hyper.alloc"}
        needed = sum(o.rtype.nbytes for o in allocs.values())
        cap = spec.mem_bytes
        if needed <= cap:
            for o in ops:
                self._run_op(o, loc)
            return
        n = launch.attrs["ub"] - launch.attrs["lb"]
        cin = {o.operands[1]: o for o in ops if o.opcode == "hyper.memcpy" and o.operands[1] in allocs}
        cout = [o for o in ops if o.opcode == "hyper.memcpy" and o.operands[0] in allocs]
        if set(allocs) != {d.msgs, d.offsets, d.out} or d.msgs not in cin or d.offsets not in cin or len(cout) != 1:
            raise ExecError(f"{loc}: varlen group is not the canonical lowering (data, offsets, digests)")
        host_off = self.value(cin[d.offsets].operands[0])
        if host_off.host is None:
            raise ExecError(f"{loc}: over-capacity varlen group needs its offsets on the host")
        s_off = cin[d.offsets].attrs.get("src_off", 0)
        offs = host_off.host.numpy().view(np.int64)[s_off:s_off + n + 1].astype(np.int64)
        dlen = DIGEST_LEN[d.alg]

        def need(c0, c1):
            return int(offs[c1] - offs[c0]) + 8 * (c1 - c0 + 1) + dlen * (c1 - c0)

        k = min(max(1, math.ceil(needed / cap)), n)
        chunks = _chunk_ranges(n, k)
        while max(need(a, b) for a, b in chunks) > cap and k < n:
            k += 1
            chunks = _chunk_ranges(n, k)
        if max(need(a, b) for a, b in chunks) > cap:
            raise ExecError(f"{loc}: a single message exceeds device capacity {cap}")
        torch = self.torch
        s0, s1 = self._stream(dev), self.streams[dev][1]
        ev = torch.cuda.Event()
        ev.record(s0)
        s1.wait_event(ev)
        out_copy = cout[0]
        for ci, (c0, c1) in enumerate(chunks):
            self.cur[dev] = ci % 2
            cn = c1 - c0
            self.env[d.msgs] = self._alloc(dev, "i8", int(offs[c1] - offs[c0]))
            self.env[d.offsets] = self._alloc(dev, allocs[d.offsets].rtype.elem, cn + 1)
            self.env[d.out] = self._alloc(dev, "i8", cn * dlen)
            self._copy(cin[d.msgs], loc, src_off=int(offs[c0]), dst_off=0, count=int(offs[c1] - offs[c0]))
            self._copy(cin[d.offsets], loc, src_off=s_off + c0, dst_off=0, count=cn + 1)
            self._launch(launch, loc, lb=0, ub=cn, shift=c0)
            self._copy(out_copy, loc, src_off=0, dst_off=out_copy.attrs.get("dst_off", 0) + c0 * dlen, count=cn * dlen)
            for r in (d.msgs, d.offsets, d.out):
                self._dealloc(self.value(r), loc)
        ev = torch.cuda.Event()
        ev.record(s1)
        s0.wait_event(ev)
        self.cur[dev] = 0


def _chunk_ranges(n: int, k: int) -> list[tuple[int, int]]:  # executor.py:702-704
    bounds = np.linspace(0, n, k + 1, dtype=np.int64)
    return [(int(bounds[i]), int(bounds[i + 1])) for i in range(k)]


def _as_program(program, param_names=None) -> Program:
    if isinstance(program, Program):
        return program
    if isinstance(program, str):
        return parse(program, param_names)
    from .program import from_hir

    try:
        return from_hir(program)
    except ProgramError:
        raise
    except Exception as e:  # not a module-like object
        raise ProgramError(f"cannot execute {type(program).__name__}: {e}") from None


def execute(program, devices: DeviceTable, inputs: dict | None = None, *, batched: bool = False,
            param_names: list[str] | None = None) -> ExecReport:
    """Run a lowered hash program (a :class:`Program`, its printed text -- whose
    parameters are ``arg0, arg1, ...`` unless ``param_names`` is given -- or a
    reference ``HirModule``) on the GPUs of ``devices``."""
    return _Executor(_as_program(program, param_names), devices, inputs, batched).run()


def execute_batched(program, devices: DeviceTable, inputs: dict | None = None, *,
                    param_names: list[str] | None = None) -> ExecReport:
    """Like :func:`execute`, but launch groups too large for their device run in sub-batches."""
    return execute(program, devices, inputs, batched=True, param_names=param_names)
