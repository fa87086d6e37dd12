"""Device-resident (kernel-only) entry points over torch CUDA tensors.

PyTorch is plumbing here: it owns device memory and streams; the hashing is
the C ABI (``hb_hash_fixed_dev`` / ``hb_hash_varlen_dev`` / ...).  Work is
enqueued on the tensor's device's *current* torch stream and is not
synchronised, so CUDA events recorded on that stream bracket exactly the
engine's kernels.
"""

from __future__ import annotations

from . import _native
from .crypto.batch import DIGEST_LEN, _check_alg


def _stream_ptr(torch, dev: int) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _check_out(torch, out, n: int, alg: str, device):
    """The kernels write n rows of dlen bytes with 16-byte (MD5/SM3) or 4-byte
    (SHA-1) stores straight through the pointer: anything but a contiguous
    uint8 (n, dlen) tensor on the batch's device, suitably aligned, would be
    an out-of-bounds or misaligned device write."""
    dlen = DIGEST_LEN[alg]
    if out is None:
        return torch.empty((n, dlen), dtype=torch.uint8, device=device)
    align = 4 if alg == "sha1" else 16
    if (out.dtype != torch.uint8 or tuple(out.shape) != (n, dlen) or out.device != device
            or not out.is_contiguous() or out.data_ptr() % align):
        raise ValueError(f"out must be a contiguous uint8 ({n}, {dlen}) tensor on {device}, "
                         f"{align}-byte aligned")
    return out


def hash_fixed(alg: str, msgs, out=None, flags: int = 0):
    """Digest each row of a 2-D uint8 CUDA tensor; returns (n, dlen) uint8 CUDA tensor."""
    import torch

    _check_alg(alg)
    if msgs.dim() != 2 or msgs.dtype != torch.uint8 or not msgs.is_cuda:
        raise ValueError("msgs must be a 2-D uint8 CUDA tensor")
    msgs = msgs.contiguous()
    n, L = msgs.shape
    dev = msgs.device.index
    out = _check_out(torch, out, n, alg, msgs.device)
    if n:
        rc = _native.lib().hb_hash_fixed_dev(_native.ALG_ID[alg], dev, msgs.data_ptr(), n, L, out.data_ptr(),
                                             _stream_ptr(torch, dev), int(flags))
        _native.check(rc, "hb_hash_fixed_dev")
    return out


def hash_varlen(alg: str, data, offsets, out=None, scratch=None, flags: int = 0, offset_base=None):
    """Digest message i = data[offsets[i]-base : offsets[i+1]-base] (CUDA tensors).

    ``offset_base`` defaults to ``offsets[0]`` (read back from the device, a
    synchronising copy); pass it when known to keep the call asynchronous."""
    import torch

    _check_alg(alg)
    if data.dtype != torch.uint8 or offsets.dtype not in (torch.int64, torch.uint64) or not data.is_cuda:
        raise ValueError("data must be uint8 and offsets int64/uint64 CUDA tensors")
    if offsets.device != data.device or offsets.dim() != 1:
        raise ValueError("offsets must be a 1-D tensor on the data's device")
    if not data.is_contiguous() or not offsets.is_contiguous():
        raise ValueError("data and offsets must be contiguous")
    n = offsets.numel() - 1
    dev = data.device.index
    out = _check_out(torch, out, max(n, 0), alg, data.device)
    if n <= 0:
        return out
    if scratch is None and not (flags & _native.HB_FLAG_NO_SORT):
        scratch = torch.empty(int(_native.lib().hb_varlen_scratch_bytes(n)), dtype=torch.uint8, device=data.device)
    elif scratch is not None and (scratch.device != data.device or not scratch.is_contiguous() or
                                  scratch.numel() * scratch.element_size() < int(_native.lib().hb_varlen_scratch_bytes(n))):
        raise ValueError("scratch must be a contiguous tensor of hb_varlen_scratch_bytes(n) bytes on the data's device")
    base = int(offsets[0].item()) if offset_base is None else int(offset_base)
    rc = _native.lib().hb_hash_varlen_dev(_native.ALG_ID[alg], dev, data.data_ptr(), data.numel(),
                                          offsets.data_ptr(), base, n, out.data_ptr(),
                                          scratch.data_ptr() if scratch is not None else None,
                                          _stream_ptr(torch, dev), int(flags))
    _native.check(rc, "hb_hash_varlen_dev")
    return out


def hash_decimal(alg: str, start: int, count: int, width: int = 9, device: int = 0, out=None):
    import torch

    _check_alg(alg)
    out = _check_out(torch, out, count, alg, torch.device("cuda", device))
    if count:
        rc = _native.lib().hb_hash_decimal_dev(_native.ALG_ID[alg], device, start, count, width, out.data_ptr(),
                                               _stream_ptr(torch, device))
        _native.check(rc, "hb_hash_decimal_dev")
    return out


def fill_random(buf, seed: int, byte_offset: int = 0):
    """Fill a uint8 CUDA tensor with the oracle-compatible counter-based bytes."""
    import torch

    dev = buf.device.index
    rc = _native.lib().hb_fill_random_dev(dev, buf.data_ptr(), buf.numel(), int(seed), int(byte_offset),
                                          _stream_ptr(torch, dev))
    _native.check(rc, "hb_fill_random_dev")
    return buf


class FixedHashGraph:
    """One device-resident fixed-width hash launch captured in a CUDA graph.

    For small batches (e.g. configs[0]: 65,536 x 64 B, a few microseconds of
    GPU work) the host-side cost of a call (Python, ctypes, launch) exceeds the
    kernel time; replaying a captured graph submits the same kernel with one
    driver call.  ``msgs`` / ``out`` are bound at capture time (their device
    addresses are baked into the graph): refill ``msgs`` in place between
    replays.  ``kernels_per_replay`` is the number of engine kernels in the
    graph (the process-wide ``launch_count`` only counts them at capture)."""

    def __init__(self, alg: str, msgs, out=None, flags: int = 0, repeats: int = 1):
        """``repeats`` > 1 captures that many back-to-back passes over the batch
        in the one graph (a launch-bound loop of small batches).  ``msgs`` may
        also be a list of same-shape batches: each repeat then makes one pass
        over every batch in order (rotating inputs, e.g. to keep them out of L2)."""
        import torch

        batches = list(msgs) if isinstance(msgs, (list, tuple)) else [msgs]
        first = batches[0]
        if any(b.shape != first.shape for b in batches):
            raise ValueError("all batches of a FixedHashGraph must have the same shape")
        if out is None:
            out = torch.empty((first.shape[0], DIGEST_LEN[alg]), dtype=torch.uint8, device=first.device)
        self.alg, self.msgs, self.out, self.flags = alg, first, out, flags
        side = torch.cuda.Stream(device=first.device)
        side.wait_stream(torch.cuda.current_stream(first.device))
        with torch.cuda.stream(side):  # warm-up outside capture: one-time attribute setup, tensor-map encoder
            hash_fixed(alg, first, out=out, flags=flags)
        torch.cuda.current_stream(first.device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        before = _native.launch_count()
        with torch.cuda.graph(self.graph):
            for _ in range(max(1, int(repeats))):
                for b in batches:
                    hash_fixed(alg, b, out=out, flags=flags)
        self.kernels_per_replay = _native.launch_count() - before
        self.repeats = max(1, int(repeats))
        self.passes = self.repeats * len(batches)

    def replay(self):
        self.graph.replay()
        return self.out


def bind_host_to_gpu(ordinal: int):
    """Restrict this process's CPU affinity to the cores NVML reports as local
    to CUDA device ``ordinal`` (its NUMA node) and return them, or None when
    NVML cannot say.  Call it before allocating pinned host buffers: the
    driver first-touches page-locked memory from the calling thread, so the
    buffers -- and the engine's host staging threads, which inherit the mask --
    then sit next to the GPU's PCIe root instead of across the socket link.
    One process per GPU (``bench.py`` under torchrun) calls it for its own GPU.
    """
    import os

    try:
        import pynvml
        import torch

        uuid = str(torch.cuda.get_device_properties(ordinal).uuid).lower().removeprefix("gpu-")
        pynvml.nvmlInit()
        try:
            for i in range(pynvml.nvmlDeviceGetCount()):
                h = pynvml.nvmlDeviceGetHandleByIndex(i)
                u = pynvml.nvmlDeviceGetUUID(h)
                u = (u.decode() if isinstance(u, bytes) else u).lower().removeprefix("gpu-")
                if u != uuid:
                    continue
                words = ((os.cpu_count() or 1) + 63) // 64
                masks = pynvml.nvmlDeviceGetCpuAffinity(h, words)
                allowed = os.sched_getaffinity(0)
                cores = sorted(64 * w + b for w, m in enumerate(masks) for b in range(64)
                               if (m >> b) & 1 and 64 * w + b in allowed)
                if not cores:
                    return None
                os.sched_setaffinity(0, cores)
                return cores
        finally:
            pynvml.nvmlShutdown()
    except Exception:  # no NVML / no GPU / unsupported: leave the affinity alone
        return None
    return None
