"""Workload runs through the lowering + executor (the reference's
``run_point`` flow, ``pkg/src/hetoc/scheduler/sweep.py:51-72``, on GPUs).

The reference sweeps the host/accelerator duty ratio; the B200 runtime has no
CPU hash path, so the split here is between GPUs (``ratios`` over
``devices.accels``, default equal shares -- the multi-GPU task splitting of
``hyper.for``).  Message bytes are the paper's workload, ``gen_messages``
(``pkg/src/hetoc/crypto/batch.py:86-99``; ``scheduler/workload.py:12-25``).
"""

from __future__ import annotations

from dataclasses import dataclass

from ..crypto.batch import DIGEST_LEN, gen_messages
from .devices import DeviceTable
from .executor import execute_batched
from .lowering import lower_hash_batch


@dataclass(frozen=True)
class Workload:  # scheduler/workload.py:12-25
    alg: str
    count: int
    width: int = 9

    def __post_init__(self):
        if self.alg not in DIGEST_LEN:
            raise ValueError(f"unknown algorithm {self.alg!r}")
        if self.count < 0 or self.width <= 0:
            raise ValueError("count must be >= 0 and width > 0")

    def message_bytes(self) -> bytes:
        return gen_messages(0, self.count, self.width).data


@dataclass
class RunRecord:
    ratios: tuple[float, ...]
    wall_s: float
    accel_s: dict
    batches: dict
    n_data: int
    alg: str
    digests: bytes = b""


def run_point(workload: Workload, devices: DeviceTable, ratios=None, *, message_bytes: bytes | None = None,
              keep_digests: bool = False) -> RunRecord:
    """Lower ``crypto.hash_batch`` over ``workload`` onto ``devices.accels``
    with ``ratios`` and execute it batched; times are device-measured."""
    accels = [a.id for a in devices.accels]
    if not accels:
        raise ValueError("no GPU in the device table")
    ratios = tuple(ratios) if ratios is not None else tuple(1.0 / len(accels) for _ in accels)
    if len(ratios) != len(accels):
        raise ValueError(f"{len(ratios)} ratios for {len(accels)} GPUs")
    prog = lower_hash_batch(workload.alg, workload.count, workload.width, list(zip(accels, ratios)), devices)
    msgs = message_bytes if message_bytes is not None else workload.message_bytes()
    rep = execute_batched(prog, devices, {"msgs": msgs})
    return RunRecord(ratios, rep.max_wall(), {a: rep.wall_time[a] for a in accels},
                     {a: rep.batch_count[a] for a in accels}, workload.count, workload.alg,
                     rep.outputs["out"] if keep_digests else b"")
