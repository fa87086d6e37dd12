"""Workload runs through the lowering + executor (the reference's
``run_point`` / ``sweep`` flow, ``pkg/src/hetoc/scheduler/sweep.py:39-128``,
on GPUs).

The reference sweeps the host/accelerator duty ratio; the B200 runtime has no
CPU hash path, so the split here is between GPUs (``ratios`` over
``devices.accels``, default equal shares -- the multi-GPU task splitting of
``hyper.for``).  Message bytes are the paper's workload, ``gen_messages``
(``pkg/src/hetoc/crypto/batch.py:86-99``; ``scheduler/workload.py:12-25``).
"""

from __future__ import annotations

import io
import math
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
    error: str | None = None

    @property
    def ratio_first(self) -> float:
        """Duty ratio of the first GPU binding (the swept coordinate)."""
        return self.ratios[0] if self.ratios else float("nan")


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


def ratio_grid(step: float) -> list[float]:
    """{0, step, 2*step, ...} up to and always including 1 (``sweep.py:39-48``)."""
    if not 0.0 < step <= 1.0:
        raise ValueError("step must be in (0, 1]")
    xs, i = [], 0
    while i * step < 1.0 - 1e-12:
        xs.append(round(i * step, 12))
        i += 1
    xs.append(1.0)
    return xs


def split_ratios(x: float, n_accels: int) -> tuple[float, ...]:
    """Share ``x`` on the first GPU binding, ``1 - x`` spread equally over the
    others -- the GPU-to-GPU counterpart of the reference's host share
    ``ratio_cpu`` (``scheduler/workload.py:28-45``: host ``x``, accelerator
    ``1 - x``)."""
    if not 0.0 <= x <= 1.0:
        raise ValueError(f"ratio {x} outside [0, 1]")
    if n_accels < 2:
        raise ValueError("a duty-ratio sweep needs at least two GPU bindings")
    rest = (1.0 - x) / (n_accels - 1)
    return (x,) + tuple(rest for _ in range(n_accels - 1))


def sweep(workload: Workload, devices: DeviceTable, step: float = 0.02, *,
          message_bytes: bytes | None = None) -> list[RunRecord]:
    """Run ``run_point`` at every ratio of ``ratio_grid(step)`` (``sweep.py:75-99``):
    strictly sequential, one lowering per point (ratios are compile-time
    attributes), message bytes generated once; a failing point is recorded
    with ``error`` set, not fatal."""
    n_acc = len(devices.accels)
    msgs = message_bytes if message_bytes is not None else workload.message_bytes()
    records = []
    for x in ratio_grid(step):
        try:
            records.append(run_point(workload, devices, split_ratios(x, n_acc), message_bytes=msgs))
        except Exception as e:  # per-point failures are recorded, not fatal
            records.append(RunRecord(split_ratios(x, max(n_acc, 2))[:max(n_acc, 1)], float("nan"), {}, {},
                                     workload.count, workload.alg, error=str(e)))
    return records


def sweep_argmin(records: list[RunRecord]) -> RunRecord:
    """Fastest successful point (``sweep.py:102-106``)."""
    good = [r for r in records if r.error is None and not math.isnan(r.wall_s)]
    if not good:
        raise ValueError("no successful sweep points")
    return min(good, key=lambda r: r.wall_s)


CSV_COLUMNS = ("ratio_first", "wall_s", "accel_s", "batches", "n_data", "alg")


def records_to_csv(records: list[RunRecord]) -> str:
    """``sweep.py:113-124``'s CSV with the GPU split: ``accel_s`` / ``batches``
    are ``;``-joined per binding in binding order; failed points are skipped."""
    out = io.StringIO()
    out.write(",".join(CSV_COLUMNS) + "\n")
    for r in records:
        if r.error is not None:
            continue
        acc = ";".join(f"{v:.6g}" for v in r.accel_s.values())
        bat = ";".join(str(v) for v in r.batches.values())
        out.write(f"{r.ratio_first:.6g},{r.wall_s:.6g},{acc},{bat},{r.n_data},{r.alg}\n")
    return out.getvalue()
