"""Device table of the B200 runtime: the host plus one ``cuda`` entry per GPU.

Mirrors the reference's ``DeviceSpec`` / ``DeviceTable`` / ``detect_hardware``
(``pkg/src/hetoc/runtime/devices.py:36-184``) with one new kind, ``cuda``
(SURVEY.md §8(f) row 1): a real GPU addressed by ``ordinal``.  Its
``mem_bytes`` is the launch-group capacity the executor sub-batches against
(``executor.py:603-699``); the default is 45 % of the GPU's HBM so that two
sub-batches (the copy/compute ping-pong) fit at once.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

HOST_ID = "host"
_KINDS = ("host", "cuda")


class DeviceConfigError(ValueError):
    pass


@dataclass(frozen=True)
class DeviceSpec:
    id: str
    kind: str = "cuda"
    ordinal: int = 0
    threads: int = 1
    mem_bytes: int = 1 << 62
    sha_accel: bool = False
    host_mapped: bool = False

    def __post_init__(self):
        bad = [what for ok, what in (
            (bool(self.id), "empty id"),
            (self.kind in _KINDS, f"kind {self.kind!r} not in {_KINDS}"),
            (self.threads >= 1, f"threads={self.threads} (need at least one)"),
            (self.mem_bytes > 0, f"mem_bytes={self.mem_bytes} (need a positive capacity)"),
            (self.kind != "cuda" or self.ordinal >= 0, f"ordinal={self.ordinal} (need a GPU index)"),
        ) if not ok]
        if bad:
            raise DeviceConfigError(f"bad device spec {self.id!r}: {', '.join(bad)}")


@dataclass(frozen=True)
class DeviceTable:
    host: DeviceSpec
    accels: tuple[DeviceSpec, ...] = ()

    def __post_init__(self):
        if self.host.kind != "host":
            raise DeviceConfigError(f"table host {self.host.id!r} is of kind {self.host.kind!r}, expected 'host'")
        seen = set()
        for d in self.all_devices():
            if d.id in seen:
                raise DeviceConfigError(f"device id {d.id!r} appears more than once")
            seen.add(d.id)
        wrong = [a.id for a in self.accels if a.kind != "cuda"]
        if wrong:
            raise DeviceConfigError(f"accelerators {wrong} are not GPUs (kind 'cuda')")

    def all_devices(self) -> tuple[DeviceSpec, ...]:
        return (self.host, *self.accels)

    def get(self, device_id: str) -> DeviceSpec | None:
        for d in self.all_devices():
            if d.id == device_id:
                return d
        return None

    def resolve(self, device_id: str) -> DeviceSpec:
        found = self.get(device_id)
        if found is None:
            raise DeviceConfigError(f"no device {device_id!r} in this table")
        return found

    def is_host_mapped(self, device_id: str) -> bool:
        d = self.resolve(device_id)
        return d.kind == "host" or d.host_mapped


def detect_hardware(mem_fraction: float = 0.45) -> DeviceTable:
    """Host (``os.cpu_count()`` threads, as devices.py:115) plus every visible
    GPU as ``gpu<i>`` (kind ``cuda``, ordinal i)."""
    from .. import _native

    host = DeviceSpec(HOST_ID, kind="host", threads=os.cpu_count() or 1)
    accels = []
    for i in range(_native.device_count()):
        info = _native.device_info(i)
        accels.append(DeviceSpec(f"gpu{i}", kind="cuda", ordinal=i,
                                 mem_bytes=max(1, int(info["total_mem"] * mem_fraction))))
    return DeviceTable(host, tuple(accels))


def from_reference(table, ordinals: dict | None = None) -> DeviceTable:
    """Map a reference ``DeviceTable`` (``devices.py:72-98``; duck-typed) onto
    GPUs: every non-host-mapped accelerator becomes a ``cuda`` device, by
    default on ordinal i for the i-th accelerator (``ordinals`` overrides by
    id), keeping its ``mem_bytes`` capacity so sub-batching is unchanged."""
    ordinals = dict(ordinals or {})
    host = DeviceSpec(table.host.id, kind="host", threads=table.host.threads, mem_bytes=table.host.mem_bytes,
                      sha_accel=bool(getattr(table.host, "sha_accel", False)))
    accels = []
    for i, a in enumerate(table.accels):
        if getattr(a, "host_mapped", False):
            raise DeviceConfigError(f"accelerator {a.id!r} is host-mapped; the B200 runtime has no CPU hash path")
        accels.append(DeviceSpec(a.id, kind="cuda", ordinal=int(ordinals.get(a.id, i)), threads=a.threads,
                                 mem_bytes=a.mem_bytes, sha_accel=bool(getattr(a, "sha_accel", False))))
    return DeviceTable(host, tuple(accels))
