"""Duty-ratio calibration: the paper's two-device
performance model (Eq. 1-3) fitted to measured B200 engine times.

Same API and arithmetic as the reference's ``hetoc.scheduler.model``
(``pkg/src/hetoc/scheduler/model.py:20-119``): a host share ``x`` of ``n``
messages costs ``n * p_cpu * x / n_core`` seconds on the host; the rest costs
``n * (1 - x) * (p_gpu_over_nthread + t_alloc + t_memcpy) + o_gpu`` on the
accelerator; a split runs as long as the slower side, and the best split is
where the two lines cross.  ``fit_model`` calibrates it from (n, seconds)
samples: host runs through the origin, device runs with an intercept.

This module only models and fits.  There is no CPU hash path in the product
(the north star excludes CPU co-execution): host-side samples come from
whoever measures a CPU implementation -- ``bench.py`` times the oracle port
of the reference algorithm -- and :func:`device_samples` measures the B200
side through the engine (H2D + kernel + D2H per call, the accelerator term of
the model).
"""

from __future__ import annotations

import logging
import time
from dataclasses import dataclass

import numpy as np

log = logging.getLogger(__name__)

_NONNEG = ("p_cpu", "p_gpu_over_nthread", "t_alloc", "t_memcpy", "o_gpu")


@dataclass(frozen=True)
class PerfModel:
    """Per-message costs in seconds (``model.py:20-38``)."""

    p_cpu: float  # one host core, per message
    n_core: int
    p_gpu_over_nthread: float  # accelerator compute, per message (aggregate)
    t_alloc: float  # accelerator allocation, per message
    t_memcpy: float  # host <-> accelerator transfer, per message
    o_gpu: float  # fixed accelerator cost per run

    def __post_init__(self):
        if self.n_core < 1:
            raise ValueError("n_core must be >= 1")
        bad = [k for k in _NONNEG if getattr(self, k) < 0]
        if bad:
            raise ValueError(f"{bad[0]} must be >= 0")

    @property
    def accel_per_message(self) -> float:
        return self.p_gpu_over_nthread + self.t_alloc + self.t_memcpy


def t_cpu(model: PerfModel, n_data: int, x: float) -> float:
    """Eq. 1: host seconds for host share x."""
    return x * n_data * model.p_cpu / model.n_core


def t_gpu(model: PerfModel, n_data: int, x: float) -> float:
    """Eq. 2: accelerator seconds for the share 1 - x."""
    return (1.0 - x) * n_data * model.accel_per_message + model.o_gpu


def t_opt(model: PerfModel, n_data: int, x: float) -> float:
    """Eq. 3: the split's run time, max of the two sides."""
    return max(t_cpu(model, n_data, x), t_gpu(model, n_data, x))


def predict_opt_ratio(model: PerfModel, n_data: int) -> float:
    """Host share at which Eq. 1 and Eq. 2 meet, clamped to [0, 1]:
    x* = (B + o_gpu) / (A + B), A / B the full-load host / accelerator times."""
    host_full = n_data * model.p_cpu / model.n_core
    accel_full = n_data * model.accel_per_message
    denom = host_full + accel_full
    if denom == 0:
        raise ValueError("model has no workload-dependent terms; optimum undefined")
    return float(np.clip((accel_full + model.o_gpu) / denom, 0.0, 1.0))


def _samples(samples, what: str) -> tuple[np.ndarray, np.ndarray]:
    arr = np.asarray(samples, dtype=np.float64).reshape(-1, 2)
    if arr.shape[0] < 2:
        raise ValueError(f"need at least 2 {what} samples")
    if np.unique(arr[:, 0]).size < 2:
        raise ValueError(f"{what} samples must cover at least 2 distinct sizes")
    return arr[:, 0], arr[:, 1]


def fit_model(cpu_samples, dev_samples, n_core: int) -> PerfModel:
    """Least-squares calibration (``model.py:74-119``): host samples (full-load
    host-only runs) through the origin, device samples (device-only runs in
    one batch regime) with slope and intercept; the host slope times n_core
    is p_cpu, the device slope goes to p_gpu_over_nthread, the intercept to
    o_gpu; a negative estimate is clamped to 0 (and logged)."""
    cn, ct = _samples(cpu_samples, "cpu")
    dn, dt = _samples(dev_samples, "device")
    host_slope = float(cn @ ct) / float(cn @ cn)
    dn_c = dn - dn.mean()
    dev_slope = float(dn_c @ (dt - dt.mean())) / float(dn_c @ dn_c)
    fitted = {"p_cpu": host_slope * n_core, "device slope": dev_slope, "o_gpu": float(dt.mean()) - dev_slope * dn.mean()}
    neg = [k for k, v in fitted.items() if v < 0]
    if neg:
        log.warning("fit produced negative %s; clamped to 0", ", ".join(neg))
    f = {k: max(0.0, v) for k, v in fitted.items()}
    return PerfModel(p_cpu=f["p_cpu"], n_core=n_core, p_gpu_over_nthread=f["device slope"], t_alloc=0.0,
                     t_memcpy=0.0, o_gpu=f["o_gpu"])


def device_samples(alg: str, msg_len: int, sizes, gpus=None, repeats: int = 3, seed: int = 0):
    """(n, seconds) of device-only runs through the engine: the drop-in
    ``batch_digest`` on page-locked host rows (H2D, kernel, D2H per call),
    best of ``repeats`` after one warm-up call per size."""
    import ctypes

    from . import _native
    from .crypto.batch import batch_digest

    lib = _native.lib()
    out = []
    rng = np.random.default_rng(seed)
    for n in sizes:
        n = int(n)
        p = lib.hb_alloc_pinned(max(1, n * msg_len))
        if not p:
            raise MemoryError(_native.last_error())
        try:
            rows = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_uint8)),
                                         shape=(max(1, n * msg_len),))[: n * msg_len].reshape(n, msg_len)
            rows[:] = rng.integers(0, 256, rows.shape, dtype=np.uint8)
            batch_digest(alg, rows, gpus=gpus)
            best = float("inf")
            for _ in range(repeats):
                t0 = time.perf_counter()
                batch_digest(alg, rows, gpus=gpus)
                best = min(best, time.perf_counter() - t0)
            out.append((n, best))
        finally:
            lib.hb_free_pinned(p)
    return out
