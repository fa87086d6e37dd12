"""§8(f) row 4: the duty-ratio model and its calibration
(paper_2407_09333_b200.scheduler) against the reference's own functions --
through the committed golden (tests/golden/scheduler_model.json, made by
running hetoc.scheduler.model in tests/golden/make_golden.py) everywhere, and
directly against the reference when it is importable (authoring container)."""
import math
import os
import random
import sys

import pytest

from paper_2407_09333_b200.scheduler import PerfModel, fit_model, predict_opt_ratio, t_cpu, t_gpu, t_opt

REF_SRC = "/root/reference/pkg/src"
FIELDS = ("p_cpu", "n_core", "p_gpu_over_nthread", "t_alloc", "t_memcpy", "o_gpu")


def close(a, b):
    return math.isclose(a, b, rel_tol=1e-12, abs_tol=1e-300)


def test_golden_fits_and_predictions(golden):
    for row in golden("scheduler_model.json"):
        if "cpu" in row:
            m = fit_model([tuple(x) for x in row["cpu"]], [tuple(x) for x in row["dev"]], row["n_core"])
        else:
            m = PerfModel(**row["model"])
        for k in FIELDS:
            assert close(getattr(m, k), row["model"][k]), (k, getattr(m, k), row["model"][k])
        if row["opt_ratio"] is None:
            with pytest.raises(ValueError):
                predict_opt_ratio(m, 1000)
        else:
            for n, x in row["opt_ratio"].items():
                assert close(predict_opt_ratio(m, int(n)), x)
        for key, v in row["t_opt"].items():
            n, x = key.split(":")
            assert close(t_opt(m, int(n), float(x)), v)


def test_model_properties():
    m = PerfModel(p_cpu=1e-6, n_core=8, p_gpu_over_nthread=1e-9, t_alloc=0.0, t_memcpy=2e-8, o_gpu=5e-4)
    n = 10**7
    x = predict_opt_ratio(m, n)
    assert 0 <= x <= 1
    assert math.isclose(t_cpu(m, n, x), t_gpu(m, n, x), rel_tol=1e-9)  # the lines cross at x*
    assert t_opt(m, n, x) <= min(t_opt(m, n, 0.0), t_opt(m, n, 1.0)) + 1e-15
    with pytest.raises(ValueError):
        PerfModel(p_cpu=-1, n_core=1, p_gpu_over_nthread=0, t_alloc=0, t_memcpy=0, o_gpu=0)
    with pytest.raises(ValueError):
        PerfModel(p_cpu=1, n_core=0, p_gpu_over_nthread=0, t_alloc=0, t_memcpy=0, o_gpu=0)
    with pytest.raises(ValueError):
        fit_model([(10, 1.0)], [(10, 1.0), (20, 2.0)], 4)
    with pytest.raises(ValueError):
        fit_model([(10, 1.0), (10, 2.0)], [(10, 1.0), (20, 2.0)], 4)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present (authoring container only)")
def test_against_reference_directly():
    sys.path.insert(0, REF_SRC)
    try:
        from hetoc.scheduler import model as ref
    finally:
        sys.path.remove(REF_SRC)
    rnd = random.Random(3)
    for _ in range(200):
        cpu = [(rnd.randint(1, 10**8), rnd.uniform(1e-4, 100.0)) for _ in range(rnd.randint(2, 8))]
        dev = [(rnd.randint(1, 10**8), rnd.uniform(1e-5, 10.0)) for _ in range(rnd.randint(2, 8))]
        if len({n for n, _ in cpu}) < 2 or len({n for n, _ in dev}) < 2:
            continue
        cores = rnd.randint(1, 512)
        a, b = fit_model(cpu, dev, cores), ref.fit_model(cpu, dev, cores)
        for k in FIELDS:
            assert close(getattr(a, k), getattr(b, k)), k
        for n in (1, 10**4, 10**9):
            try:
                want = ref.predict_opt_ratio(b, n)
            except ValueError:
                with pytest.raises(ValueError):
                    predict_opt_ratio(a, n)
                continue
            assert close(predict_opt_ratio(a, n), want)
            for x in (0.0, 0.3, 1.0):
                assert close(t_opt(a, n, x), ref.t_opt(b, n, x))


@pytest.mark.gpu
def test_device_samples_calibrate():
    """B200 device-only samples through the engine fit a non-negative model
    whose accelerator term predicts the measured times."""
    from paper_2407_09333_b200.scheduler import device_samples

    dev = device_samples("md5", 1024, [1 << 14, 1 << 16, 1 << 18], gpus=[0])
    assert all(t > 0 for _, t in dev)
    m = fit_model([(1000, 1.0), (2000, 2.0)], dev, 16)
    assert m.p_gpu_over_nthread > 0
    n, t = dev[-1]
    assert math.isclose(t_gpu(m, n, 0.0), t, rel_tol=0.5)
