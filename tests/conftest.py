import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "ab: exercises an A/B kernel arm; needs the -DHB_AB library "
                                       "(HETOC_B200_LIB=libhetoc_b200_ab.so, `make -C paper_2407_09333_b200/csrc ab`)")
    config.addinivalue_line("markers", "zero_copy: test_gpu_parity runs it with the small-call zero-copy path at "
                                       "its default (every other test there pins $HB_ZERO_COPY_MAX=0)")


def _gpu_visible() -> bool:
    try:
        from paper_2407_09333_b200 import _native

        return _native.device_count() > 0
    except Exception:
        return False


def _ab_library() -> bool:
    try:
        from paper_2407_09333_b200 import _native

        return _native.built_with_ab()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    """`gpu` tests skip (not fail) where no CUDA device is visible, so a plain
    `pytest` passes on a CPU box; `ab` tests skip unless the loaded library was
    built with the A/B kernel arms."""
    need_gpu = [it for it in items if "gpu" in it.keywords]
    if need_gpu and not _gpu_visible():
        skip = pytest.mark.skip(reason="no CUDA device visible")
        for it in need_gpu:
            it.add_marker(skip)
    need_ab = [it for it in items if "ab" in it.keywords]
    if need_ab and not _ab_library():
        skip = pytest.mark.skip(reason="A/B kernel arms not built (default library)")
        for it in need_ab:
            it.add_marker(skip)


def load_golden(name):
    import json

    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden():
    return load_golden


class _HbEnv:
    """$HB_* tuning knobs for one test: the library parses them once, so every
    change is followed by hb_tuning_reload(); teardown restores the
    environment and reloads again."""

    def __init__(self, mp):
        self.mp = mp

    def _reload(self):
        from paper_2407_09333_b200 import _native

        _native.reload_tuning()

    def set(self, **kv):
        for k, v in kv.items():
            self.mp.setenv(k, str(v))
        self._reload()

    def clear(self, *keys):
        for k in keys:
            self.mp.delenv(k, raising=False)
        self._reload()

    def reset(self, keys, **kv):
        for k in keys:
            self.mp.delenv(k, raising=False)
        self.set(**kv)


@pytest.fixture
def hb_env(monkeypatch):
    env = _HbEnv(monkeypatch)
    yield env
    monkeypatch.undo()
    env._reload()
