import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


@pytest.fixture(scope="session")
def ph():
    import paper_2511_03109_b200 as mod

    mod.lib()
    return mod


@pytest.fixture(scope="session")
def po():
    from oracle import pyoracle

    pyoracle.lib()
    return pyoracle


@pytest.fixture(scope="session")
def pr():
    """The compiled reference (oracle/_ref/libphmat_ref.so, test infrastructure)."""
    from oracle import pyref

    pyref.lib()
    return pyref


PARITY = {}


@pytest.fixture(scope="session")
def parity_log():
    """Records worst relative errors per test (dumped to $PHM_PARITY_REPORT)."""

    def log(test, key, value):
        rec = PARITY.setdefault(test, {})
        rec[key] = max(float(value), rec.get(key, 0.0))

    return log


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("PHM_PARITY_REPORT")
    if path and PARITY:
        import json

        with open(path, "w") as f:
            json.dump(PARITY, f, indent=1, sort_keys=True)
