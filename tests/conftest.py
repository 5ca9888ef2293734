import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size parity cases")


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    if not os.path.exists(os.path.join(oracle.HERE, "liboracle.so")):
        oracle.build(ref=False)
    return oracle.Oracle()


@pytest.fixture(scope="session")
def reference_lib():
    import oracle
    if not oracle.Reference.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle.Reference()


@pytest.fixture(scope="session")
def reference_lib_optional():
    """The threaded reference when built (fast), else the C oracle."""
    import oracle
    if oracle.Reference.available():
        ref = oracle.Reference()

        class _R:
            def nn1(self, q, db, w):
                return ref.nn1_threads(q, db, w, threads=os.cpu_count() or 1)
        return _R()
    return oracle.Oracle()
