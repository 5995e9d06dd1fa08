import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running test")
    # the tests always run against the current sources: (re)build libpa.so when it is missing
    # or older than any source (nvcc cross-compiles on CPU hosts too; no-op when fresh)
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "pa_build", os.path.join(ROOT, "paper_1805_02372_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build()


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
