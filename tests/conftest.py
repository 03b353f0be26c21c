import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: longer CPU cases")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


def build_product():
    """Build libxlmimo.so without importing the package (whose import loads the library)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_xl_build", os.path.join(ROOT, "paper_2503_18118_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()


# the package refuses to import without its library: make sure it is built (nvcc cross-compiles here)
if not os.path.exists(os.path.join(ROOT, "paper_2503_18118_b200", "libxlmimo.so")):
    build_product()
