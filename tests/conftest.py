import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: large-shape parity (still within the gpu tier)")


@pytest.fixture(autouse=True)
def _clear_b200_options():
    """Tuning options / test hooks (aires_b200_set_option) never leak from one test into the next."""
    yield
    mod = sys.modules.get("paper_2507_02006_b200")
    if mod is not None and getattr(mod, "_lib", None) is not None:
        mod.clear_options()
