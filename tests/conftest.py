import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture
def lib_options():
    """Set librbf options (rbf_set_option) for one test; the defaults are restored after."""
    import paper_0909_5413_b200 as P

    saved = {}

    def set_(**kw):
        for k, v in kw.items():
            if k not in saved:
                saved[k] = P.get_option(k)
            P.set_option(k, v)

    yield set_
    for k, v in saved.items():
        P.set_option(k, v)
