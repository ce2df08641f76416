"""pytest configuration: registers the `gpu` marker and puts the repo root on sys.path.

`-m "not gpu"` tests run on the CPU container (oracle pins, host logic, ABI
symbol checks); `-m gpu` tests need a B200 and call the CUDA path through the
C-ABI (`paper_2204_03418_b200`), comparing it with the fp64 oracle (`oracle/`).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


import pytest


@pytest.fixture(autouse=True)
def _reset_co_options():
    """Planner options (co_set_option) are process-wide: restore the defaults
    after every test that loaded the library."""
    yield
    from paper_2204_03418_b200 import _abi
    if _abi._lib is not None:
        _abi.check(_abi._lib.co_set_option(None, 0))
