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
