import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: larger CPU oracle cases")


def pytest_sessionstart(session):
    # build the in-tree shared libraries once (no-op when up to date)
    subprocess.check_call(["make", "-s", "all"], cwd=ROOT, stdout=subprocess.DEVNULL)
