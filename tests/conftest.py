import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


def has_gpu() -> bool:
    try:
        from paper_2509_22462_b200 import device_count
        return device_count() > 0
    except Exception:
        return False
