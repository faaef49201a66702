import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running full-size case")


def pytest_collection_modifyitems(config, items):
    """Full-size cases last, grouped by config (each 1.6-32 GB instance is generated once):
    the fast parity suite runs first."""
    def key(it):
        if "test_gpu_fullsize" not in it.nodeid:
            return (0, 0, 0)
        cs = getattr(it, "callspec", None)
        idx = cs.params.get("idx", 0) if cs else 0
        return (1, idx, 0)
    items.sort(key=key)  # stable: original order inside each group
