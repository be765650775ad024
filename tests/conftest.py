import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs via gpurun")
    config.addinivalue_line("markers", "slow: long-running oracle check (skipped by default on CPU)")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("LORPC_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow; set LORPC_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)
