import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI path)")
    config.addinivalue_line("markers", "gpu2: needs two GPUs (NVLink pair)")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    for item in items:
        if "gpu2" in item.keywords and "gpu" not in item.keywords:
            item.add_marker(pytest.mark.gpu)
