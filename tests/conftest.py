import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_sessionstart(session):
    # libkvd.so and liboracle.so are build artefacts (git-ignored); build them
    # in-tree before collection imports the binding (nvcc cross-compiles here).
    from paper_2501_14743_b200 import build
    from oracle import oracle
    build.build()
    oracle.build()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI path)")
    config.addinivalue_line("markers", "gpu2: needs two GPUs (NVLink pair)")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    for item in items:
        if "gpu2" in item.keywords and "gpu" not in item.keywords:
            item.add_marker(pytest.mark.gpu)
