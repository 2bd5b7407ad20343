import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the built libdcp_b200.so")


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly (no silent skip) when selected with -m gpu on a box
    # without a GPU; CPU runs (-m "not gpu") never collect them.
    pass
