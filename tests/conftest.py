"""pytest configuration: the ``gpu`` marker and shared fixtures.

``-m "not gpu"`` runs on any CPU box (oracle pins, host logic, ABI symbol
checks, gloo multi-process tests); ``-m gpu`` needs a B200 and the built
``libstereo_b200.so``.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device and libstereo_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")) as f:
        return json.load(f)
