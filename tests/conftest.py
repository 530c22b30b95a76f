import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device); runs through the C ABI")
    config.addinivalue_line("markers", "slow: larger CPU cases (still minutes at most)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        return json.load(f)


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
