import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) — parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda_ok():
    if not has_cuda():  # -m gpu runs only on a B200 box: a missing device is a failure
        pytest.fail("no CUDA device visible to a gpu-marked test")
    return True
