import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the driver's GPU tier)")
    config.addinivalue_line("markers", "slow: long CPU test")


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


_PARITY_RECORDS = []


@pytest.fixture(scope="session")
def parity_log():
    """Flip counts and parity outcomes of the GPU parity tests (the north star: samples bit-exact
    except |u - p| < tol, "those flips are counted and reported").  Written at session end to
    gpurun_out/parity_flips.json; the committed copy is profiles/parity_r2.json."""
    yield _PARITY_RECORDS
    if _PARITY_RECORDS:
        import json
        out = os.path.join(ROOT, "gpurun_out")
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "parity_flips.json"), "w") as f:
            json.dump({"tol_flip": 1e-5, "records": _PARITY_RECORDS}, f, indent=1)
