import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def load_golden_buckets():
    z = np.load(os.path.join(GOLDEN, "buckets.npz"))
    cases = []
    for ci in range(int(z["n"])):
        nm = int(z[f"c{ci}_nmem"])
        mem = []
        for mi in range(nm):
            idx = tuple(int(x) for x in z[f"c{ci}_m{mi}_idx"])
            mem.append((idx, z[f"c{ci}_m{mi}_data"].reshape((2,) * len(idx))))
        ridx = tuple(int(x) for x in z[f"c{ci}_res_idx"])
        cases.append((int(z[f"c{ci}_bidx"]), mem, ridx,
                      z[f"c{ci}_res_data"].reshape((2,) * len(ridx))))
    return cases


def load_json(name):
    import json
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)
