"""Test configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` runs here (no GPU): oracle vs golden fixtures, ABI exports,
host logic and the 2-rank gloo engine test.  `-m gpu` runs on a B200 and
calls the CUDA path through the C-ABI; those tests compare against the CPU
oracle (oracle/) and the committed golden fixtures (tests/golden/).
"""
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer-running parity case")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_cs():
    return np.load(os.path.join(GOLDEN, "countsketch_small.npz"))


def small_cs_cases(z):
    i = 0
    out = []
    while f"cs{i}_cols" in z:
        n, r, s, seed = [int(x) for x in z[f"cs{i}_params"]]
        out.append((i, n, r, s, seed))
        i += 1
    return out
