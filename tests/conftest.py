import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


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


def load_npz(name):
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    out = {}
    for k in z.files:
        if "__" in k:
            case, field = k.split("__", 1)
            out.setdefault(case, {})[field] = z[k]
        else:
            out[k] = z[k]
    return out


@pytest.fixture(scope="session")
def golden_kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_minmax():
    return load_npz("minmax.npz")


@pytest.fixture(scope="session")
def golden_search():
    arrays = load_npz("search.npz")
    with open(os.path.join(GOLDEN, "search.json")) as f:
        meta = json.load(f)
    cases = {}
    for name, m in meta.items():
        cases[name] = dict(sigs=arrays[m["sigs"]], trip=arrays[name]["trip"],
                           cfg=m["cfg"], stats=m["stats"])
    return cases


@pytest.fixture(scope="session")
def golden_fingerprint():
    return load_npz("fingerprint.npz")
