"""Test configuration: the `gpu` marker, fixture paths, shared helpers.

`-m "not gpu"` runs here (no GPU): oracle vs golden fixtures, host-side
planning / mesh / dispatch logic (thread and gloo meshes on CPU tensors),
and the C-ABI library's exported symbols.  `-m gpu` runs on a B200 and
compares the CUDA path with the oracle (tests/golden + oracle/).
"""

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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libdpb200.so")


@pytest.fixture(scope="session")
def plans_golden():
    with open(os.path.join(GOLDEN, "plans.json")) as f:
        return json.load(f)


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def rel_err(got, want, floor=1e-300):
    """The reference's metric (domainpar/verify.py:55-64): max|got-want| /
    max|want|, with an optional absolute floor for all-zero references."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if want.size == 0:
        return 0.0
    scale = max(np.abs(want).max(), floor)
    return float(np.abs(got - want).max() / scale)


def to_np(t):
    import torch

    if isinstance(t, torch.Tensor):
        t = t.detach()
        if t.dtype == torch.bfloat16:
            t = t.float()
        return t.cpu().numpy()
    return np.asarray(t)


def gpu_ready():
    try:
        import torch

        if not torch.cuda.is_available():
            return False
        from paper_2605_11111_b200 import _lib

        _lib.load()
        return True
    except Exception:
        return False
