import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running case")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def sample_idx(n, k=257):
    """Same strided sample as oracle/gen_golden.py."""
    return (np.arange(k, dtype=np.int64) * 7919) % n


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d > 0 else 1.0)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test needs a CUDA device")
    return torch.device("cuda:0")


def kept_fp_torch(stack2d):
    """Per band (count, sum of kept flat indices, sum of (index mod 1000003)^2) of
    a [R, N] CUDA stack: the kept-position fingerprint oracle/gen_golden.py
    stores from the reference's thresholded stack."""
    import torch
    out = np.zeros((stack2d.shape[0], 3), dtype=np.int64)
    for b in range(stack2d.shape[0]):
        idx = torch.nonzero(stack2d[b]).squeeze(1)
        r = idx % 1000003
        out[b] = (idx.numel(), int(idx.sum().item()), int((r * r).sum().item()))
    return out


def golden_fan(order):
    """maxflat_fan(order) of the reference (fan_design.cpp:70-108) from the golden
    fixture, as a custom FanFilter (the fan design tool is out of scope for the
    library; the library consumes fan taps)."""
    import paper_1402_5670_b200 as P
    t = golden("maxflat_fans")[f"order{order}"]
    return P.FanFilter(np.array(t), (t.shape[0] - 1) // 2, (t.shape[1] - 1) // 2, f"dmaxflat{order}")
