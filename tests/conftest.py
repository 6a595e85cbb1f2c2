import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def read_golden(name):
    """Parse a tests/golden/*.txt fixture into {key: value-string} (comments dropped)."""
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, v = line.split(":", 1) if ":" in line.split()[0] else (line.split()[0], line[len(line.split()[0]):])
            out[k.strip()] = v.strip()
    return out


def labels_to_mask(s):
    """'1,2,3' (paper labels, 1-based) -> bitmask over vertex ids 0..n-1."""
    m = 0
    for x in s.split(","):
        m |= 1 << (int(x) - 1)
    return m
