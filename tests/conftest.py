"""Shared test helpers.

* ``gpu`` marker: tests that need a B200 (run with ``-m gpu`` on the GPU box).
* ``relative_error`` mirrors the reference's helper (pkg/tests/conftest.py:42-46).
* ``golden(name)`` loads vectors produced by the reference (tests/golden/make_golden.py).
"""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")

# parity tolerances (north_star): complex128 1e-10, complex64 1e-5
TOL = {"c128": 1e-10, "c64": 1e-5}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


def relative_error(a, b, floor=1e-8):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return float(np.max(np.abs(a - b) / scale))


def normwise_error(a, b, floor=1e-300):
    """‖a − b‖∞ / max(‖b‖∞, floor) — the c64 gradient criterion (elementwise
    relative error of near-zero gradient entries is ill-conditioned in float32)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), floor))


def parity_log(name, **errs):
    """Append measured parity errors to $PARITY_LOG (JSON lines) when set —
    the evidence behind the tolerances stated in DESIGN.md §4."""
    path = os.environ.get("PARITY_LOG")
    if path:
        import json
        with open(path, "a") as f:
            f.write(json.dumps({"case": name, **{k: float(v) for k, v in errs.items()}}) + "\n")


def golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden file {name}.npz not generated")
    return dict(np.load(path))


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
