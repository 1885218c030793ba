import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running case")


@pytest.fixture(scope="session")
def port():
    import oracle as O
    return O.get("port")


@pytest.fixture(scope="session")
def ref():
    import oracle as O
    if not O.reference_available():
        pytest.skip("oracle/_ref (reference oracle built from /root/reference) not present")
    return O.get("reference")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


# ---- the reference's comparison metrics (proj/tests/test_util.hpp:23-93) -------------
def max_component_rel(a, b):
    a, b = np.asarray(a, float).ravel(), np.asarray(b, float).ravel()
    den = np.maximum(np.abs(a), np.abs(b))
    if np.any((den == 0) & (a != b)):
        return 1.0
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.where(den > 0, np.abs(a - b) / np.where(den > 0, den, 1.0), 0.0)
    return float(r.max()) if r.size else 0.0


def max_rel_vs_peak(a, b):
    a, b = np.asarray(a, float).ravel(), np.asarray(b, float).ravel()
    peak = max(np.abs(a).max(), np.abs(b).max())
    diff = np.abs(a - b).max()
    return float(diff / peak) if peak > 0 else float(diff)


def max_rel_global_floor(a, b, floor_frac=1e-2):
    a, b = np.asarray(a, float), np.asarray(b, float)
    scale = max(np.abs(a).max(), np.abs(b).max())
    if scale == 0:
        return 0.0
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor_frac * scale)
    return float((np.abs(a - b) / den).max())


def max_rowwise_rel(a, b, row_floor=1e-2):
    a, b = np.asarray(a, float), np.asarray(b, float)
    if a.ndim == 1:
        a, b = a[:, None], b[:, None]
    rs = np.maximum(np.abs(a).max(axis=1), np.abs(b).max(axis=1))[:, None]
    keep = rs[:, 0] > 0
    if not keep.any():
        return 0.0
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), row_floor * rs)
    return float((np.abs(a - b)[keep] / den[keep]).max())


def max_log_rel(a, b):
    """BASELINE.json tolerance metric: max_j |log a_j - log b_j| / |log b_j|."""
    la, lb = np.log(np.asarray(a, float)), np.log(np.asarray(b, float))
    return float(np.max(np.abs(la - lb) / np.abs(lb)))
