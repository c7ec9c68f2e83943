import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through the C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


def load_golden(name):
    """Parse a tests/golden/*.txt fixture: '# comments', then 'key: values' lines."""
    path = os.path.join(ROOT, "tests", "golden", name)
    out = {}
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, val = line.split(":", 1)
            out[key.strip()] = val.split()
    n, d, m = int(out["n"][0]), int(out["d"][0]), int(out["m"][0])
    X = np.array([float(v) for v in out["X"]], dtype=np.float32).reshape(n, d)
    Z = np.array([float(v) for v in out["Z"]], dtype=np.float32).reshape(n, m)
    Y = np.array([float(v) for v in out["Y"]], dtype=np.float64).reshape(n, m)
    return X, Z, Y


def golden_p(name):
    """The fixture's exponent p (l_p^p fixtures carry a 'p:' line; l1 fixtures are p = 1)."""
    path = os.path.join(ROOT, "tests", "golden", name)
    for line in open(path):
        if line.startswith("p:"):
            return int(line.split(":", 1)[1])
    return 1


GOLDEN = ["q1_three_points.txt", "q2_identity.txt", "q20_two_dim.txt", "q21_ties_negative.txt"]
GOLDEN_LP = ["lp3_three_points.txt", "lp5_two_dim.txt"]
GOLDEN_TV = ["tv_two_points.txt"]
GOLDEN_EVEN = ["l2sq_three_points.txt", "lp4_two_points.txt"]


def col_rel_l2(Y, Yref, floor=0.0):
    """Max over columns of ||Y[:,c]-Yref[:,c]||_2 / max(||Yref[:,c]||_2, floor).

    A column whose reference is exactly zero (and floor == 0) scores 0 if Y matches
    it exactly and inf otherwise."""
    Y = np.asarray(Y, dtype=np.float64).reshape(Yref.shape[0], -1)
    Yref = np.asarray(Yref, dtype=np.float64).reshape(Yref.shape[0], -1)
    worst = 0.0
    for c in range(Yref.shape[1]):
        num = np.linalg.norm(Y[:, c] - Yref[:, c])
        den = np.linalg.norm(Yref[:, c])
        den = max(den, floor)
        worst = max(worst, num / den if den > 0 else (0.0 if num == 0 else float("inf")))
    return worst


def q12_rows(X, count=64, seed=12):
    """SURVEY §8(c) SAMPLE rows (Q12): `count` seeded random rows plus rows 0 and n-1 and the
    points with the smallest and largest coordinate sum (the extremes of |x|, where the
    prefix sums' cancellation is largest)."""
    X = np.asarray(X)
    n = X.shape[0]
    h = X.astype(np.float64).sum(axis=1)
    r = set(np.random.default_rng(seed).integers(0, n, size=count).tolist())
    r |= {0, n - 1, int(np.argmin(h)), int(np.argmax(h))}
    return np.array(sorted(r), dtype=np.int64)
