"""VEC oracle, serial fp64 (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

PAPER.md §V-B: "computes the sum of differences of 2 squared
vectors"; Fig. 4 code L431-441 (square kernels, then a sum over X, Y into Z).
Out-of-place squares (x1, y1) follow Table I's footprint.

Pins (tests/test_oracle_vec.py): closed form z = -3*H_N^(2) for
x_i = 1/(i+1), y_i = 2/(i+1) against scipy.special.polygamma; exact squares of
small integers.
"""
import numpy as np


def square(x):
    """K1 (L431, L438-439): x1[i] = x[i]^2."""
    x = np.asarray(x, dtype=np.float64)
    return x * x


def reduce_diff(x1, y1):
    """K2 (L432-433, L440, Fig. 6 "SUM(X-Y)" L680): z = sum_i (x1[i] - y1[i])."""
    d = np.asarray(x1, dtype=np.float64) - np.asarray(y1, dtype=np.float64)
    return float(np.sum(d))


def vec(x, y):
    """Whole VEC DAG in program order: X2, Y2, then SUM(X-Y)."""
    x1 = square(x)
    y1 = square(y)
    return x1, y1, reduce_diff(x1, y1)
