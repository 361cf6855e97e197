"""Evaluation metrics for tracking quality (NEXT-3; host-side, not the hot path).

OSPA (Schuhmacher, Vo & Vo 2008), the metric the paper uses with p = 1 and
c = 100: for finite sets X = {x_1..x_m}, Y = {y_1..y_n}, m <= n,

    d_p^(c)(X, Y) = ( (1/n) ( min_pi sum_{i<=m} d^(c)(x_i, y_pi(i))^p + c^p (n - m) ) )^(1/p),

d^(c)(x, y) = min(c, ||x - y||), and d = 0 when both sets are empty.  The
optimal assignment is found with the Hungarian algorithm
(scipy.optimize.linear_sum_assignment); tests pin it against brute force over
all permutations.
"""
import numpy as np


def ospa(X, Y, c=100.0, p=1.0):
    X = np.asarray(X, dtype=np.float64).reshape(-1, 2) if len(X) else np.zeros((0, 2))
    Y = np.asarray(Y, dtype=np.float64).reshape(-1, 2) if len(Y) else np.zeros((0, 2))
    m, n = len(X), len(Y)
    if m == 0 and n == 0:
        return 0.0
    if m == 0 or n == 0:
        return float(c)
    if m > n:
        X, Y, m, n = Y, X, n, m
    from scipy.optimize import linear_sum_assignment
    D = np.minimum(c, np.linalg.norm(X[:, None, :] - Y[None, :, :], axis=2)) ** p
    r, col = linear_sum_assignment(D)
    return float(((D[r, col].sum() + (c ** p) * (n - m)) / n) ** (1.0 / p))


def positions(states):
    """(x, y) of estimate states in the paper's (x, vx, y, vy) order."""
    s = np.asarray(states, dtype=np.float64).reshape(-1, 4)
    return s[:, [0, 2]]
