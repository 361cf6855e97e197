"""OSPA (p = 1, c = 100): Hungarian implementation vs the plain
definition (minimum over all permutations) on small random sets, plus closed cases."""
import itertools
import math

import numpy as np

from paper_1503_03769_b200.metrics import ospa


def ospa_brute(X, Y, c=100.0, p=1.0):
    X = np.asarray(X, float).reshape(-1, 2)
    Y = np.asarray(Y, float).reshape(-1, 2)
    m, n = len(X), len(Y)
    if m == 0 and n == 0:
        return 0.0
    if m > n:
        X, Y, m, n = Y, X, n, m
    if m == 0:
        return c
    best = math.inf
    for perm in itertools.permutations(range(n), m):
        s = sum(min(c, float(np.linalg.norm(X[i] - Y[perm[i]]))) ** p for i in range(m))
        best = min(best, s)
    return ((best + c ** p * (n - m)) / n) ** (1 / p)


def test_ospa_matches_brute_force():
    rng = np.random.default_rng(0)
    for _ in range(200):
        m, n = int(rng.integers(0, 6)), int(rng.integers(0, 6))
        X = rng.uniform(0, 300, (m, 2))
        Y = rng.uniform(0, 300, (n, 2))
        for p in (1.0, 2.0):
            assert abs(ospa(X, Y, 100.0, p) - ospa_brute(X, Y, 100.0, p)) < 1e-9


def test_ospa_closed_cases():
    assert ospa([], []) == 0.0
    assert ospa([[0, 0]], []) == 100.0
    assert ospa([[0, 0]], [[3, 4]]) == 5.0                     # one pair, distance 5
    assert ospa([[0, 0]], [[300, 0]]) == 100.0                 # cut-off c
    assert abs(ospa([[0, 0]], [[3, 4], [50, 50]]) - (5 + 100) / 2) < 1e-12  # cardinality penalty
    assert ospa([[1, 2], [5, 5]], [[5, 5], [1, 2]]) == 0.0      # order-free
