"""Pins of the oracle's t = 0 population (orc_init_population; "t=0:
Generate M particles for each group ... same weights omega_0 = 1/M", reading S23 of
SURVEY.md §8(c): y-stratified over the box, x uniform, v uniform in [-v_max, v_max]^2,
total mass m0, optionally only inside a mass box), -m "not gpu".

Sources of truth other than the oracle's own code: the stratification is checked
against exact rational stratum bounds, the uniform draws by KS tests against scipy's
uniform cdf, the noise words against ATen's independent Philox (stream 5, step 0), the
weights against the stated mass invariants.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from scenario.configs import Model, POSITION
from test_oracle_pins import aten_kat  # noqa: F401  (fixture)

M0 = Model(meas=POSITION, seed=11)
BOX = (-1000.0, 1000.0, -1000.0, 1000.0)


def test_init_stratified_in_y(orc):
    """Particle g lies in stratum g of [y0, y1) (up to the fp32 rounding of y), one per stratum."""
    n = 10007
    soa, w, _ = orc.init_population(M0, n, BOX, 20.0, 3.0)
    y = soa[2]
    for g in [0, 1, 2, 5000, n - 2, n - 1] + list(range(17, n, 997)):
        lo = Fraction(-1000) + Fraction(2000) * g / n
        hi = Fraction(-1000) + Fraction(2000) * (g + 1) / n
        ulp = Fraction(math.ulp(np.float32(abs(float(lo)) + 1.0)))  # fp32 spacing near the bound
        assert lo - ulp <= Fraction(float(y[g])) <= hi + ulp, g
    # monotone (strata are ordered) and inside the box
    assert np.all(np.diff(y) >= 0) and y[0] >= -1000.0 and y[-1] <= 1000.0


def test_init_draws_are_uniform_and_independent(orc):
    from scipy import stats
    n = 40000
    soa, _, _ = orc.init_population(M0, n, (-500.0, 1500.0, 0.0, 1000.0), 12.5, 1.0)
    x, vx, y, vy = soa
    off = (y - 0.0) * n / 1000.0 - np.arange(n)  # position inside its stratum, U(0,1)
    assert stats.kstest(off, "uniform").pvalue > 1e-3
    assert stats.kstest((x + 500.0) / 2000.0, "uniform").pvalue > 1e-3
    assert stats.kstest((vx + 12.5) / 25.0, "uniform").pvalue > 1e-3
    assert stats.kstest((vy + 12.5) / 25.0, "uniform").pvalue > 1e-3
    for a, b in [(x, off), (x, vx), (vx, vy), (off, vy)]:
        assert abs(np.corrcoef(a, b)[0, 1]) < 4 / math.sqrt(n)
    assert np.max(np.abs(vx)) <= 12.5 and np.max(np.abs(vy)) <= 12.5


def test_init_words_are_philox_stream5(orc, aten_kat):
    """The draws of particle g are the words of Philox({g, 0, 5, g >> 32}, seed) (ATen's
    independent implementation), each mapped by conv23 (pinned exactly elsewhere)."""
    n = 1 << 20
    gs = [0, 1, 77, 123456, n - 1]
    soa, _, _ = orc.init_population(M0, n, BOX, 20.0, 1.0, g_lo=0, g_hi=n)
    triples = [(M0.seed, 5 | ((g >> 32) << 32), (g & 0xFFFFFFFF)) for g in gs]
    words = aten_kat(triples)
    for g, wd in zip(gs, words):
        u = [orc.conv23(v) for v in wd]
        assert soa[0, g] == np.float32(-1000.0 + 2000.0 * u[1])
        assert soa[1, g] == np.float32(20.0 * (2.0 * u[2] - 1.0))
        assert soa[3, g] == np.float32(20.0 * (2.0 * u[3] - 1.0))
        assert soa[2, g] == np.float32(-1000.0 + 2000.0 * (g + u[0]) / n)


def test_init_mass_uniform(orc):
    """equal weights; they carry the total mass m0."""
    for n, m0 in [(1, 1.0), (1000, 3.0), (65536, 1024.0)]:
        _, w, inside = orc.init_population(M0, n, BOX, 20.0, m0)
        assert inside == n
        assert np.all(w == np.float32(m0 / n))
        assert abs(math.fsum(w) - m0) <= n * 2.0**-24 * m0


def test_init_mass_box(orc):
    """Mass only inside the (closed) mass box, shared equally; empty box -> all zero."""
    n = 50000
    mb = (0.0, 1000.0, 0.0, 1000.0)
    soa, w, inside = orc.init_population(M0, n, BOX, 20.0, 1024.0, mass_box=mb)
    x, y = soa[0], soa[2]
    ins = (x >= 0) & (x <= 1000) & (y >= 0) & (y <= 1000)
    assert inside == int(ins.sum()) and abs(inside / n - 0.25) < 0.01
    assert np.all(w[~ins] == 0) and np.all(w[ins] == np.float32(1024.0 / inside))
    assert abs(math.fsum(w) - 1024.0) <= inside * 2.0**-24 * 1024.0
    # contiguous index blocks are y-bands: the lower half of the indices holds no mass
    assert np.all(w[: n // 2 - 1] == 0)
    _, w0, i0 = orc.init_population(M0, n, BOX, 20.0, 5.0, mass_box=(2000.0, 3000.0, 0.0, 1.0))
    assert i0 == 0 and np.all(w0 == 0)


def test_init_groups_partition_the_population(orc):
    """A group's particles are the block of the global population at the same indices;
    its weights share the mass within the group (omega_0 = 1/M per group)."""
    n, K = 9001, 3
    full, _, _ = orc.init_population(M0, n, BOX, 20.0, 2.0)
    for j in range(K):
        lo, hi = n * j // K, n * (j + 1) // K
        part, w, _ = orc.init_population(M0, n, BOX, 20.0, 2.0, g_lo=lo, g_hi=hi)
        assert np.array_equal(part, full[:, lo:hi])
        assert np.all(w == np.float32(2.0 / (hi - lo)))
