"""Pins of the fp64 oracle against things other than itself (-m "not gpu").

Each test names what it pins and the passage it follows.  Sources of truth:
ATen's independent Philox implementation, exact rational arithmetic, closed
forms (textbook Gaussian / Kalman results, numerical quadrature), invariants
of the PHD update (Eqs 8, 12-17), brute force on tiny inputs in
40-digit mpmath, and hand-derived systematic-resampling cases.
"""
import math
import os
import subprocess
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import scenario
from scenario.configs import Model, POSITION, RANGE_BEARING

HERE = os.path.dirname(os.path.abspath(__file__))
TORCH_INC = None


def _torch_include():
    import importlib.util
    spec = importlib.util.find_spec("torch")
    return os.path.join(os.path.dirname(spec.origin), "include")


@pytest.fixture(scope="module")
def aten_kat(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("kat") / "aten_philox_kat")
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-I" + _torch_include(), "-o", exe,
                           os.path.join(HERE, "pins", "aten_philox_kat.cpp")])

    def run(triples):
        inp = "\n".join(f"{s} {a} {b}" for s, a, b in triples) + "\n"
        out = subprocess.run([exe], input=inp.encode(), stdout=subprocess.PIPE, check=True).stdout
        return [list(map(int, l.split())) for l in out.decode().strip().splitlines()]
    return run


POS = Model(meas=POSITION, sigma_z=(10.0, 10.0), p_d=0.98, clutter_rate=10.0,
            region=(-1000.0, 1000.0, -1000.0, 1000.0))
RB = Model(meas=RANGE_BEARING, sigma_z=(10.0, 0.01), p_d=0.98, clutter_rate=50.0,
           region=(0.0, 2000.0, -math.pi, math.pi), sensor_xy=(0.0, 0.0))


# --------------------------------------------------------------------------
# Philox4x32-10 (DESIGN.md §2 "noise") vs ATen at::philox_engine
# ATen counter = (offset lo, offset hi, subseq lo, subseq hi); ours = (g lo, k, stream, g hi)
def test_philox_matches_aten(orc, aten_kat):
    rng = np.random.default_rng(5)
    cases = []
    for _ in range(2000):
        seed = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        g = int(rng.integers(0, 2**40))
        k = int(rng.integers(0, 2**32))
        stream = int(rng.integers(0, 8))
        cases.append((seed, g, k, stream))
    cases += [(1, 0, 0, 0), (0, 0, 0, 0), (1, 2**24 - 1, 10, 1), (2**64 - 1, 2**32 + 5, 3, 5)]
    triples = [(s, st | ((g >> 32) << 32), (g & 0xFFFFFFFF) | (k << 32)) for s, g, k, st in cases]
    ref = aten_kat(triples)
    for (s, g, k, st), r in zip(cases, ref):
        got = orc.philox([g & 0xFFFFFFFF, k, st, g >> 32], [s & 0xFFFFFFFF, s >> 32])
        assert got == r, (s, g, k, st)


# --------------------------------------------------------------------------
# uint -> uniform conversions: exact rational values of the stated convention
def test_conv23_exact(orc):
    for w in [0, 1, 0x1FF, 0x200, 0x20000000, 0x80000000, 0xFFFFFFFF, 123456789]:
        want = (Fraction(w >> 9) + Fraction(1, 2)) / 2**23
        assert Fraction(orc.conv23(w)) == want
    assert orc.conv23(0) == 2.0**-24
    assert orc.conv23(0xFFFFFFFF) == 1.0 - 2.0**-24
    assert orc.conv23(0x80000000) == 0.500000059604644775390625


def test_u52_exact(orc):
    rng = np.random.default_rng(3)
    for _ in range(200):
        a, b = int(rng.integers(0, 2**32)), int(rng.integers(0, 2**32))
        want = (Fraction(a >> 6) * 2**26 + Fraction(b >> 6) + Fraction(1, 2)) / 2**52
        assert Fraction(orc.u52(a, b)) == want
    assert Fraction(orc.u52(0x80000000, 0)) == Fraction(1, 2) + Fraction(1, 2**53)
    assert 0.0 < orc.u52(0, 0) and orc.u52(0xFFFFFFFF, 0xFFFFFFFF) < 1.0


def test_box_muller_closed_form(orc):
    # Box & Muller (1958): sqrt(-2 ln u1) (cos, sin)(2 pi u2), evaluated at 40 digits
    mpmath.mp.dps = 40
    for w1, w2 in [(0x80000000, 0x20000000), (1, 0xFFFFFFFF), (0xFFFFFFFF, 0x40000000), (12345, 987654321)]:
        u1, u2 = orc.conv23(w1), orc.conv23(w2)
        r = mpmath.sqrt(-2 * mpmath.log(mpmath.mpf(u1)))
        n1, n2 = orc.box_muller(u1, u2)
        assert abs(n1 - float(r * mpmath.cos(2 * mpmath.pi * mpmath.mpf(u2)))) < 1e-15 * max(1, abs(n1))
        assert abs(n2 - float(r * mpmath.sin(2 * mpmath.pi * mpmath.mpf(u2)))) < 1e-15 * max(1, abs(n2))
    n1, n2 = orc.box_muller(orc.conv23(0x80000000), orc.conv23(0x20000000))
    assert abs(n1 - 0.83255422776763955) < 1e-15 and abs(n2 - 0.83255485136269256) < 1e-15


def test_box_muller_is_standard_normal(orc):
    """Philox -> conv23 -> Box-Muller draws are N(0,1): KS test vs scipy's cdf."""
    from scipy import stats
    m = Model(sigma_a=1.0, T=1.0, p_s=1.0)
    n = 20000
    soa = np.zeros((4, n))
    s, _ = orc.predict(m, 7, soa, np.ones(n))
    # zero state, T=1, sigma_a=1: vx' = n1, vy' = n2 exactly
    for comp in (s[1], s[3]):
        assert stats.kstest(comp, "norm").pvalue > 1e-3
    assert abs(np.corrcoef(s[1], s[3])[0, 1]) < 4 / math.sqrt(n)


# --------------------------------------------------------------------------
# CV prediction (Eq 5)
def test_predict_zero_noise_is_F_x(orc):
    m = Model(sigma_a=0.0, T=1.0, p_s=0.99)
    soa = np.array([[0.0, 10.0], [3.0, 0.0], [0.0, 20.0], [-3.0, 0.0]])
    s, w = orc.predict(m, 1, soa, np.array([1.0, 0.5]))
    assert np.array_equal(s[:, 0], [3.0, 3.0, -3.0, -3.0])
    assert np.array_equal(s[:, 1], [10.0, 0.0, 20.0, 0.0])
    assert np.allclose(w, [0.99, 0.495], rtol=0, atol=1e-16)      # Eq 5, q = prior
    m2 = Model(sigma_a=0.0, T=2.5)
    s2, _ = orc.predict(m2, 1, np.array([[1.0], [2.0], [3.0], [4.0]]), np.ones(1))
    assert np.allclose(s2[:, 0], [1 + 2.5 * 2, 2, 3 + 2.5 * 4, 4], rtol=0, atol=1e-14)


def test_predict_moments_match_GQGT(orc):
    """Sample mean F x and covariance sigma_a^2 G G^T (T=2 so every G entry is distinct)."""
    T, sa, n = 2.0, 5.0, 200000
    m = Model(sigma_a=sa, T=T)
    x0 = np.array([0.0, 3.0, 0.0, -3.0])
    soa = np.tile(x0[:, None], (1, n))
    s, _ = orc.predict(m, 3, soa, np.ones(n))
    F = np.array([[1, T, 0, 0], [0, 1, 0, 0], [0, 0, 1, T], [0, 0, 0, 1]], float)
    G = np.array([[T * T / 2, 0], [T, 0], [0, T * T / 2], [0, T]], float)
    cov = sa * sa * G @ G.T
    mean_err = s.mean(axis=1) - F @ x0
    assert np.all(np.abs(mean_err) < 5 * np.sqrt(np.diag(cov) / n))
    emp = np.cov(s)
    # entries of a sample covariance have std ~ sqrt((s_ii s_jj + s_ij^2)/n)
    sd = np.sqrt((np.outer(np.diag(cov), np.diag(cov)) + cov ** 2) / n)
    assert np.all(np.abs(emp - cov) < 6 * sd + 1e-9)


# --------------------------------------------------------------------------
# Sensor models and clutter
def test_kappa_closed_form(orc):
    m = Model(clutter_rate=10.0, region=(0.0, 200.0, -math.pi / 2, math.pi / 2), meas=RANGE_BEARING)
    assert abs(orc.kappa(m) - 10.0 / (math.pi * 200.0)) < 1e-18
    assert orc.kappa(POS) == 10.0 / 4e6


def test_position_likelihood_values(orc):
    peak = orc.likelihood(POS, (5.0, -7.0), (5.0, -7.0))
    assert abs(peak - 1.0 / (2 * math.pi * 100.0)) < 1e-18
    one_sigma = orc.likelihood(POS, (15.0, -7.0), (5.0, -7.0))
    assert abs(one_sigma / peak - math.exp(-0.5)) < 1e-15
    assert abs(orc.likelihood(POS, (10.0, 0.0), (0.0, 0.0)) - 9.6532352630053908e-4) < 1e-18


def test_position_likelihood_integrates_to_one(orc):
    from scipy import integrate
    m = Model(meas=POSITION, sigma_z=(7.0, 12.0))
    f = lambda zy, zx: orc.likelihood(m, (zx, zy), (3.0, -4.0))
    val, err = integrate.dblquad(f, 3 - 80, 3 + 80, -4 - 130, -4 + 130, epsabs=1e-11)
    assert abs(val - 1.0) < 1e-8


def test_range_bearing_likelihood(orc):
    # h(3,4) = (5, atan2(4,3)); residual 0 gives the peak 1/(2 pi s_r s_t)
    peak = 1.0 / (2 * math.pi * 10.0 * 0.01)
    assert abs(orc.likelihood(RB, (5.0, math.atan2(4.0, 3.0)), (3.0, 4.0)) - peak) < 1e-13
    assert abs(orc.likelihood(RB, (15.0, math.atan2(4.0, 3.0)), (3.0, 4.0)) - peak * math.exp(-0.5)) < 1e-13
    # wrap symmetry: target at bearing pi; residuals +-0.005 across the seam
    a = orc.likelihood(RB, (1000.0, math.pi - 0.005), (-1000.0, 0.0))
    b = orc.likelihood(RB, (1000.0, -math.pi + 0.005), (-1000.0, 0.0))
    assert abs(a - b) < 1e-12 * a and a > 0.1 * peak
    # degenerate target on the sensor: bearing 0
    assert abs(orc.likelihood(RB, (0.0, 0.0), (0.0, 0.0)) - peak) < 1e-13


def test_range_bearing_likelihood_integrates_to_one(orc):
    from scipy import integrate
    m = Model(meas=RANGE_BEARING, sigma_z=(10.0, 0.3), sensor_xy=(50.0, -20.0))
    tx, ty = 50.0 - 400.0, -20.0 + 1.0  # bearing close to pi: the integral crosses the seam
    f = lambda th, r: orc.likelihood(m, (r, th), (tx, ty))
    val, _ = integrate.dblquad(f, 400 - 100, 400 + 100, -math.pi, math.pi, epsabs=1e-10)
    assert abs(val - 1.0) < 1e-7


# --------------------------------------------------------------------------
# Update (Eqs 7-8, 10-17): brute force and invariants
def _mp_update(model, soa, w, z):
    """40-digit brute force of Eqs 7/11 (C), 8/12-15 (w'), 16 (dW), Eq 18 numerators."""
    mpmath.mp.dps = 40
    pd = mpmath.mpf(model.p_d)
    V = (mpmath.mpf(model.region[1]) - model.region[0]) * (mpmath.mpf(model.region[3]) - model.region[2])
    kap = mpmath.mpf(model.clutter_rate) / V
    s0, s1 = mpmath.mpf(model.sigma_z[0]), mpmath.mpf(model.sigma_z[1])

    def g(zz, x, y):
        if model.meas == POSITION:
            d0, d1 = mpmath.mpf(zz[0]) - x, mpmath.mpf(zz[1]) - y
        else:
            px, py = mpmath.mpf(x) - model.sensor_xy[0], mpmath.mpf(y) - model.sensor_xy[1]
            d0 = mpmath.mpf(zz[0]) - mpmath.sqrt(px * px + py * py)
            d1 = mpmath.mpf(zz[1]) - mpmath.atan2(py, px)
            while d1 > mpmath.pi:
                d1 -= 2 * mpmath.pi
            while d1 <= -mpmath.pi:
                d1 += 2 * mpmath.pi
        return mpmath.exp(-(d0 ** 2 / (2 * s0 ** 2) + d1 ** 2 / (2 * s1 ** 2))) / (2 * mpmath.pi * s0 * s1)

    n, M = len(w), len(z)
    G = [[pd * g(z[p], mpmath.mpf(soa[0, i]), mpmath.mpf(soa[2, i])) for p in range(M)] for i in range(n)]
    C = [mpmath.fsum(G[i][p] * mpmath.mpf(w[i]) for i in range(n)) for p in range(M)]
    wn = [mpmath.mpf(w[i]) * ((1 - pd) + mpmath.fsum(G[i][p] / (kap + C[p]) for p in range(M)))
          for i in range(n)]
    acc = [[mpmath.fsum(G[i][p] / (kap + C[p]) * mpmath.mpf(w[i]) * (1 if c == 0 else mpmath.mpf(soa[c - 1, i]))
                        for i in range(n)) for c in range(5)] for p in range(M)]
    return C, wn, acc, kap


@pytest.mark.parametrize("model", [POS, RB], ids=["position", "range_bearing"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_update_brute_force_mpmath(orc, model, seed):
    rng = np.random.default_rng(seed)
    n, M = int(rng.integers(1, 9)), int(rng.integers(1, 5))
    if model.meas == POSITION:
        z = rng.uniform(-50, 50, (M, 2))
        soa = np.stack([z[rng.integers(0, M, n), 0] + rng.normal(0, 12, n), rng.normal(0, 5, n),
                        z[rng.integers(0, M, n), 1] + rng.normal(0, 12, n), rng.normal(0, 5, n)])
    else:
        z = np.stack([rng.uniform(100, 300, M), rng.uniform(-math.pi, math.pi, M)], axis=1)
        z[0, 1] = math.pi - 0.004  # a measurement on the seam
        pick = rng.integers(0, M, n)
        r = z[pick, 0] + rng.normal(0, 8, n)
        th = z[pick, 1] + rng.normal(0, 0.008, n)
        soa = np.stack([r * np.cos(th), rng.normal(0, 5, n), r * np.sin(th), rng.normal(0, 5, n)])
    w = rng.uniform(0.01, 1.0, n)
    C = orc.normalizers(model, soa, w, z)
    wn, acc = orc.update(model, soa, w, z, C)
    Cm, wm, am, _ = _mp_update(model, soa, w, z)
    for p in range(M):
        assert abs(C[p] - float(Cm[p])) <= 1e-13 * float(Cm[p]) + 1e-300
        for c in range(5):
            assert abs(acc[p, c] - float(am[p][c])) <= 1e-12 * max(abs(float(am[p][c])), float(am[p][0]) * 100) + 1e-300
    for i in range(n):
        assert abs(wn[i] - float(wm[i])) <= 1e-13 * float(wm[i])


def _cloud(seed, n, M, model=POS):
    rng = np.random.default_rng(seed)
    z = scenario.random_measurements(M, seed, meas=model.meas, region=model.region).astype(np.float64)
    soa, w = scenario.clustered_particles(n, z, seed, meas=model.meas, sensor=model.sensor_xy)
    return soa.astype(np.float64), w.astype(np.float64), z


@pytest.mark.parametrize("model", [POS, RB], ids=["position", "range_bearing"])
def test_update_mass_identity(orc, model):
    """sum_i w'_i = (1-pD) W + sum_p C_p/(kappa+C_p)  and  dW_p = C_p/(kappa+C_p) (north_star; S1)."""
    soa, w, z = _cloud(4, 3000, 40, model)
    C = orc.normalizers(model, soa, w, z)
    wn, acc = orc.update(model, soa, w, z, C)
    kap = orc.kappa(model)
    lhs = math.fsum(wn)
    rhs = (1 - model.p_d) * math.fsum(w) + math.fsum(C / (kap + C))
    assert abs(lhs - rhs) < 1e-12 * rhs
    assert np.allclose(acc[:, 0], C / (kap + C), rtol=1e-12, atol=0)
    assert np.all(acc[:, 0] < 1.0)


def test_update_special_cases(orc):
    from dataclasses import replace
    soa, w, z = _cloud(5, 500, 7)
    # pD = 0: nothing detected -> C = 0, weights unchanged
    m0 = replace(POS, p_d=0.0)
    C = orc.normalizers(m0, soa, w, z)
    wn, acc = orc.update(m0, soa, w, z, C)
    assert np.all(C == 0) and np.array_equal(wn, w) and np.all(acc == 0)
    # Z empty -> w' = (1 - pD) w
    wn, acc = orc.update(POS, soa, w, np.zeros((0, 2)), np.zeros(0))
    assert np.allclose(wn, (1 - POS.p_d) * w, rtol=1e-15, atol=0)
    # kappa = 0 and M = 1: dW = 1
    mk = replace(POS, clutter_rate=0.0)
    z1 = z[:1]
    C = orc.normalizers(mk, soa, w, z1)
    _, acc = orc.update(mk, soa, w, z1, C)
    assert abs(acc[0, 0] - 1.0) < 1e-14
    # kappa = 0 and C = 0 (measurement far from every particle): term defined as 0
    zfar = np.array([[1e7, 1e7]])
    C = orc.normalizers(mk, soa, w, zfar)
    wn, acc = orc.update(mk, soa, w, zfar, C)
    assert C[0] == 0.0 and np.all(np.isfinite(wn)) and acc[0, 0] == 0.0


def test_update_worked_example_single_particle(orc):
    """Ex1: one particle at 0, w = 1, z = (10, 0), sigma = 10, pD = 0.98, kappa = 2.5e-6.
    Closed form: g = e^{-1/2}/(200 pi); C = pD g; w' = (1-pD) + pD g/(kappa + C); dW = C/(kappa+C)."""
    m = Model(meas=POSITION, sigma_z=(10.0, 10.0), p_d=0.98, clutter_rate=10.0)
    soa = np.array([[0.0], [1.5], [0.0], [-2.0]])
    z = np.array([[10.0, 0.0]])
    C = orc.normalizers(m, soa, [1.0], z)
    wn, acc = orc.update(m, soa, [1.0], z, C)
    g = math.exp(-0.5) / (200 * math.pi)
    assert abs(C[0] - 9.4601705577452829e-4) < 1e-18 and abs(C[0] - 0.98 * g) < 1e-18
    assert abs(wn[0] - 1.0173643067514916) < 1e-15
    assert abs(acc[0, 0] - 0.99736430675149159) < 1e-15
    zeta = acc[0, 1:] / acc[0, 0]
    assert np.allclose(zeta, soa[:, 0], rtol=0, atol=1e-15)  # single particle -> its state


def test_update_kalman_special_case(orc):
    """Linear-Gaussian, one measurement: particles ~ N(0, 100 I) on position with equal
    weights, R = 100 I, z = (20, 0).  zeta_pos -> Kalman posterior mean (10, 0) (gain 1/2);
    C -> pD N(z; 0, 200 I) (predictive density)."""
    rng = np.random.default_rng(11)
    n = 200000
    m = Model(meas=POSITION, sigma_z=(10.0, 10.0), p_d=0.98, clutter_rate=10.0)
    soa = np.stack([rng.normal(0, 10, n), np.zeros(n), rng.normal(0, 10, n), np.zeros(n)])
    w = np.full(n, 1.0 / n)
    z = np.array([[20.0, 0.0]])
    C = orc.normalizers(m, soa, w, z)
    _, acc = orc.update(m, soa, w, z, C)
    zeta = acc[0, 1:] / acc[0, 0]
    assert abs(zeta[0] - 10.0) < 0.1 and abs(zeta[2]) < 0.1
    assert abs(C[0] - 0.98 * math.exp(-400.0 / 400.0) / (2 * math.pi * 200.0)) < 0.02 * C[0]


# --------------------------------------------------------------------------
# Extraction
def test_extract_rules(orc):
    m = POS
    acc = np.zeros((4, 5))
    acc[:, 0] = [0.3, 0.9, 0.3, 0.0]
    acc[:, 1:] = np.arange(16).reshape(4, 4) * acc[:, :1]
    e = orc.extract(m, acc, 1.15, 2.0)              # mass 1.15 -> LT 1
    assert e["LT"] == 1 and list(e["labels"]) == [1]
    assert np.allclose(e["states"][0], [4, 5, 6, 7])
    e = orc.extract(m, acc, 2.5, 2.0)               # round half away: 2.5 -> 3; tie 0.3/0.3 -> smaller label first
    assert e["LT"] == 3 and list(e["labels"]) == [1, 0, 2] and e["lt_clamped"] == 0
    e = orc.extract(m, acc, 4.0, 2.0)               # LT 4 > 3 eligible (dW = 0 excluded) -> clamp + flag
    assert e["LT"] == 4 and len(e["labels"]) == 3 and e["lt_clamped"] == 1
    e = orc.extract(m, acc, 0.49, 2.0)              # LT = 0 -> empty
    assert e["LT"] == 0 and len(e["labels"]) == 0
    assert abs(e["undetected_mass"] - 0.02 * 2.0) < 1e-16   # Eq 17 = (1-pD) W_pred
    assert orc.round_half_away(1.5) == 2 and orc.round_half_away(2.4999) == 2


# --------------------------------------------------------------------------
# Systematic resampling
def test_resample_known_cases(orc):
    anc, W = orc.resample([0.1, 0.5, 0.2, 0.2], 0.3, 4)
    assert list(anc) == [0, 1, 1, 3] and abs(W - 1.0) < 1e-15
    anc, _ = orc.resample([1.0, 1.0, 1.0, 1.0], 0.0, 4)    # exact-boundary convention t in [B_{i-1}, B_i)
    assert list(anc) == [0, 1, 2, 3]
    anc, W = orc.resample([2.0], 0.5, 4)
    assert list(anc) == [0, 0, 0, 0] and W == 2.0
    anc, _ = orc.resample([1.0, 0.0, 0.0, 0.0], 0.7, 5)
    assert list(anc) == [0] * 5
    anc, W = orc.resample([0.0, 0.0, 0.0], 0.5, 6)          # zero mass: spread, flagged by W == 0
    assert W == 0.0 and list(anc) == [0, 0, 1, 1, 2, 2]


def _exact_counts(w, U, n_out):
    """count_i = #{ j : B_{i-1} <= t_j < B_i } in exact rational arithmetic."""
    wf = [Fraction(x) for x in w]
    W = sum(wf)
    Uf = Fraction(U)
    counts, B = [], Fraction(0)
    for x in wf:
        lo, hi = B, B + x
        # j with lo <= (j+U) W/n < hi  <=>  lo n/W - U <= j < hi n/W - U
        a = math.ceil(lo * n_out / W - Uf)
        b = math.ceil(hi * n_out / W - Uf)
        counts.append(max(0, min(b, n_out)) - max(0, min(a, n_out)))
        B = hi
    return counts


@pytest.mark.parametrize("seed", range(6))
def test_resample_vs_exact_rational(orc, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    w = rng.uniform(0, 1, n) * (rng.uniform(size=n) < 0.7)
    if w.sum() == 0:
        w[0] = 1.0
    n_out = int(rng.integers(1, 500))
    U = orc.resample_U(seed, 3)
    anc, W = orc.resample(w, U, n_out)
    counts = np.bincount(anc, minlength=n)
    exact = _exact_counts(w, U, n_out)
    assert list(counts) == exact
    assert np.all(np.diff(anc) >= 0) and counts.sum() == n_out
    share = n_out * w / w.sum()
    assert np.all(counts >= np.floor(share) - 1e-9) and np.all(counts <= np.ceil(share) + 1e-9)


def test_resample_U_is_philox_u52(orc):
    o = orc.philox([0, 9, 3, 0], [7, 0])
    assert orc.resample_U(7, 9) == orc.u52(o[0], o[1])


# --------------------------------------------------------------------------
# Births (S10, S27)
def test_births_measurement_driven(orc):
    m = Model(meas=POSITION, sigma_z=(10.0, 10.0), birth_mass=0.1, birth_sigma_v=10.0)
    zprev = np.array([[100.0, -200.0], [-500.0, 700.0], [0.0, 0.0]])
    J = 30000
    s, w = orc.births(m, 2, 1000, J, zprev)
    assert np.allclose(w, 0.1 / J) and abs(math.fsum(w) - 0.1) < 1e-12
    for p in range(3):
        sel = np.arange(J) % 3 == p
        nn = sel.sum()
        assert abs(s[0, sel].mean() - zprev[p, 0]) < 5 * 10 / math.sqrt(nn)
        assert abs(s[2, sel].mean() - zprev[p, 1]) < 5 * 10 / math.sqrt(nn)
        assert abs(s[0, sel].std() - 10.0) < 0.5 and abs(s[1, sel].std() - 10.0) < 0.5
    # uniform over the region when no previous measurement exists
    s, _ = orc.births(m, 1, 1000, J, None)
    assert s[0].min() >= -1000 and s[0].max() <= 1000 and abs(s[0].mean()) < 30 and abs(s[2].mean()) < 30


def test_births_range_bearing_inverse_sensor(orc):
    m = Model(meas=RANGE_BEARING, sigma_z=(10.0, 0.01), sensor_xy=(5.0, -3.0),
              region=(0.0, 2000.0, -math.pi, math.pi))
    zprev = np.array([[800.0, math.pi - 0.001]])
    s, _ = orc.births(m, 2, 0, 20000, zprev)
    px, py = s[0] - 5.0, s[2] + 3.0
    r, th = np.hypot(px, py), np.arctan2(py, px)
    dth = np.angle(np.exp(1j * (th - zprev[0, 1])))
    assert abs(r.mean() - 800.0) < 0.5 and abs(r.std() - 10.0) < 0.3
    assert abs(dth.mean()) < 2e-4 and abs(dth.std() - 0.01) < 3e-4


# --------------------------------------------------------------------------
# Golden SPEC examples (tests/golden/spec_examples.json; each cites SPEC.md)
def test_golden_spec_examples(orc):
    import json
    with open(os.path.join(HERE, "golden", "spec_examples.json")) as f:
        g = json.load(f)
    for ex in g["examples"]:
        if ex["op"] == "kappa":
            m = Model(clutter_rate=ex["lambda"], region=tuple(ex["region"]))
            assert abs(orc.kappa(m) - ex["expect"]) < ex["tol"], ex["cite"]
        elif ex["op"] == "round":
            assert orc.round_half_away(ex["mass"]) == ex["expect"], ex["cite"]
        elif ex["op"] == "resample":
            anc, W = orc.resample(ex["w"], ex["U"], ex["n_out"])
            assert list(anc) == ex["expect_anc"] and abs(W / ex["n_out"] - ex["expect_w"]) < 1e-15, ex["cite"]
        elif ex["op"] == "peak":
            m = Model(meas=RANGE_BEARING, sigma_z=tuple(ex["sigma"]))
            assert abs(orc.likelihood(m, (5.0, math.atan2(4, 3)), (3.0, 4.0)) - ex["expect"]) < ex["tol"], ex["cite"]
        else:
            raise AssertionError(ex)


def test_births_gaussian_model(orc):
    """birth intensity N(x-bar, Q), x-bar = (0,3,0,-3), Q = diag(10,1,10,1)."""
    m = Model(birth_model=1, birth_mass=0.2)
    J = 40000
    s, w = orc.births(m, 3, 500, J, np.array([[100.0, 100.0]]))  # Z_{k-1} is ignored by this model
    assert np.allclose(w, 0.2 / J)
    mean, std = s.mean(axis=1), s.std(axis=1)
    assert np.all(np.abs(mean - np.array([0.0, 3.0, 0.0, -3.0])) < 5 * np.array(m.birth_std) / math.sqrt(J))
    assert np.all(np.abs(std - np.array(m.birth_std)) < 0.02 * np.array(m.birth_std))
    assert abs(np.corrcoef(s[0], s[2])[0, 1]) < 4 / math.sqrt(J)
    # zero covariance -> exact copies of x-bar
    m0 = Model(birth_model=1, birth_std=(0.0, 0.0, 0.0, 0.0))
    s0, _ = orc.births(m0, 1, 0, 3, None)
    assert np.array_equal(s0, np.tile(np.array([[0.0], [3.0], [0.0], [-3.0]]), (1, 3)))


# --------------------------------------------------------------------------
# NEXT-4: Eq 5 with a proposal q_k != transition prior, Eq 6 with the full ratio
def test_predict_importance_proposal(orc):
    """Eq 5: w~ = phi/q w with q the CV model of noise std s sigma_a.
    Pins: (i) E_q[f/q] = 1 and the weighted noise moments equal the transition's
    (importance-sampling identities, Monte Carlo); (ii) the closed form through the
    Box-Muller radius, n1^2 + n2^2 = -2 ln u1, so phi/q = p_s s^2 u1^(s^2 - 1) exactly,
    with u1 from ATen-pinned Philox; (iii) s = 1 is the transition prior."""
    n = 400000
    T, sa, ps, s = 1.0, 5.0, 0.99, 2.0
    m = Model(T=T, sigma_a=sa, p_s=ps, proposal_scale=s, seed=11)
    soa = np.tile(np.array([[10.0], [1.0], [-20.0], [-1.0]]), (1, n))
    x, w = orc.predict(m, 3, soa, np.ones(n), g0=100)
    a_x, a_y = (x[1] - 1.0) / T, (x[3] + 1.0) / T
    # (i) unbiasedness and moments
    assert abs(w.mean() - ps) < 5 * w.std() / math.sqrt(n)
    assert abs(a_x.std() - s * sa) < 0.01 * s * sa  # drawn from q
    for a in (a_x, a_y):
        m2 = np.sum(w * a * a) / np.sum(w)
        assert abs(m2 - sa * sa) < 0.02 * sa * sa  # weighted: the transition's variance
    # (ii) closed form via the Box-Muller radius
    for i in (0, 1, 7, 12345):
        o = orc.philox([100 + i, 3, 1, 0], [11, 0])
        u1 = orc.conv23(o[0])
        assert abs(w[i] - ps * s * s * u1 ** (s * s - 1)) < 1e-12 * max(1.0, w[i])
    # (iii) s = 1 -> q = f, ratio p_s
    x1, w1 = orc.predict(Model(T=T, sigma_a=sa, p_s=ps, proposal_scale=1.0, seed=11), 3, soa[:, :10], np.ones(10))
    assert np.all(w1 == ps)


def _is_model(meas, **kw):
    base = dict(birth_model=2, birth_mass=0.3, birth_sigma_v=4.0, seed=5)
    if meas == POSITION:
        base.update(meas=POSITION, sigma_z=(10.0, 10.0), birth_mean=(50.0, 1.0, -30.0, -2.0),
                    birth_std=(40.0, 2.0, 30.0, 2.0))
    else:
        base.update(meas=RANGE_BEARING, sigma_z=(10.0, 0.02), sensor_xy=(0.0, 0.0),
                    region=(0.0, 2000.0, -math.pi, math.pi),
                    birth_mean=(400.0, 1.0, 300.0, -2.0), birth_std=(40.0, 2.0, 30.0, 2.0))
    base.update(kw)
    return Model(**base)


@pytest.mark.parametrize("meas", [POSITION, RANGE_BEARING])
def test_births_importance_weights_unbiased(orc, meas):
    """Eq 6 with gamma(x) = gamma N(x; x-bar, Q)
    and the measurement-driven proposal: the importance-sampling estimator is unbiased,
    E[sum_b w_b h(x_b)] = gamma E_N[h], for h = 1, x, vy, (x - x-bar)^2.  A dropped
    velocity density, a missing 1/J or a missing range-bearing Jacobian 1/r breaks it."""
    m = _is_model(meas)
    if meas == POSITION:
        gx, gy = np.meshgrid(np.arange(-150.0, 251.0, 20.0), np.arange(-180.0, 121.0, 20.0))
        zprev = np.stack([gx.ravel(), gy.ravel()], axis=1)
    else:
        r, th = np.meshgrid(np.arange(300.0, 701.0, 15.0), np.arange(0.35, 0.95, 0.02))
        zprev = np.stack([r.ravel(), th.ravel()], axis=1)
    J, blo = 200003, 17  # J not a multiple of M_{k-1}; the filter's births start at blo
    s, w = orc.births(m, 4, 1000, J, zprev, b0=blo, nb=J, blo=blo)
    tot = w.sum()
    se = math.sqrt(J) * w.std()
    assert abs(tot - m.birth_mass) < 5 * se and se < 0.02 * m.birth_mass
    mx = np.sum(w * s[0]) / tot
    assert abs(mx - m.birth_mean[0]) < 1.5
    assert abs(np.sum(w * s[3]) / tot - m.birth_mean[3]) < 0.05
    assert abs(math.sqrt(np.sum(w * (s[0] - m.birth_mean[0]) ** 2) / tot) - m.birth_std[0]) < 1.0


@pytest.mark.parametrize("meas", [POSITION, RANGE_BEARING])
def test_births_importance_uniform_first_step(orc, meas):
    """k = 1, no Z_{k-1}: the proposal is uniform over the region (1/V, or 1/(V r) in the
    Cartesian plane for a uniform (r, theta)); the estimator of gamma stays unbiased.  The
    region covers the intensity to >= 4.3 std (mass outside < 2e-5)."""
    if meas == POSITION:
        m = _is_model(meas, region=(-150.0, 250.0, -180.0, 120.0))
    else:
        m = _is_model(meas, region=(300.0, 700.0, 0.35, 0.95))
    J = 400000
    s, w = orc.births(m, 1, 0, J, None)
    se = math.sqrt(J) * w.std()
    assert abs(w.sum() - m.birth_mass) < 5 * se and se < 0.05 * m.birth_mass


def test_births_importance_stratified_counts(orc):
    """Births [blo, blo+J) take component b mod M deterministically, so p_k is the mixture
    with weights n_c / J.  With M = 2, J = 3, blo = 1 the counts are (1, 2): over many steps
    the estimator of gamma is unbiased with those weights; the equal-weight mixture would
    converge to gamma * int N(x; 6, 9) p(x)/p'(x) dx (computed here by quadrature), which
    the test tells apart."""
    m = _is_model(POSITION, birth_mean=(6.0, 0.0, 0.0, 0.0), birth_std=(3.0, 3.0, 3.0, 3.0))
    zprev = np.array([[-6.0, 0.0], [6.0, 0.0]])
    tot = []
    for k in range(1, 20001):
        s, w = orc.births(m, k, 0, 3, zprev, b0=1, nb=3, blo=1)
        tot.append(w.sum())
    tot = np.array(tot)
    mean, se = tot.mean(), tot.std() / math.sqrt(len(tot))
    assert abs(mean - m.birth_mass) < 5 * se, (mean, se)
    x = np.linspace(-40.0, 50.0, 200001)
    q0, q1 = np.exp(-(x + 6.0) ** 2 / 200.0), np.exp(-(x - 6.0) ** 2 / 200.0)
    g = np.exp(-(x - 6.0) ** 2 / 18.0) / math.sqrt(18.0 * math.pi)
    wrong = m.birth_mass * np.trapezoid(g * (q0 / 3 + 2 * q1 / 3) / (q0 / 2 + q1 / 2), x)
    assert abs(wrong - m.birth_mass) > 8 * se, (wrong, se)


def test_all_core_timing_variant_matches_oracle(orc):
    """The all-core CPU baseline (oracle/phd_oracle_mt.c) computes the oracle's
    normalisers and update: identical per-particle weights, sums over particles
    equal up to fp64 summation order."""
    import scenario
    rng = np.random.default_rng(3)
    for cname in ("cfg1", "cfg2"):
        m = scenario.get(cname).model
        soa = rng.uniform(-1000, 1000, (4, 3001)).astype(np.float32)
        w = rng.uniform(0, 1e-3, 3001).astype(np.float32)
        z = scenario.random_measurements(37, 5, meas=m.meas, region=m.region)
        C = orc.normalizers(m, soa, w, z)
        wo, acc = orc.update(m, soa, w, z, C)
        for nt in (1, 3, 8):
            Cm = orc.normalizers_mt(m, soa, w, z, nt)
            wm, am = orc.update_mt(m, soa, w, z, C, nt)
            assert np.allclose(Cm, C, rtol=1e-13, atol=0)
            assert np.array_equal(wm, wo)
            assert np.allclose(am, acc, rtol=1e-12, atol=1e-300)


# --------------------------------------------------------------------------
# Worked examples of SURVEY.md §8(c) (values computed there independently of this
# oracle, from the closed forms of PAPER.md Eqs 7-8, 12-18)
def test_worked_example_two_particles_two_measurements(orc):
    """Ex2: position sigma = 10, p_D = 0.98, kappa = 2.5e-6; particles (0,0) w = 0.6 and
    (15,5) w = 0.9; z = (10,0), (12,9): C, w', dW, zeta and the mass identity."""
    m = Model(meas=POSITION, sigma_z=(10.0, 10.0), p_d=0.98, clutter_rate=10.0,
              region=(-1000.0, 1000.0, -1000.0, 1000.0))
    assert orc.kappa(m) == 2.5e-6
    soa = np.array([[0.0, 15.0], [0.0, 0.0], [0.0, 5.0], [0.0, 0.0]])
    w = np.array([0.6, 0.9])
    z = np.array([[10.0, 0.0], [12.0, 9.0]])
    C = orc.normalizers(m, soa, w, z)
    wn, acc = orc.update(m, soa, w, z, C)
    rel = lambda a, b: np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.abs(np.asarray(b)))
    assert rel(C, [1.66084918327586e-3, 1.54262188921722e-3]) < 1e-12
    assert rel(wn, [0.549877034245137, 1.47700197873555]) < 1e-12
    assert rel(acc[:, 0], [0.998497008310019, 0.998382004670669]) < 1e-12
    zeta = np.stack([acc[:, 1] / acc[:, 0], acc[:, 3] / acc[:, 0]], axis=1)
    assert np.max(np.abs(zeta - [[9.87361430062, 3.29120476687], [12.0457453003, 4.01524843343]])) < 1e-9
    assert abs(math.fsum(wn) - 2.0268790129806885) < 1e-14
    assert abs(math.fsum(wn) - ((1 - 0.98) * 1.5 + math.fsum(C / (2.5e-6 + C)))) < 1e-14


def test_worked_example_range_bearing(orc):
    """Ex3: sensor at the origin, sigma_r = 10, sigma_theta = 0.01, kappa = 50 / (2000 2 pi);
    particle (3, 4) (h = (5, atan2(4, 3))), w = 1, z = (15, atan2(4, 3)): a one-sigma range
    residual, g = e^(-1/2) / (2 pi sigma_r sigma_theta), w' = 1.0158116940774555."""
    m = Model(meas=RANGE_BEARING, sigma_z=(10.0, 0.01), p_d=0.98, clutter_rate=50.0,
              region=(0.0, 2000.0, -math.pi, math.pi), sensor_xy=(0.0, 0.0))
    assert abs(orc.kappa(m) - 3.9788735772973834e-3) < 1e-18
    soa = np.array([[3.0], [0.0], [4.0], [0.0]])
    z = np.array([[15.0, 0.92729521800161223]])
    C = orc.normalizers(m, soa, np.array([1.0]), z)
    assert abs(C[0] / 0.98 - 0.96532352630053908) < 1e-14
    wn, acc = orc.update(m, soa, np.array([1.0]), z, C)
    assert abs(wn[0] - 1.0158116940774555) < 1e-14
    assert abs(acc[0, 1] / acc[0, 0] - 3.0) < 1e-12 and abs(acc[0, 3] / acc[0, 0] - 4.0) < 1e-12
