"""The gated update's exactness claim, checked on the CPU (-m "not gpu").

DESIGN.md §5 "Gated update": a (tile, measurement) pair is skipped iff
    e_max = -alpha0 dx^2 - alpha1 dy^2 + max_i log2(p_D c w_i) < -130
with (dx, dy) the measurement's distance to the tile's bounding box (arc distance
in bearing), and the claim is that every skipped term is then exactly 0 in the
dense kernels, i.e. each particle's fp32 exponent
    e_i = fma(fma(d1, d1, d0 * d0), -alpha, lw_i)        (position)
    e_i = fma(d1 * d1, -alpha1, fma(d0 * d0, -alpha0, lw_i))   (range-bearing)
is below -126, where ex2.approx.ftz returns +0.  This test restates both rules
in numpy fp32 (fma emulated: an fp32 product is exact in fp64, one rounding)
and checks the claim by brute force on tiles built to stress it: particles on
the box corners, measurements just outside the gate radius, the bearing seam.
It is independent of the CUDA code (no shared source).
"""
import math

import numpy as np

F = np.float32
LOG2E = 1.4426950408889634
GATE_MIN = -130.0


def fma32(a, b, c):
    return (np.asarray(a, np.float64) * np.asarray(b, np.float64) + np.asarray(c, np.float64)).astype(F)


def dist_iv(v, a, b):
    return np.maximum(F(0), np.maximum(F(a) - v, v - F(b)))


def dist_arc(v, a, b):
    two_pi = F(2 * math.pi)
    length = F(b) - F(a)
    t = (v - F(a)).astype(F)
    t = (t - two_pi * np.floor(t / two_pi)).astype(F)
    d = np.minimum(t - length, two_pi - t) - F(1e-5)
    out = np.maximum(F(0), d).astype(F)
    out[(length >= two_pi) | (t <= length)] = 0
    return out


def e_max(z0, z1, box, lw_max, na0, na1, wrap):
    b0, b1, e0, e1 = box
    dx = dist_iv(z0, b0, b1)
    dy = dist_arc(z1, e0, e1) if wrap else dist_iv(z1, e0, e1)
    return fma32(F(na0), (dx * dx).astype(F), fma32(F(na1), (dy * dy).astype(F), F(lw_max)))


def exponents_position(x, y, lw, z0, z1, na):
    d0 = (x[:, None] + (-z0)[None, :]).astype(F)
    d1 = (y[:, None] + (-z1)[None, :]).astype(F)
    q = fma32(d1, d1, (d0 * d0).astype(F))
    return fma32(q, F(na), lw[:, None])


def exponents_rb(r_hi, r_lo, th_hi, th_lo, lw, z0, z1, na0, na1):
    # one bearing representation per measurement class, as in the kernels
    d0 = ((r_hi[:, None] + (-z0)[None, :]).astype(F) + r_lo[:, None]).astype(F)
    d1 = ((th_hi[:, None] + (-z1)[None, :]).astype(F) + th_lo[:, None]).astype(F)
    e = fma32((d0 * d0).astype(F), F(na0), lw[:, None])
    return fma32((d1 * d1).astype(F), F(na1), e)


def _check(skipped, e):
    # every particle's term of a skipped pair is below 2^-126 (flushed to +0)
    assert not skipped.any() or np.all(e[:, skipped] < -126.0), float(np.max(e[:, skipped]))


def test_gate_skips_only_underflowing_terms_position():
    rng = np.random.default_rng(5)
    for sigma, w in ((10.0, 6e-5), (3.0, 1e-2), (40.0, 1e-9), (10.0, 0.8)):
        alpha = LOG2E / (2 * sigma * sigma)
        na = F(-alpha)
        c = 1.0 / (2 * math.pi * sigma * sigma)
        for trial in range(20):
            n = 512
            cx, cy = rng.uniform(-900, 900, 2)
            half = rng.uniform(0.1, 40.0)
            x = F(cx) + rng.uniform(-half, half, n).astype(F)
            y = F(cy) + rng.uniform(-half, half, n).astype(F)
            x[:4] = F([cx - half, cx + half, cx - half, cx + half])  # box corners
            y[:4] = F([cy - half, cy - half, cy + half, cy + half])
            lw = np.log2(F(0.98 * c) * (F(w) * rng.uniform(0.5, 1.0, n).astype(F))).astype(F)
            box = (x.min(), x.max(), y.min(), y.max())
            lwm = lw.max()
            R = math.sqrt(max(0.0, (float(lwm) - GATE_MIN) / alpha))
            # measurements on rings just inside / outside the gate radius around the box
            m = 4000
            ang = rng.uniform(0, 2 * math.pi, m)
            rad = R * rng.uniform(0.97, 1.03, m) + half
            z0 = (F(cx) + (rad * np.cos(ang)).astype(F)).astype(F)
            z1 = (F(cy) + (rad * np.sin(ang)).astype(F)).astype(F)
            em = e_max(z0, z1, box, lwm, na, na, False)
            skipped = em < GATE_MIN
            assert skipped.any() and (~skipped).any()
            _check(skipped, exponents_position(x, y, lw, z0, z1, na))


def test_gate_skips_only_underflowing_terms_range_bearing_seam():
    rng = np.random.default_rng(6)
    sr, st = 10.0, 0.01
    na0, na1 = F(-LOG2E / (2 * sr * sr)), F(-LOG2E / (2 * st * st))
    c = 1.0 / (2 * math.pi * sr * st)
    for trial in range(20):
        n = 512
        r = rng.uniform(300, 1800, n)
        # a tile hugging the seam from one side (sorted tiles lie in one cell column);
        # measurements on both sides of the seam
        side = 1.0 if trial % 2 == 0 else -1.0
        th = side * (math.pi - np.abs(rng.normal(0, 0.03, n)))
        th[0] = math.pi if side > 0 else -math.pi + 1e-7  # on the seam itself ((-pi, pi])
        r_hi = r.astype(F)
        r_lo = (r - r_hi.astype(np.float64)).astype(F)
        th_hi = th.astype(F)
        th_lo = (th - th_hi.astype(np.float64)).astype(F)
        lw = np.log2(F(0.98 * c) * F(1e-4)).astype(F) * np.ones(n, F)
        box = (r_hi.min(), r_hi.max(), th_hi.min(), th_hi.max())
        m = 3000
        z0 = rng.uniform(200, 1900, m).astype(F)
        z1 = (math.pi + rng.uniform(-0.4, 0.4, m))
        z1 = np.arctan2(np.sin(z1), np.cos(z1)).astype(F)
        em = e_max(z0, z1, box, lw.max(), na0, na1, True)
        skipped = em < GATE_MIN
        assert skipped.any() and (~skipped).any()
        # the kernels' residual uses the representation of the measurement's class:
        # (-pi, pi] for |z| <= pi/2, [0, 2 pi) above, (-2 pi, 0] below
        for cls, sel in ((0, np.abs(z1) <= np.pi / 2), (1, z1 > np.pi / 2), (2, z1 < -np.pi / 2)):
            if not sel.any():
                continue
            thr = th.copy()
            if cls == 1:
                thr = np.where(thr < 0, thr + 2 * math.pi, thr)
            elif cls == 2:
                thr = np.where(thr > 0, thr - 2 * math.pi, thr)
            t_hi = thr.astype(F)
            t_lo = (thr - t_hi.astype(np.float64)).astype(F)
            e = exponents_rb(r_hi, r_lo, t_hi, t_lo, lw, z0[sel], z1[sel], na0, na1)
            _check(skipped[sel], e)
