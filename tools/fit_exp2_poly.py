"""Fit the degree-5 polynomial for 2^r, |r| <= 1/2, used by ex2_poly() in
csrc/k_update.cu (the MUFU.EX2 offload of pass 1), and
report its relative error when evaluated by fp32 Horner with fused multiply-add.

Near-minimax by iteratively reweighted least squares on Chebyshev nodes.
Usage: python tools/fit_exp2_poly.py
"""
import numpy as np


def fit(deg=5, iters=30):
    r = np.cos(np.pi * (np.arange(4000) + 0.5) / 4000) * 0.5
    A = np.vander(r, deg + 1, increasing=True)
    y = 2.0 ** r
    w = 1.0 / y
    c = np.linalg.lstsq(A * w[:, None], y * w, rcond=None)[0]
    for _ in range(iters):
        e = (A @ c - y) / y
        w2 = w * (1 + 20 * np.abs(e) / np.abs(e).max())
        c = np.linalg.lstsq(A * w2[:, None], y * w2, rcond=None)[0]
    return c.astype(np.float32)


def horner_fp32(c32, r):
    """fp32 Horner with one rounding per step (an FMA), as the kernel computes it."""
    r = np.asarray(r, dtype=np.float32)
    p = np.full_like(r, c32[-1])
    for k in range(len(c32) - 2, -1, -1):
        p = (p.astype(np.float64) * r.astype(np.float64) + np.float64(c32[k])).astype(np.float32)
    return p


def max_rel_error(c32):
    r = np.linspace(-0.5, 0.5, 200001).astype(np.float32)
    p = horner_fp32(c32, r).astype(np.float64)
    return float(np.max(np.abs(p / 2.0 ** r.astype(np.float64) - 1.0)))


if __name__ == "__main__":
    c = fit()
    print("coefficients (c0..c5):", ["%.8e" % v for v in c])
    print("max relative error (fp32 Horner):", max_rel_error(c))
