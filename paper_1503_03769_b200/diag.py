"""Near-tie diagnostics for the parity claims (north_star: "resampled indices bit-exact
except where a threshold lies within 1e-9 of a cumulative-sum boundary, with that
count reported"; SURVEY.md §8(c) S8 for the label sets).

Host-side counting on results the CUDA path already produced (the weights it
resampled, the accumulators it extracted from); nothing here is on the filter's
path and nothing here computes a filter result.
"""
import numpy as np


def resample_near_ties(w, U, n_out, W=None, O=0.0, j_lo=0, j_hi=None, tol=1e-9):
    """Boolean mask over the thresholds t_j = (j + U) W / n_out, j in [j_lo, j_hi), that
    lie within `tol` (unnormalised mass units) of a cumulative-sum boundary
    B_i = O + sum_{l <= i} w_l of this weight block (t in
    [B_{i-1}, B_i)).  O is the block's offset (the mass of the ranks before it);
    W defaults to the block's own total (one rank)."""
    B = O + np.cumsum(np.asarray(w, np.float64))
    if W is None:
        W = float(B[-1]) if len(B) else 0.0
    if j_hi is None:
        j_hi = n_out
    if j_hi <= j_lo or len(B) == 0:
        return np.zeros(max(0, j_hi - j_lo), bool)
    t = (np.arange(j_lo, j_hi, dtype=np.float64) + U) * W / n_out
    idx = np.searchsorted(B, t)
    d = np.abs(O - t)  # the block's lower boundary
    for off in (-1, 0):
        k = np.clip(idx + off, 0, len(B) - 1)
        d = np.minimum(d, np.abs(B[k] - t))
    return d <= tol


def label_threshold_near_ties(dW, LT, rel=1e-5):
    """Labels (other than the LT-th itself) whose dW lies within `rel` of the LT-th
    largest eligible dW: where the top-LT selection (ties by label) may
    legitimately differ between fp32 and fp64."""
    dW = np.asarray(dW, np.float64)
    elig = np.sort(dW[dW > 0])[::-1]
    if LT <= 0 or len(elig) == 0:
        return 0
    thr = elig[min(LT, len(elig)) - 1]
    return int(np.sum(np.abs(elig - thr) <= rel * thr)) - 1
