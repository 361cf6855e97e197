"""TEST INFRASTRUCTURE, NOT PRODUCT CODE: serial oracle of the paper-literal
distributed filter DCPFPHD (§3, Algorithm 1, Steps 1-6
lines 260-359), NEXT-1 of SURVEY.md §8(f).

K groups, run one after the other in a plain loop, each with its own particle
population and the FULL measurement set:
  Step 1 (line 266): survivors predicted (Eq 5); the J births are divided
         equally over the groups (group j gets the block [jJ/K, (j+1)J/K)),
         each weighted gamma / J_j (Eq 6 with the group's J_k): every group is a
         separate particle PHD filter of the full intensity (line 221; omega_0 =
         1/M per group, line 260), so callers give each group a full-mass population.
  Step 2 (lines 269-297): the group's own normaliser C_j(z) (Eq 11 sums over
         the group's particles only) and weights (Eqs 12-15).
  Step 3 (lines 299-324): local estimation: LT_j = round(W_j), top-LT_j labels
         by dW^{j,p}, zeta = S/dW.
  Step 4 (lines 331-333): the CU keeps a label when more than K/2 groups report
         it and averages their states.
  Step 5 (line 339, Algorithm 1): each group resamples its particles
         into max(LT_j, 1) R offspring (fixed-count configs: its block of N_out).
  Step 6 (lines 340-352): ring exchange: group j hands L particles to group
         j+1 (K -> 1) and refills the same slots with the L particles it gets
         from group j-1 (swap semantics, S21), weights travelling with
         the particles.

Readings ("DCP"): for K > 1 group j's Philox counters live in
their own space c3 = 0x40000000 + j (survivor/birth slot = local index); the
resampling offset of group j is u52(Philox({j, k, 3, 0x40000000})); the L ring
slots of group j are floor((i + v_j) N_j / L), v_j = u52(Philox({j, k, 4, 0x40000000}));
K = 1 uses the serial filter's counters (so K = 1 is the serial filter);
L = min(L_param, floor(min_j N_j / 2)) with L_param = 0 meaning floor(min_j N_j / 10).
"""
import math

import numpy as np

from . import births, extract, normalizers, philox, predict, resample, u52, update, round_half_away

SPACE = 0x40000000


def group_base(j, K):
    """Philox counter base of group j; K = 1 uses the serial filter's space, so that
    a one-group DCPFPHD is exactly the serial particle PHD step."""
    return 0 if K == 1 else (SPACE + j) << 32


def block(n, K, j):
    return (n * j) // K, (n * (j + 1)) // K


def group_U(seed, k, j, stream, K):
    ctr = [0, k, stream, 0] if K == 1 else [j, k, stream, SPACE]
    o = philox(ctr, [seed & 0xFFFFFFFF, seed >> 32])
    return u52(o[0], o[1])


def ring_slots(seed, k, j, n, L, K):
    """floor(((i + v) * n) / L) in fp64 (one rounding per operation)."""
    v = group_U(seed, k, j, 4, K)
    return [int(math.floor(((float(i) + v) * float(n)) / float(L))) for i in range(L)]


def fuse(local, K):
    """Step 4: labels reported by more than K/2 groups; state = mean of the
    supporters' states.  local: list over groups of (labels, states).
    Returns (labels ascending, states, support counts)."""
    sup = {}
    for labels, states in local:
        for lab, st in zip(labels, states):
            sup.setdefault(int(lab), []).append(np.asarray(st, dtype=np.float64))
    labs = sorted(l for l, v in sup.items() if len(v) * 2 > K)
    states = np.array([np.mean(sup[l], axis=0) for l in labs]).reshape(-1, 4)
    counts = np.array([len(sup[l]) for l in labs], dtype=np.int64)
    return np.array(labs, dtype=np.int64), states, counts


def dcp_step(m, k, groups, z, zprev, n_out_rule, L_param=0):
    """One DCPFPHD scan.  groups: list of (soa [4, n_j], w [n_j]) entering step k.
    n_out_rule(j, LT_j) -> offspring count of group j.  Returns a dict with every
    per-group intermediate and the post-exchange groups."""
    K = len(groups)
    J = m.births_per_step
    per = []
    for j, (soa, w) in enumerate(groups):
        n_j = soa.shape[1]
        ps, pw = predict(m, k, soa, w, g0=group_base(j, K))                   # Eq 5
        b0, b1 = block(J, K, j)
        # Eq 6 with the group's own J_k: each group is a separate PHD filter of the full
        # intensity, so its births carry the full birth mass gamma
        bs, bw = births(m, k, group_base(j, K) + n_j - b0, b1 - b0, zprev, b0=b0, nb=b1 - b0, blo=b0)
        xs = np.concatenate([ps, bs], axis=1)
        ws = np.concatenate([pw, bw])
        C = normalizers(m, xs, ws, z)                                          # Eq 11 (group-local)
        wn, acc = update(m, xs, ws, z, C)                                      # Eqs 12-16
        W = 0.0
        for v in wn.tolist():
            W += v
        Wp = 0.0
        for v in ws.tolist():
            Wp += v
        est = extract(m, acc, W, Wp)                                           # Step 3
        per.append({"pred": xs, "w_pred": ws, "C": C, "w_upd": wn, "acc": acc, "W": W, "W_pred": Wp,
                    "est": est})
    fused = fuse([(p["est"]["labels"], p["est"]["states"]) for p in per], K)   # Step 4
    res = []
    for j, p in enumerate(per):                                                # Step 5
        n_out = int(n_out_rule(j, p["est"]["LT"]))
        U = group_U(m.seed, k, j, 3, K)
        anc, W = resample(p["w_upd"], U, n_out)
        res.append((p["pred"][:, anc].copy(), np.full(n_out, W / n_out if n_out else 0.0), anc, U, n_out))
    n_min = min(r[4] for r in res)
    L = L_param if L_param > 0 else n_min // 10
    L = min(L, n_min // 2) if K > 1 else 0
    slots = [ring_slots(m.seed, k, j, res[j][4], L, K) if L > 0 else [] for j in range(K)]
    new = [(r[0].copy(), r[1].copy()) for r in res]
    for j in range(K):                                                         # Step 6 (ring)
        src = (j - 1) % K
        for i in range(L):
            new[j][0][:, slots[j][i]] = res[src][0][:, slots[src][i]]
            new[j][1][slots[j][i]] = res[src][1][slots[src][i]]
    return {"groups": per, "fused": fused, "resampled": res, "L": L, "slots": slots, "next": new,
            "W": sum(p["W"] for p in per), "LT": round_half_away(sum(p["W"] for p in per))}
