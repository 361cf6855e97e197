"""Pins of the DCPFPHD oracle (oracle/dcp.py; §3; NEXT-1)."""
import math

import numpy as np
import pytest

import scenario
from scenario.configs import Model, POSITION, COUNT_FIXED


def _groups(soa, w, K):
    n = soa.shape[1]
    return [(soa[:, (n * j) // K:(n * (j + 1)) // K], w[(n * j) // K:(n * (j + 1)) // K]) for j in range(K)]


def test_one_group_is_the_serial_filter(orc):
    """SPEC.md:509 acceptance #1: K = 1 reproduces the serial particle PHD step exactly."""
    from oracle import dcp
    cfg = scenario.get("cfg1")
    m = cfg.model
    Z = scenario.measurements(cfg)
    soa, w = scenario.initial_population(cfg)
    soa, w = soa.astype(np.float64), w.astype(np.float64)
    zprev = None
    for k in range(1, 4):
        rule = lambda j, LT: max(LT, 1) * m.particles_per_target
        d = dcp.dcp_step(m, k, [(soa, w)], Z[k - 1], zprev, rule)
        s = orc.step(m, k, soa, w, Z[k - 1], zprev, lambda LT: max(LT, 1) * m.particles_per_target,
                     m.births_per_step)
        g = d["groups"][0]
        assert np.array_equal(g["pred"], s["pred"]) and np.array_equal(g["w_upd"], s["w_upd"])
        assert list(d["fused"][0]) == sorted(s["est"]["labels"].tolist())
        assert np.array_equal(d["resampled"][0][2], s["anc"]) and d["L"] == 0
        soa, w = d["next"][0]
        zprev = Z[k - 1]


def test_fusion_rule_examples():
    """SPEC.md:290-298 (Step 4): strict majority of groups."""
    from oracle import dcp
    st = lambda v: np.full(4, float(v))
    local = [([7, 3], [st(1), st(10)]), ([7], [st(2)]), ([3], [st(20)]), ([7, 5], [st(6), st(0)])]
    labs, states, counts = dcp.fuse(local, 4)
    assert list(labs) == [7] and list(counts) == [3] and np.allclose(states[0], 3.0)  # {1,2,4}: 3 > 2
    labs, _, _ = dcp.fuse(local[:2] + [([3], [st(0)])], 4)  # label 3 by 2 of 4 groups: rejected
    assert 3 not in list(labs)
    labs, states, _ = dcp.fuse([([5, 2], [st(1), st(2)])], 1)  # K = 1: every label valid
    assert list(labs) == [2, 5] and np.allclose(states[1], 1.0)


@pytest.mark.parametrize("K", [2, 3, 4])
def test_ring_exchange_conserves(orc, K):
    """Step 6: counts per group unchanged, mass conserved, and the transferred couples
    appear verbatim in the destination group."""
    from oracle import dcp
    cfg = scenario.get("cfg3")
    m = Model(meas=POSITION, sigma_z=(10.0, 10.0), births_per_step=K * 50, fixed_count=600 * K,
              count_mode=COUNT_FIXED, capacity=1 << 14, clutter_rate=20.0)
    z = scenario.random_measurements(25, 4)
    soa, w = scenario.clustered_particles(600 * K, z, 5)
    soa, w = soa.astype(np.float64), w.astype(np.float64)
    d = dcp.dcp_step(m, 2, _groups(soa, w, K), z, z, lambda j, LT: 600)
    L = d["L"]
    assert L == 60
    tot_before = sum(math.fsum(r[1]) for r in d["resampled"])
    tot_after = sum(math.fsum(g[1]) for g in d["next"])
    assert abs(tot_before - tot_after) <= 1e-12 * tot_before
    for j in range(K):
        src = (j - 1) % K
        assert d["next"][j][0].shape[1] == d["resampled"][j][0].shape[1]
        for i in range(L):
            a = d["next"][j][0][:, d["slots"][j][i]]
            b = d["resampled"][src][0][:, d["slots"][src][i]]
            assert np.array_equal(a, b)
        assert len(set(d["slots"][j])) == L


def test_group_mass_identity(orc):
    """Each group's local update satisfies the north_star identity with its own C_j."""
    from oracle import dcp
    m = Model(meas=POSITION, sigma_z=(10.0, 10.0), births_per_step=300, fixed_count=3000,
              count_mode=COUNT_FIXED, capacity=1 << 14, clutter_rate=20.0)
    z = scenario.random_measurements(30, 8)
    soa, w = scenario.clustered_particles(3000, z, 9)
    d = dcp.dcp_step(m, 1, _groups(soa.astype(np.float64), w.astype(np.float64), 3), z, None, lambda j, LT: 1000)
    kap = orc.kappa(m)
    for g in d["groups"]:
        rhs = (1 - m.p_d) * g["W_pred"] + math.fsum(g["C"] / (kap + g["C"]))
        assert abs(g["W"] - rhs) <= 1e-12 * rhs
