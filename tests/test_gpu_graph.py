"""One-sync and CUDA-graph steps (-m gpu).  With one rank, phd_step computes the
resampling count / offset / mass on the device and synchronises once (the default,
DESIGN.md §4 "one-sync step"); with PHD_GRAPH=1 and a dense update it replays a captured
graph of its whole kernel chain.  Both must be bitwise the classic step (PHD_ONESYNC=0:
host-computed resampling scalars, a synchronisation before the resampling): the same
kernels with the same arguments, the per-step scalars read from the device.  Configs with varying M (cfg 1-3), the adaptive count (cfg 1, 2), range-bearing
(cfg 2), fixed count (cfg 3), host and device measurement pointers."""
import numpy as np
import pytest
from dataclasses import replace

import scenario

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def phd():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1503_03769_b200 as p
    p.load()
    return p


def _run(phd, cfg, steps, graph, monkeypatch, device_z=False, onesync=True):
    import torch
    monkeypatch.setenv("PHD_GRAPH", "1" if graph else "0")
    monkeypatch.setenv("PHD_ONESYNC", "1" if onesync else "0")
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    f = phd.Filter(cfg.model)
    f.init_population(**scenario.init_args(cfg, truth))
    out = []
    for k in range(1, steps + 1):
        if device_z:
            zt = torch.from_numpy(Z[k - 1]).cuda()
            f.step_raw(k, zt.data_ptr(), len(Z[k - 1]))
        else:
            f.step(k, Z[k - 1])
        s = f._sum.as_dict()
        e = f.estimates()
        a, _ = f.ancestors()
        p, w, _ = f.get_particles()
        out.append((s, e, a, p, w, f.resample_meta()))
    stats = f.graph_stats()
    f.close()
    return out, stats


@pytest.mark.parametrize("cname,device_z", [("cfg1", False), ("cfg2", False), ("cfg3", False), ("cfg3", True)])
def test_graph_step_equals_eager(phd, cname, device_z, monkeypatch):
    cfg = scenario.get(cname)
    steps = min(cfg.scenario.steps, 12)
    ref, st0 = _run(phd, cfg, steps, False, monkeypatch, onesync=False)
    one, _ = _run(phd, cfg, steps, False, monkeypatch, device_z)
    got, st1 = _run(phd, cfg, steps, True, monkeypatch, device_z)
    assert st0 == (0, 0)
    assert st1[1] == steps and 1 <= st1[0] <= steps  # every step replayed a graph
    for k, ((s0, e0, a0, p0, w0, m0), (s1, e1, a1, p1, w1, m1), (s2, e2, a2, p2, w2, m2)) in \
            enumerate(zip(ref, got, one)):
        assert s2 == s0 and np.array_equal(e2["labels"], e0["labels"]) and np.array_equal(e2["states"], e0["states"])
        assert np.array_equal(a2, a0) and np.array_equal(p2, p0) and np.array_equal(w2, w0) and m2["U"] == m0["U"]
        for key in ("W", "W_pred", "LT", "N", "N_out", "M", "n_est", "zero_mass", "count_clamped"):
            assert s0[key] == s1[key], (k, key, s0[key], s1[key])
        assert np.array_equal(e0["labels"], e1["labels"]) and np.array_equal(e0["states"], e1["states"])
        assert np.array_equal(a0, a1) and np.array_equal(p0, p1) and np.array_equal(w0, w1)
        assert m0["U"] == m1["U"] and m0["W"] == m1["W"] and m0["N_out"] == m1["N_out"]


def test_graph_step_zero_mass_and_stphd_all(phd, monkeypatch):
    """stphd_all = 1 (LT from W, no index set) and a zero-mass population (the resampling
    spread decided on the device)."""
    base = scenario.get("cfg3")
    cfg = replace(base, model=replace(base.model, stphd_all=1, birth_mass=0.0, births_per_step=0))
    for graph in (False, True):
        monkeypatch.setenv("PHD_GRAPH", "1" if graph else "0")
        monkeypatch.setenv("PHD_ONESYNC", "1" if graph else "0")
        truth = scenario.simulate_truth(cfg)
        Z = scenario.measurements(cfg, truth)
        f = phd.Filter(cfg.model)
        f.init_population(0.0)  # zero mass
        f.step(1, Z[0])
        s = f._sum.as_dict()
        a, _ = f.ancestors()
        if not graph:
            ref = (s, a)
        else:
            assert f.graph_stats()[1] == 1
            assert s["zero_mass"] == ref[0]["zero_mass"] == 1 and np.array_equal(a, ref[1])
        f.close()


def test_onesync_more_estimates_than_eager_copy(phd, monkeypatch):
    """LT above the 256 estimates k_step_out stores with the step's results: the rest
    are copied after the synchronisation; bitwise the classic step."""
    base = scenario.get("cfg3")
    cfg = replace(base, scenario=replace(base.scenario, n_targets=420, steps=3))
    ref, _ = _run(phd, cfg, 3, False, monkeypatch, onesync=False)
    one, _ = _run(phd, cfg, 3, False, monkeypatch, onesync=True)
    assert max(s["n_est"] for s, *_ in ref) > 256
    for (s0, e0, a0, p0, w0, m0), (s1, e1, a1, p1, w1, m1) in zip(ref, one):
        assert s0 == s1 and np.array_equal(e0["labels"], e1["labels"]) and np.array_equal(e0["states"], e1["states"])
        assert np.array_equal(e0["mass"], e1["mass"]) and np.array_equal(a0, a1) and np.array_equal(w0, w1)


@pytest.mark.parametrize("onesync", [False, True])
def test_nan_measurement_reported_then_cleared(phd, monkeypatch, onesync):
    """A NaN measurement makes C non-finite: the step reports PHD_EMODEL (the one-sync
    step through k_step_out's flags).  The counters start from zero again for the next
    filter step (k_step_out clears them; the classic update clears them first)."""
    monkeypatch.setenv("PHD_ONESYNC", "1" if onesync else "0")
    cfg = scenario.get("cfg3")
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    f = phd.Filter(cfg.model)
    f.init_population(**scenario.init_args(cfg, truth))
    f.step(1, Z[0])
    zbad = Z[1].copy()
    zbad[3, 0] = np.nan
    with pytest.raises(RuntimeError, match="non-finite"):
        f.step(2, zbad)
    f.close()
    g = phd.Filter(cfg.model)  # a fresh filter on the same device: no stale flag
    g.init_population(**scenario.init_args(cfg, truth))
    g.step(1, Z[0])
    g.step(2, Z[1])
    g.close()
