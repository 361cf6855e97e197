"""Multi-rank path of the library on one GPU (-m gpu).

`world` contexts of one process form an in-process rank group (phd_group:
host barriers + device-to-device copies in place of NCCL); one
host thread drives each rank, so the exact multi-rank orchestration of
phd_update (C1/C2 all-reduces, per-rank mass slots) and phd_resample_exchange
(rank-local exact resampling, planner, exchange) runs.  Results must be
P-invariant: equal to the world = 1 run up to fp64 summation order (counted
near-ties in the resampling) -- and the P = 1 run is itself pinned to the
oracle by test_gpu_parity.py.
"""
import threading
from dataclasses import replace

import numpy as np
import pytest

import scenario
from scenario.configs import COUNT_FIXED

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def phd():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1503_03769_b200 as p
    p.load()
    return p


def _cfg(meas="cfg3"):
    cfg = scenario.get(meas)
    m = replace(cfg.model, fixed_count=60000, births_per_step=4096, capacity=64096, count_mode=COUNT_FIXED,
                max_meas=4096)
    s = replace(cfg.scenario, n_targets=40, steps=4, init_mass_box=(0.0, 1000.0, 0.0, 1000.0),
                start_box=(0.0, 1000.0, 0.0, 1000.0))
    if cfg.model.meas == 1:
        s = replace(s, init_mass_box=None)
    return replace(cfg, model=m, scenario=s)


def _run(phd, cfg, world, steps):
    m = cfg.model
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    group = phd.LocalGroup(world) if world > 1 else None
    fs = [phd.Filter(m, rank=r, world=world, group=group) for r in range(world)]
    ia = scenario.init_args(cfg, truth)
    out = {"summ": [], "est": [], "anc": [], "pop": []}
    errs = []

    def init(r):
        try:
            fs[r].init_population(**ia)  # t = 0 on the device, collective (mass-box count)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=init, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not errs, errs

    def drive(r, k):
        try:
            fs[r].step(k, Z[k - 1])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    for k in range(1, steps + 1):
        th = [threading.Thread(target=drive, args=(r, k)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        assert not errs, errs
        out["summ"].append(fs[0]._sum.as_dict())
        out.setdefault("xpath", set()).add(fs[0].exchange_path())
        out["est"].append(fs[0]._estimates())
        anc = []
        for f in fs:
            a, first = f.ancestors()
            anc.append((first, a))
        out["anc"].append(np.concatenate([a for _, a in sorted(anc, key=lambda t: t[0])]))
        parts = [f.get_particles() for f in fs]
        parts.sort(key=lambda t: t[2])
        out["pop"].append((np.concatenate([p[0] for p in parts], axis=1), np.concatenate([p[1] for p in parts])))
    for f in fs:
        f.close()
    if group is not None:
        group.close()
    return out


@pytest.mark.parametrize("cname", ["cfg3", "cfg4"])
@pytest.mark.parametrize("world,gate,xch", [(2, 0, "p2p"), (3, 0, "p2p"), (4, 0, "p2p"), (2, 2, "p2p"), (3, 1, "p2p"),
                                            (3, 0, "nccl"), (4, 2, "nccl")])
def test_p_invariance(phd, cname, world, gate, xch, monkeypatch):
    """gate = 1/2: the gated update (collective gated/dense decision, per-rank
    tiles) against its own world = 1 run.  xch: the fused gather + exchange over
    the peer-memory window (default) or the send/recv exchange (PHD_EXCHANGE=nccl)."""
    if xch == "nccl":
        monkeypatch.setenv("PHD_EXCHANGE", "nccl")
    cfg = _cfg(cname)
    cfg = replace(cfg, model=replace(cfg.model, gate=gate))
    steps = 3
    ref = _run(phd, cfg, 1, steps)
    got = _run(phd, cfg, world, steps)
    assert got["xpath"] == {2 if xch == "p2p" else 1}
    identical_so_far = True
    for k in range(steps):
        s1, sp = ref["summ"][k], got["summ"][k]
        a1, ap = ref["anc"][k], got["anc"][k]
        p1, pp = ref["pop"][k], got["pop"][k]
        e1, ep = ref["est"][k], got["est"][k]
        assert s1["N"] == sp["N"] and len(a1) == len(ap) == cfg.model.fixed_count
        assert np.all(np.diff(ap) >= 0) and p1[0].shape == pp[0].shape
        if identical_so_far:
            # same inputs: only the fp64 summation order differs (C, W per rank
            # partition; d = 1/D may round to a neighbouring fp32)
            assert abs(s1["W"] - sp["W"]) <= 1e-6 * max(1.0, s1["W"])
            assert s1["LT"] == sp["LT"] or s1["near_half"]
            assert len(e1["labels"]) == len(ep["labels"])
            same = e1["labels"] == ep["labels"]
            assert np.mean(same) >= 0.99
            assert np.all(np.abs(e1["states"][same] - ep["states"][same]) <= 1e-3)
            # ancestors: equal except thresholds within rounding of a cumsum boundary.  The
            # rank partition changes C in its last fp64 bits; 1/D rounds to a neighbouring
            # fp32 now and then, and pass 2 folds log2(1/D) into the exponent,
            # where one ulp of the folded constant moves a slot's terms by <= 1e-6 relative:
            # offspring boundaries that close to a threshold may go to the neighbour
            assert np.mean(a1 != ap) <= 4e-4, int(np.sum(a1 != ap))
            same_pop = np.all(p1[0] == pp[0], axis=0)
            assert np.mean(same_pop) >= 1.0 - 4e-4
            identical_so_far = bool(np.all(a1 == ap))
        else:
            # a near-tie changed an ancestor earlier: the filters stay statistically equal
            assert abs(s1["W"] - sp["W"]) <= 1e-2 * max(1.0, s1["W"])


def test_exchange_moves_mass_to_every_rank(phd):
    """cfg-5-style imbalance: all initial mass on the upper ranks; after one step
    every rank holds its equal block of equal-weight offspring."""
    cfg = _cfg("cfg3")
    world = 4
    m = cfg.model
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    soa, w = scenario.initial_population(cfg, truth)
    n0 = soa.shape[1]
    masses = [float(w[min(lo, n0):min(hi, n0)].astype(np.float64).sum())
              for lo, hi in (phd.rank_block(n0 + m.births_per_step, world, r) for r in range(world))]
    assert masses[0] == 0.0 and masses[-1] > 0  # imbalanced start
    group = phd.LocalGroup(world)
    fs = [phd.Filter(m, rank=r, group=group) for r in range(world)]
    for r, f in enumerate(fs):
        lo, hi = phd.rank_block(n0 + m.births_per_step, world, r)
        f.set_particles(np.ascontiguousarray(soa[:, min(lo, n0):min(hi, n0)]),
                        np.ascontiguousarray(w[min(lo, n0):min(hi, n0)]), n0)
    th = [threading.Thread(target=lambda f=f: f.step(1, Z[0])) for f in fs]
    [t.start() for t in th]
    [t.join() for t in th]
    W = fs[0]._sum.W
    for r, f in enumerate(fs):
        s, ww, g0 = f.get_particles()
        lo, hi = phd.rank_block(m.fixed_count + m.births_per_step, world, r)
        assert g0 == lo and s.shape[1] == min(hi, m.fixed_count) - min(lo, m.fixed_count)
        assert np.allclose(ww, W / m.fixed_count, rtol=1e-6)
    for f in fs:
        f.close()
    group.close()


@pytest.mark.parametrize("gate", [0, 2])
def test_rank_with_no_particles(phd, gate):
    """Tiny population over 4 ranks: some ranks hold no survivors (and no births) in a step;
    the collectives still line up and the result equals the 1-rank run."""
    from dataclasses import replace as rp
    cfg = _cfg("cfg3")
    m = rp(cfg.model, fixed_count=3, births_per_step=2, capacity=64, max_meas=4096, gate=gate)
    cfg = rp(cfg, model=m)
    ref = _run(phd, cfg, 1, 2)
    got = _run(phd, cfg, 4, 2)
    for k in range(2):
        assert abs(ref["summ"][k]["W"] - got["summ"][k]["W"]) <= 1e-6 * max(1.0, ref["summ"][k]["W"])
        assert np.array_equal(ref["anc"][k], got["anc"][k])


@pytest.mark.parametrize("gate", [0, 2])
def test_nan_particle_reported_on_every_rank(phd, gate):
    """A NaN particle held by one rank: every rank's step reports PHD_EMODEL (the dense
    C is NaN after C1; the gated sort poisons the rank's W_pred, which C1 spreads)."""
    cfg = _cfg()
    m = replace(cfg.model, gate=gate)
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    soa, w = scenario.initial_population(cfg, truth)
    n0, world = soa.shape[1], 2
    soa[0, n0 - 10] = np.nan  # on the last rank
    soa[2, n0 - 10] = 9000.0
    group = phd.LocalGroup(world)
    fs, status = [], [None] * world
    for r in range(world):
        f = phd.Filter(m, rank=r, world=world, group=group)
        lo, hi = phd.rank_block(n0 + m.births_per_step, world, r)
        a, b = min(lo, n0), min(hi, n0)
        f.set_particles(np.ascontiguousarray(soa[:, a:b]), np.ascontiguousarray(w[a:b]), n0)
        fs.append(f)

    def drive(r):
        try:
            fs[r].step(1, Z[0])
            status[r] = 0
        except phd.PhdError as e:
            status[r] = e.status

    th = [threading.Thread(target=drive, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert status == [4] * world, status
    for f in fs:
        f.close()
    group.close()


def _parallel(fs, fn):
    errs = []

    def drive(r):
        try:
            fn(r, fs[r])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=drive, args=(r,)) for r in range(len(fs))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs


@pytest.mark.parametrize("xch", ["p2p", "nccl"])
def test_rank_local_resampling_equals_oracle_large(phd, orc, xch, monkeypatch, near_tie_report):
    """P = 4 in-process ranks with 1.15 M particles each (rank-local fp64 scans over
    > 1024 weight blocks, > 1024 offspring blocks per rank, imbalanced mass: the lower
    half of the ranks holds 1e-3 of it): the concatenated ancestors equal the oracle's
    sequential systematic resampling of the concatenated updated weights
     except near-ties, which are counted."""
    from scenario.configs import Model, POSITION
    if xch == "nccl":
        monkeypatch.setenv("PHD_EXCHANGE", "nccl")
    world, N, M = 4, 4 * 1150 * 1024, 256
    J = 8192
    m = Model(meas=POSITION, sigma_z=(10.0, 10.0), p_d=0.98, p_s=0.99, clutter_rate=50.0,
              region=(-1000.0, 1000.0, -1000.0, 1000.0), births_per_step=J, fixed_count=N - J,
              count_mode=COUNT_FIXED, capacity=N, max_meas=4096, seed=3)
    z = scenario.random_measurements(M, 9)
    soa, w = scenario.clustered_particles(N, z, 4)
    w = w.astype(np.float64)
    w[: N // 2] *= 1e-3  # ranks 0, 1 carry little mass
    w = (w * (100.0 / w.sum())).astype(np.float32)
    group = phd.LocalGroup(world)
    fs = [phd.Filter(m, rank=r, world=world, group=group) for r in range(world)]
    blocks = [phd.rank_block(N, world, r) for r in range(world)]
    for r, f in enumerate(fs):
        lo, hi = blocks[r]
        f.set_particles(np.ascontiguousarray(soa[:, lo:hi]), np.ascontiguousarray(w[lo:hi]), N,
                        stage=phd.STAGE_PREDICTED)
    _parallel(fs, lambda r, f: f.update(z))
    wn = np.concatenate([fs[r].get_particles()[1] for r in range(world)])
    _parallel(fs, lambda r, f: f.extract())
    k = 2
    _parallel(fs, lambda r, f: f.resample_exchange(k))
    parts = sorted((f.ancestors()[1], f.ancestors()[0]) for f in fs)
    anc = np.concatenate([a for _, a in parts])
    meta = fs[0].resample_meta()
    assert meta["N_out"] == N - J and len(anc) == N - J and np.all(np.diff(anc) >= 0)
    assert fs[0].exchange_path() == (2 if xch == "p2p" else 1)
    from test_gpu_parity import check_ancestors
    check_ancestors(orc, anc, wn, meta["U"], meta["N_out"], near_tie_report, world=world, exchange=xch)
    # the exchanged population: every rank holds its block of the offspring
    for r, f in enumerate(fs):
        s, ww, g0 = f.get_particles()
        lo, hi = phd.rank_block(N, world, r)
        assert g0 == lo and s.shape[1] == min(hi, N - J) - min(lo, N - J)
        assert np.array_equal(s, soa[:, anc[min(lo, N - J):min(hi, N - J)]])
    for f in fs:
        f.close()
    group.close()


@pytest.mark.parametrize("mname", ["position", "range_bearing"])
@pytest.mark.parametrize("world,gate", [(2, 0), (3, 0), (3, 2)])
def test_multirank_update_equals_oracle(phd, orc, mname, world, gate):
    """P ranks (uneven blocks) against the oracle directly, not only against the P = 1 GPU
    run: the global C after the C1 all-reduce, every rank's updated
    weights, the accumulators after the C2 all-reduce and the extracted label set on the
    CU, within the single-device parity tolerances."""
    from test_gpu_parity import MODELS, _meas, _cloud, _check_update
    m = replace(MODELS[mname], max_meas=4096, gate=gate)
    N, M = 3 * 10007 + 2, 600
    z = _meas(m, M, 21)
    soa, w = _cloud(m, N, z, 21)
    group = phd.LocalGroup(world)
    fs = [phd.Filter(m, rank=r, world=world, group=group) for r in range(world)]
    for r, f in enumerate(fs):
        lo, hi = phd.rank_block(N, world, r)
        f.set_particles(np.ascontiguousarray(soa[:, lo:hi]), np.ascontiguousarray(w[lo:hi]), N,
                        stage=phd.STAGE_PREDICTED)
    _parallel(fs, lambda r, f: f.update(z))
    C = fs[0].normalizers(M)
    acc = fs[0].accumulators(M)
    wn = np.concatenate([fs[r].get_particles()[1] for r in range(world)])
    res = {}
    _parallel(fs, lambda r, f: res.__setitem__(r, f.extract()))
    est, summ = res[0]
    Co = orc.normalizers(m, soa, w, z)
    wo, acco = orc.update(m, soa, w, z, Co)
    _check_update(orc, m, C, acc, wn, w, Co, wo, acco)
    # the other ranks hold the same global C
    for f in fs[1:]:
        assert np.array_equal(f.normalizers(M), C)
    import math
    eo = orc.extract(m, acco, math.fsum(wo), math.fsum(w.astype(np.float64)))
    assert summ["LT"] == eo["LT"] or summ["near_half"]
    # label sets agree except near-ties of dW at the selection threshold (S8, as
    # test_extract_parity); states of the common labels within the 1e-3 tolerance
    ga, oa = set(est["labels"].tolist()), set(eo["labels"].tolist())
    if len(eo["labels"]):
        thr = acco[eo["labels"][-1], 0]
        for lab in ga ^ oa:
            assert abs(acco[lab, 0] - thr) <= 1e-5 * thr, (lab, acco[lab, 0], thr)
    for i, lab in enumerate(est["labels"]):
        if lab in oa:
            j = list(eo["labels"]).index(lab)
            assert np.all(np.abs(est["states"][i] - eo["states"][j]) <= 1e-3)
    for f in fs:
        f.close()
    group.close()
