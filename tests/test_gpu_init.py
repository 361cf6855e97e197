"""phd_init_population (t = 0; reading S23) against the oracle's
orc_init_population: bit-exact states and weights (the arithmetic is fp64 with one
rounding to fp32 on both sides; the inside test of the mass box is taken on the
stored fp32 positions on both sides), -m gpu."""
import threading
from dataclasses import replace

import numpy as np
import pytest

import scenario
from scenario.configs import Model, POSITION, RANGE_BEARING, COUNT_FIXED, COUNT_ADAPTIVE

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def phd():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1503_03769_b200 as p
    p.load()
    return p


POS = Model(meas=POSITION, fixed_count=100003, births_per_step=997, capacity=101000, count_mode=COUNT_FIXED,
            seed=5)
RB = Model(meas=RANGE_BEARING, sigma_z=(10.0, 0.01), region=(0.0, 2000.0, -np.pi, np.pi), sensor_xy=(30.0, -40.0),
           fixed_count=70001, births_per_step=512, capacity=71000, count_mode=COUNT_FIXED, seed=9)


def _oracle(orc, m, n_out, box, mass, mbox, v_max, lo=0, hi=None):
    soa, w, _ = orc.init_population(m, n_out, box, v_max, mass, mass_box=mbox, g_lo=lo, g_hi=hi)
    return soa.astype(np.float32), w.astype(np.float32)


@pytest.mark.parametrize("m,box,mbox,mass", [
    (POS, None, None, 3.0),
    (POS, (-500.0, 1500.0, 0.0, 1000.0), (0.0, 1000.0, 0.0, 1000.0), 1024.0),
    (POS, None, (5000.0, 6000.0, 0.0, 1.0), 2.0),   # empty mass box: all weights 0
    (POS, None, None, 0.0),
    (RB, None, None, 10.0),                          # default box: side r_max around the sensor
])
def test_init_population_parity(phd, orc, m, box, mbox, mass):
    f = phd.Filter(m)
    f.init_population(mass, box=box, mass_box=mbox, v_max=17.5)
    s, w, g0 = f.get_particles()
    b = box
    if b is None:
        b = m.region if m.meas == POSITION else (30.0 - 1000.0, 30.0 + 1000.0, -40.0 - 1000.0, -40.0 + 1000.0)
    so, wo = _oracle(orc, m, m.fixed_count, b, mass, mbox, 17.5)
    assert g0 == 0 and s.shape == so.shape
    assert np.array_equal(s, so)
    assert np.array_equal(w, wo)
    # the population steps like any other: predict at k = 1 (uniform births)
    f.predict(1)
    f.close()


def test_init_population_adaptive_count(phd, orc):
    m = replace(POS, count_mode=COUNT_ADAPTIVE, particles_per_target=1000, births_per_step=200, capacity=50000)
    f = phd.Filter(m)
    f.init_population(2.5)  # round half away: 3 targets -> 3000 particles
    s, w, _ = f.get_particles()
    so, wo = _oracle(orc, m, 3000, m.region, 2.5, None, 20.0)
    assert np.array_equal(s, so) and np.array_equal(w, wo)
    f.init_population(1e6)  # clamped to capacity - J
    s, w, _ = f.get_particles()
    assert s.shape[1] == 50000 - 200
    f.close()


def _par(fs, fn):
    errs = []

    def drive(r):
        try:
            fn(r, fs[r])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=drive, args=(r,)) for r in range(len(fs))]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not errs, errs


@pytest.mark.parametrize("world", [2, 3])
def test_init_population_ranks(phd, orc, world):
    """Every rank generates its block of the same global population; the mass-box count
    is summed over ranks (one all-reduce), so the weights equal the 1-rank oracle's."""
    m = POS
    mb = (0.0, 1000.0, 0.0, 1000.0)
    group = phd.LocalGroup(world)
    fs = [phd.Filter(m, rank=r, world=world, group=group) for r in range(world)]
    _par(fs, lambda r, f: f.init_population(1024.0, mass_box=mb))
    parts = sorted((f.get_particles() for f in fs), key=lambda t: t[2])
    s = np.concatenate([p[0] for p in parts], axis=1)
    w = np.concatenate([p[1] for p in parts])
    so, wo = _oracle(orc, m, m.fixed_count, m.region, 1024.0, mb, 20.0)
    assert np.array_equal(s, so) and np.array_equal(w, wo)
    for r, (ps, pw, g0) in enumerate(parts):
        lo, hi = phd.rank_block(m.fixed_count + m.births_per_step, world, r)
        assert g0 == lo and ps.shape[1] == min(hi, m.fixed_count) - min(lo, m.fixed_count)
    for f in fs:
        f.close()
    group.close()


def test_init_population_dcp_groups(phd, orc):
    """DCP: group j holds block j of the population with its own mass."""
    world = 2
    m = replace(POS, mode=1)
    group = phd.LocalGroup(world)
    fs = [phd.Filter(m, rank=r, world=world, group=group) for r in range(world)]
    _par(fs, lambda r, f: f.init_population(4.0))
    for r, f in enumerate(fs):
        s, w, _ = f.get_particles()
        lo, hi = phd.rank_block(m.fixed_count, world, r)
        so, wo = _oracle(orc, m, m.fixed_count, m.region, 4.0, None, 20.0, lo, hi)
        assert np.array_equal(s, so) and np.array_equal(w, wo)
    for f in fs:
        f.close()
    group.close()


def test_init_population_full_size_cfg5(phd, orc):
    """The bench's t = 0 population (cfg 5, 2^24 - 65,536 particles, mass box): bit-exact."""
    cfg = scenario.get("cfg5")
    ia = scenario.init_args(cfg)
    f = phd.Filter(cfg.model)
    f.init_population(**ia)
    s, w, _ = f.get_particles()
    so, wo = _oracle(orc, cfg.model, cfg.model.fixed_count, ia["box"], ia["total_mass"], ia["mass_box"], ia["v_max"])
    assert np.array_equal(s, so) and np.array_equal(w, wo)
    f.close()


def test_init_population_errors(phd):
    f = phd.Filter(POS)
    for kw in [dict(total_mass=-1.0), dict(total_mass=float("nan")), dict(total_mass=1.0, v_max=-1.0),
               dict(total_mass=1.0, box=(1.0, 1.0, 0.0, 1.0))]:
        with pytest.raises(phd.PhdError) as e:
            f.init_population(**kw)
        assert e.value.status == 1
    f.close()
