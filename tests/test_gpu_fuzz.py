"""Seeded randomized parity sweep (-m gpu): one update + extraction + resampling on
random sizes and options against the oracle, so that the layout machinery (tile sizes,
ZL / warps / z-blocks, the per-warp state-sum layout and its two pass-2 instances,
whole-z-block layouts, the gated path, ragged tails) is exercised at combinations the
hand-written cases do not name.  Tolerances are those of test_gpu_parity.py."""
import math
import os
from dataclasses import replace

import numpy as np
import pytest

from test_gpu_parity import MODELS, _meas, _cloud, _check_update, _near_ties

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def phd():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1503_03769_b200 as p
    p.load()
    return p

CASES = int(os.environ.get("PHD_FUZZ_CASES", "48"))  # longer sweeps: PHD_FUZZ_CASES=400


def _case(i):
    r = np.random.default_rng(1000 + i)
    mname = ["position", "range_bearing", "aniso"][r.integers(3)]
    n = int(r.choice([1, 7, 255, 257, 1000, 4099, 20011, 65537]) + r.integers(0, 300))
    M = int(r.choice([1, 2, 31, 130, 600, 1100, 2047, 3001, 4090]))
    env = {}
    if r.random() < 0.4:
        env["PHD_TILE"] = str(r.choice([64, 256]))
    if r.random() < 0.4:
        env["PHD_JS_SPLIT"] = str(r.integers(2))
    if r.random() < 0.25:
        env["PHD_SUM_LAYOUT"] = str(r.choice(["lane", "zblock"]))
    gate = int(r.choice([0, 0, 2]))
    stphd_all = int(r.integers(2))
    clutter = float(r.choice([5.0, 50.0, 500.0]))
    return mname, n, M, env, gate, stphd_all, clutter, int(r.integers(1 << 30))


@pytest.mark.parametrize("i", range(CASES))
def test_random_update_extract_resample(phd, orc, i, monkeypatch, near_tie_report):
    mname, n, M, env, gate, stphd_all, clutter, seed = _case(i)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    m = replace(MODELS[mname], gate=gate, stphd_all=stphd_all, clutter_rate=clutter, capacity=max(1 << 16, n + 1024))
    z = _meas(m, M, seed % 997)
    soa, w = _cloud(m, n, z, seed % 991)
    f = phd.Filter(m)
    f.set_particles(soa, w, soa.shape[1], stage=phd.STAGE_PREDICTED)
    f.update(z)
    C = f.normalizers(M)
    acc = f.accumulators(M)
    _, wn, _ = f.get_particles()
    est, summ = f.extract()
    Co = orc.normalizers(m, soa, w, z)
    wo, acco = orc.update(m, soa, w, z, Co)
    _check_update(orc, m, C, acc, wn, w, Co, wo, acco)
    kap = orc.kappa(m)
    rhs = (1 - m.p_d) * math.fsum(w.astype(np.float64)) + math.fsum(Co / (kap + Co))
    assert abs(summ["W"] - rhs) <= 2e-6 * max(rhs, 1e-30) + 1e-12
    # extraction on the GPU accumulators equals the oracle's selection on them
    eg = orc.extract(m, acc, summ["W"], summ["W_pred"])
    if not summ["near_half"]:
        assert list(est["labels"]) == list(eg["labels"])
        assert np.allclose(est["states"], eg["states"], rtol=1e-6, atol=1e-4)
    # resampling: every ancestor vs the oracle's, mismatches only at counted near-ties
    f.resample_exchange(3)
    anc, _ = f.ancestors()
    meta = f.resample_meta()
    ao, _ = orc.resample(wn.astype(np.float64), meta["U"], meta["N_out"])
    mism = anc != ao
    ties = _near_ties(wn, meta["U"], meta["N_out"])
    assert not np.any(mism & ~ties), int(np.sum(mism & ~ties))
    if mism.any():
        near_tie_report(n_out=int(meta["N_out"]), mismatches=int(mism.sum()), near_ties=int(ties.sum()),
                        non_tie_mismatches=0)
    f.close()


MR_CASES = int(os.environ.get("PHD_FUZZ_MR_CASES", "12"))


@pytest.mark.parametrize("i", range(MR_CASES))
def test_random_multirank_against_oracle(phd, orc, i, monkeypatch):
    """P in-process ranks (2-4, uneven blocks, sometimes a rank with no particles) on random
    sizes: the global C, every rank's weights, the accumulators, and the concatenated
    ancestors of the rank-local resampling + exchange against the oracle."""
    from test_gpu_multirank import _parallel
    r = np.random.default_rng(5000 + i)
    world = int(r.integers(2, 5))
    mname = ["position", "range_bearing"][r.integers(2)]
    n = int(r.choice([world - 1, 300, 5000, 30011]) + r.integers(0, 50))
    M = int(r.choice([3, 130, 700, 2500]))
    gate = int(r.choice([0, 2]))
    if r.random() < 0.5:
        monkeypatch.setenv("PHD_EXCHANGE", "nccl")
    m = replace(MODELS[mname], gate=gate, stphd_all=0, max_meas=4096)
    z = _meas(m, M, 31 + i)
    soa, w = _cloud(m, n, z, 37 + i)
    group = phd.LocalGroup(world)
    fs = [phd.Filter(m, rank=q, world=world, group=group) for q in range(world)]
    for q, f in enumerate(fs):
        lo, hi = phd.rank_block(n, world, q)
        f.set_particles(np.ascontiguousarray(soa[:, lo:hi]), np.ascontiguousarray(w[lo:hi]), n,
                        stage=phd.STAGE_PREDICTED)
    _parallel(fs, lambda q, f: f.update(z))
    C = fs[0].normalizers(M)
    acc = fs[0].accumulators(M)
    wn = np.concatenate([fs[q].get_particles()[1] for q in range(world)])
    _parallel(fs, lambda q, f: f.extract())
    Co = orc.normalizers(m, soa, w, z)
    wo, acco = orc.update(m, soa, w, z, Co)
    _check_update(orc, m, C, acc, wn, w, Co, wo, acco)
    _parallel(fs, lambda q, f: f.resample_exchange(4))
    parts = sorted((f.ancestors()[1], f.ancestors()[0]) for f in fs)
    anc = np.concatenate([a for _, a in parts])
    meta = fs[0].resample_meta()
    ao, _ = orc.resample(wn.astype(np.float64), meta["U"], meta["N_out"])
    mism = anc != ao
    assert not np.any(mism & ~_near_ties(wn, meta["U"], meta["N_out"]))
    for f in fs:
        f.close()
    group.close()
