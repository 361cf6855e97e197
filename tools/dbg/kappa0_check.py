"""kappa = 0 (no clutter) with measurements far from every particle: dense vs gated vs the oracle (probe)."""
import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, math
from dataclasses import replace
import paper_1503_03769_b200 as phd, oracle as orc
from test_gpu_parity import MODELS, _meas, _cloud
for mname in ("position", "range_bearing"):
    m0 = replace(MODELS[mname], clutter_rate=0.0, stphd_all=0)
    z = _meas(m0, 300, 5)
    soa, w = _cloud(m0, 30011, z[:200], 5)   # 100 measurements with no particles near them
    res = {}
    for gate in (0, 2):
        m = replace(m0, gate=gate)
        f = phd.Filter(m)
        f.set_particles(soa, w, soa.shape[1], stage=phd.STAGE_PREDICTED)
        f.update(z)
        C = f.normalizers(len(z)); _, wn, _ = f.get_particles(); est, s = f.extract()
        res[gate] = (C, wn, s)
        f.close()
    Co = orc.normalizers(m0, soa, w, z)
    wo, acco = orc.update(m0, soa, w, z, Co)
    for gate in (0, 2):
        C, wn, s = res[gate]
        rel = np.abs(wn - wo) / np.maximum(wo, 1e-30)
        print(mname, "gate", gate, "W", s["W"], "W_oracle", float(np.sum(wo)), "max rel w err", float(rel.max()),
              "n C=0", int(np.sum(C == 0)), "oracle C<1e-30", int(np.sum(Co < 1e-30)), "finite", bool(np.all(np.isfinite(wn))))
