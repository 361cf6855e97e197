"""Run-to-run determinism (-m gpu): the same inputs give the same bits.  Every reduction
of the path has a fixed order (fp64 partials per CTA summed in CTA order, label-sorted
entries in the gated path, the multi-CTA resampling scan's chunk totals added in order
by the last CTA), no floating-point atomics; so two filters stepping the same
measurements must agree exactly: particles, weights, ancestors, estimates, summaries."""
from dataclasses import replace

import numpy as np
import pytest

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


def _trace(phd, cfg, steps):
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    f = phd.Filter(cfg.model)
    f.init_population(**scenario.init_args(cfg, truth))
    out = []
    for k in range(1, steps + 1):
        f.step(k, Z[k - 1])
        p, w, _ = f.get_particles()
        a, _ = f.ancestors()
        e = f.estimates()
        out.append((f._sum.as_dict(), p, w, a, e["labels"], e["states"], e["mass"]))
    f.close()
    return out


@pytest.mark.parametrize("cname,gate,steps", [("cfg2", 0, 8), ("cfg3", 0, 4), ("cfg3", 1, 4), ("cfg4", 0, 2),
                                              ("cfg4", 1, 2)])
def test_same_inputs_same_bits(phd, cname, gate, steps):
    base = scenario.get(cname)
    cfg = replace(base, model=replace(base.model, gate=gate))
    r1 = _trace(phd, cfg, steps)
    r2 = _trace(phd, cfg, steps)
    for k, (a, b) in enumerate(zip(r1, r2)):
        assert a[0] == b[0], (k, a[0], b[0])
        for x, y in zip(a[1:], b[1:]):
            assert np.array_equal(x, y), k
