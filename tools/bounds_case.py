"""Small runs through every kernel (both sensors, the dense passes,
zero mass, M = 0, the gated path with multi-chunk tiles and M > 4096).  Run with
PHD_LIB pointing at the -DPHD_DEBUG_BOUNDS build (tests/test_gpu_debug_bounds.py):
every device bounds check traps on a violation."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, scenario, paper_1503_03769_b200 as phd
from dataclasses import replace
# small runs through every kernel: position + range-bearing, zero mass, M=0
for name in ("cfg1", "cfg2"):
    cfg = scenario.get(name); m = cfg.model
    Z = scenario.measurements(cfg); soa, w = scenario.initial_population(cfg)
    f = phd.Filter(m); f.set_particles(soa, w, soa.shape[1])
    for k in range(1, 4):
        f.step(k, Z[k-1])
    f.predict(4); f.update(np.zeros((0, 2), np.float32)); f.extract(); f.resample_exchange(4)
    f.close()
m = replace(scenario.get("cfg3").model, fixed_count=3000, births_per_step=256, capacity=4096, max_meas=4096)
z = scenario.random_measurements(2600, 3)
soa, w = scenario.random_particles(3256, 4)
f = phd.Filter(m); f.set_particles(soa, w, 3256, stage=phd.STAGE_PREDICTED); f.update(z); f.extract(); f.resample_exchange(1); f.close()
w[:] = 0
f = phd.Filter(m); f.set_particles(soa, w, 3256, stage=phd.STAGE_PREDICTED); f.update(z); f.extract(); f.resample_exchange(1); f.close()
# gated update (gate = 2): both sensors, a chunk of > 256 candidates per tile, M > 4096
# (two-pass label sort), zero-weight tiles, ragged tail
for meas_cfg in ("cfg3", "cfg4"):
    base = scenario.get(meas_cfg).model
    mg = replace(base, gate=2, fixed_count=6000, births_per_step=512, capacity=8192, max_meas=8192)
    z = scenario.random_measurements(5000, 7, meas=mg.meas, region=mg.region)
    soa, w = scenario.clustered_particles(6512, z, 7, meas=mg.meas, sensor=mg.sensor_xy,
                                          box=(-1000.0, 1000.0, -1000.0, 1000.0))
    w[1000:1600] = 0
    f = phd.Filter(mg); f.set_particles(soa, w, 6512, stage=phd.STAGE_PREDICTED); f.update(z)
    print("gated", meas_cfg, f.gate_stats()); f.extract(); f.resample_exchange(1); f.close()
print("bounds case done")
