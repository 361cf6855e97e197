import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, scenario, paper_1503_03769_b200 as phd
from dataclasses import replace
# small runs through every kernel: position + range-bearing, fused + two-sweep, zero mass, M=0
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
os.environ["PHD_FUSE"] = "1"
f = phd.Filter(m); f.set_particles(soa, w, 3256, stage=phd.STAGE_PREDICTED); f.update(z); f.extract(); f.resample_exchange(1); f.close()
os.environ["PHD_FUSE"] = "0"
w[:] = 0
f = phd.Filter(m); f.set_particles(soa, w, 3256, stage=phd.STAGE_PREDICTED); f.update(z); f.extract(); f.resample_exchange(1); f.close()
print("sanitizer case done")
