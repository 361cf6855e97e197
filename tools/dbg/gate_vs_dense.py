"""Debug: at each step of a dense cfg trajectory, run the gated update on the
same predicted particles and compare C and w' (position of the largest gaps)."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, scenario, paper_1503_03769_b200 as phd
from dataclasses import replace
cname = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = scenario.get(cname)
truth = scenario.simulate_truth(cfg); Z = scenario.measurements(cfg, truth)
soa, w = scenario.initial_population(cfg, truth)
fd = phd.Filter(replace(cfg.model, gate=0)); fd.set_particles(soa, w, soa.shape[1])
for k in range(1, steps + 1):
    z = Z[k - 1]
    fd.predict(k)
    ps, pw, _ = fd.get_particles()
    fd.update(z)
    Cd = fd.normalizers(len(z)); _, wd, _ = fd.get_particles()
    fg = phd.Filter(replace(cfg.model, gate=2)); fg.set_particles(ps, pw, ps.shape[1], stage=phd.STAGE_PREDICTED)
    fg.update(z)
    Cg = fg.normalizers(len(z)); _, wg, _ = fg.get_particles(); gs = fg.gate_stats(); fg.close()
    rc = np.abs(Cg - Cd) / np.maximum(Cd, 1e-300)
    rw = np.abs(wg - wd) / np.maximum(wd, 1e-30)
    i = int(np.argmax(rc)); j = int(np.argmax(rw))
    print("k=%d M=%d gate=%s  C maxrel %.3e at %d (Cd=%.3e Cg=%.3e z=%s)  w maxrel %.3e at %d (wd=%.3e wg=%.3e x=%s)" % (
        k, len(z), gs, rc[i], i, Cd[i], Cg[i], z[i], rw[j], j, wd[j], wg[j], ps[:, j]))
    print("   count C rel>1e-5: %d, w rel>1e-4: %d" % ((rc > 1e-5).sum(), (rw > 1e-4).sum()))
    fd.extract(); fd.resample_exchange(k)
