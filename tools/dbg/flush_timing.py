"""Debug: per-stage device timings of cfg3 steps with and without the bench's L2 flush."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch, scenario, paper_1503_03769_b200 as phd
cfg = scenario.get(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
truth = scenario.simulate_truth(cfg); Z = scenario.measurements(cfg, truth)
soa, w = scenario.initial_population(cfg, truth)
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)
f = phd.Filter(cfg.model, stream=stream.cuda_stream)
f.set_particles(soa, w, soa.shape[1]); f.set_timing(True)
Zd = [torch.from_numpy(z).to(dev) for z in Z]
buf = torch.empty(252 << 20, dtype=torch.uint8, device=dev)
names = ["predict", "pass1", "pass2", "update", "extract", "resample", "exchange", "step"]
k = 0
for mode in ("none", "flush", "flush+sync", "none"):
    rows = []
    for it in range(8):
        k += 1
        if mode.startswith("flush"):
            buf.zero_()
        if mode == "flush+sync":
            torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        f.step_raw(k, Zd[k - 1].data_ptr(), int(Zd[k - 1].shape[0]))
        a1.record(stream)
        torch.cuda.synchronize()
        rows.append([a0.elapsed_time(a1)] + list(f.timing().values()))
    r = np.median(np.array(rows[2:]), 0)
    print("%-11s step(ev) %.4f  " % (mode, r[0]) + "  ".join("%s %.4f" % (n, v) for n, v in zip(names, r[1:])))
