"""bench.py's protocol (init population, 3 warm-up steps, then 10 steps each after an L2
flush + synchronize, events on the legacy stream around phd_step, filter on its own
stream) with device-resident vs pinned-host measurement sets, alternated, plus the host
wall time of each step call.  usage: python tools/dbg/flush_dev_host.py cfg2"""
import os, sys, json, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1503_03769_b200 as phd, scenario
from dataclasses import replace

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = scenario.get(name)
cfg = replace(cfg, scenario=replace(cfg.scenario, steps=max(cfg.scenario.steps, 15)))
truth = scenario.simulate_truth(cfg)
Z = scenario.measurements(cfg, truth)
Zd = [torch.from_numpy(z).cuda() for z in Z]
Zh = [torch.from_numpy(z).pin_memory() for z in Z]
stream = torch.cuda.current_stream()
flush = torch.empty(252 << 20, dtype=torch.uint8, device="cuda")
f = phd.Filter(cfg.model, stream=stream.cuda_stream)
res = {}
for rnd in range(3):
    for mode in ("dev", "host"):
        zs = Zd if mode == "dev" else Zh
        f.init_population(**scenario.init_args(cfg, truth))
        for k in range(1, 4):
            f.step_raw(k, zs[k - 1].data_ptr(), int(zs[k - 1].shape[0]))
        ts, hw = [], []
        for k in range(4, 14):
            flush.zero_()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            t0 = time.perf_counter()
            f.step_raw(k, zs[k - 1].data_ptr(), int(zs[k - 1].shape[0]))
            hw.append(time.perf_counter() - t0)
            a1.record(stream)
            ts.append((a0, a1))
        torch.cuda.synchronize()
        r = res.setdefault(mode, {"event_ms": [], "host_ms": []})
        r["event_ms"].append(round(sum(a.elapsed_time(b) for a, b in ts) / 10, 4))
        r["host_ms"].append(round(sum(hw) * 1e3 / 10, 4))
print(json.dumps({"config": name, **res}))
