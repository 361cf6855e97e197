"""Graph vs eager phd_step on a small config: mean step time over back-to-back steps
(CUDA events around the loop; no L2 flush), and per-step time with a flush + sync before
each step (the bench's protocol).  usage: python tools/dbg/graph_timing.py cfg3"""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1503_03769_b200 as phd, scenario
from dataclasses import replace

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = scenario.get(name)
cfg = replace(cfg, scenario=replace(cfg.scenario, steps=80))
truth = scenario.simulate_truth(cfg)
Z = scenario.measurements(cfg, truth)
Zd = [torch.from_numpy(z).cuda() for z in Z]
stream = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
for mode in ["eager", "graph"]:
    os.environ["PHD_GRAPH"] = "1" if mode == "graph" else "0"
    f = phd.Filter(cfg.model, stream=stream.cuda_stream)
    f.init_population(**scenario.init_args(cfg, truth))
    for k in range(1, 31):
        f.step_raw(k, Zd[k - 1].data_ptr(), len(Z[k - 1]))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(31, 51):
        f.step_raw(k, Zd[k - 1].data_ptr(), len(Z[k - 1]))
    e1.record(stream)
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / 20
    ts = []
    for k in range(51, 71):
        flush.zero_()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        f.step_raw(k, Zd[k - 1].data_ptr(), len(Z[k - 1]))
        a1.record(stream)
        ts.append((a0, a1))
    torch.cuda.synchronize()
    fl = sum(a.elapsed_time(b) for a, b in ts) / len(ts)
    res[mode] = {"back_to_back_ms": b2b, "flushed_ms": fl, "graph_stats": f.graph_stats()}
    f.close()
print(json.dumps({"config": name, "pdl": os.environ.get("PHD_PDL", "1"), **res}))
