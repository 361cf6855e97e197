"""Is a small-config step host-bound?  Per-step GPU time back to back (the host issues
while the GPU runs) vs. the same step queued behind a long sleep kernel (every launch
already queued when the chain starts: pure GPU chain time).
usage: python tools/dbg/host_vs_gpu.py cfg2"""
import os, sys, json, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1503_03769_b200 as phd, scenario
from dataclasses import replace

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = scenario.get(name)
cfg = replace(cfg, scenario=replace(cfg.scenario, steps=80))
truth = scenario.simulate_truth(cfg)
Z = scenario.measurements(cfg, truth)
Zd = [torch.from_numpy(z).cuda() for z in Z]
stream = torch.cuda.Stream()  # non-default: the filter launches on it (0 = its own stream)
torch.cuda.set_stream(stream)
f = phd.Filter(cfg.model, stream=stream.cuda_stream)
f.init_population(**scenario.init_args(cfg, truth))
for k in range(1, 21):
    f.step_raw(k, Zd[k - 1].data_ptr(), len(Z[k - 1]))
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)
e0, e1 = E(), E()
t0 = time.perf_counter()
e0.record(stream)
for k in range(21, 41):
    f.step_raw(k, Zd[k - 1].data_ptr(), len(Z[k - 1]))
e1.record(stream)
torch.cuda.synchronize()
host = (time.perf_counter() - t0) * 1e3 / 20
b2b = e0.elapsed_time(e1) / 20
ts = []
for k in range(41, 61):
    a0, a1 = E(), E()
    torch.cuda._sleep(4_000_000)  # ~2 ms: the host queues the whole step meanwhile
    a0.record(stream)
    f.step_raw(k, Zd[k - 1].data_ptr(), len(Z[k - 1]))
    a1.record(stream)
    torch.cuda.synchronize()
    ts.append(a0.elapsed_time(a1))
ts.sort()
print(json.dumps({"config": name, "host_wall_ms": host, "b2b_gpu_ms": b2b, "queued_gpu_ms_median": ts[len(ts) // 2],
                  "queued_gpu_ms_min": ts[0]}))
f.close()
