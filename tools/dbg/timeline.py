"""GPU timeline of a few small-config steps (torch.profiler / CUPTI activity records of
every kernel, memcpy and memset in the process): per-op start offsets, durations and the
idle gaps between them.  usage: python tools/dbg/timeline.py cfg2 > gpurun_out/tl_cfg2.txt"""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1503_03769_b200 as phd, scenario
from dataclasses import replace
from torch.profiler import profile, ProfilerActivity

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = scenario.get(name)
cfg = replace(cfg, scenario=replace(cfg.scenario, steps=40))
if os.environ.get("NPART"):  # NPART=n: the config's model at n particles (capacity n + births)
    n_ = int(os.environ["NPART"])
    cfg = scenario.scaled(cfg, n_out=n_ - cfg.model.births_per_step, capacity=n_)
if os.environ.get("GATE"):  # GATE=1: the gated update
    cfg = replace(cfg, model=replace(cfg.model, gate=int(os.environ["GATE"])))
NPROF = int(os.environ.get("NPROF", "4"))
truth = scenario.simulate_truth(cfg)
Z = scenario.measurements(cfg, truth)
Zd = [torch.from_numpy(z).cuda() for z in Z]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
f = phd.Filter(cfg.model, stream=stream.cuda_stream)
f.init_population(**scenario.init_args(cfg, truth))
for k in range(1, 9 if cfg.model.fixed_count > 1000000 else 21):
    f.step_raw(k, Zd[k - 1].data_ptr(), len(Z[k - 1]))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    k0 = 9 if cfg.model.fixed_count > 1000000 else 21
    for k in range(k0, k0 + NPROF):
        f.step_raw(k, Zd[k - 1].data_ptr(), len(Z[k - 1]))
    torch.cuda.synchronize()
path = "/tmp/tl_%s.json" % name
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
prev_end = t0
for e in gpu:
    gap = e["ts"] - prev_end
    print("%9.2f  dur %7.2f  gap %7.2f  s%-3s %s" % (e["ts"] - t0, e["dur"], gap, e.get("args", {}).get("stream", "?"),
                                                  e["name"][:70]))
    prev_end = max(prev_end, e["ts"] + e["dur"])
cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"]
from collections import Counter
c = Counter(e["name"] for e in cpu)
print("runtime calls per %d steps:" % NPROF, dict(c))
busy = sum(e["dur"] for e in gpu)
span = gpu[-1]["ts"] + gpu[-1]["dur"] - gpu[0]["ts"]
print("gpu ops %d, busy %.1f us, span %.1f us (%.1f us per step)" % (len(gpu), busy, span, span / NPROF))
big = sorted(gpu, key=lambda e: -e["dur"])[:12]
for e in big:
    print("  %8.1f us  %s" % (e["dur"], e["name"][:80]))
f.close()
