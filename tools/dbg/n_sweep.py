"""Dense update throughput against the particle count on one GPU (cfg 5's model and
measurement sets, N = 2^18 .. 2^27, M = 4096): step ms and update pairs/s, back-to-back
steps, CUDA events on the filter stream.  GATE=1: the gated update (pairs/s is then the
"effective" N*M per second).  usage: [GATE=1] python tools/dbg/n_sweep.py > out.json"""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1503_03769_b200 as phd, scenario
from dataclasses import replace

base = scenario.get("cfg5")
J = base.model.births_per_step
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
rows = []
for lg in range(18, 28):
    N = 1 << lg
    m = replace(base.model, fixed_count=N - J, capacity=N, gate=int(os.environ.get("GATE", "0")))
    cfg = replace(base, model=m, scenario=replace(base.scenario, steps=8))
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    Zd = [torch.from_numpy(z).cuda() for z in Z]
    f = phd.Filter(m, stream=stream.cuda_stream)
    f.init_population(**scenario.init_args(cfg, truth))
    for k in range(1, 4):
        f.step_raw(k, Zd[k - 1].data_ptr(), len(Z[k - 1]))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pairs = 0
    e0.record(stream)
    for k in range(4, 8):
        f.step_raw(k, Zd[k - 1].data_ptr(), len(Z[k - 1]))
        pairs += int(f._sum.N) * len(Z[k - 1])
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 4
    rows.append({"N": N, "M": len(Z[0]), "step_ms": ms, "pairs_per_s": pairs / 4 / (ms * 1e-3)})
    f.close()
    print(json.dumps(rows[-1]), file=sys.stderr)
what = "gated (gate = 1) step" if os.environ.get("GATE", "0") != "0" else "dense step"
print(json.dumps({"what": what + ", cfg 5 model, N = 2^18..2^27, back to back, 1 GPU", "rows": rows}, indent=1))
