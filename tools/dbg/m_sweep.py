"""Dense update throughput against the measurement count (cfg 5's model, N = 2^22, random
measurement sets of M = 64 .. 8192 over the region, clustered particles): step ms, update
pairs/s and the passes' layout (ZL, warps, z-blocks, tile).  usage: python tools/dbg/m_sweep.py"""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1503_03769_b200 as phd, scenario
from dataclasses import replace

base = scenario.get("cfg5")
N = 1 << 22
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
rows = []
for M in (64, 256, 512, 1024, 2048, 3000, 4096, 6000, 8192):
    m = replace(base.model, fixed_count=N - base.model.births_per_step, capacity=N, max_meas=8192)
    z = scenario.random_measurements(M, 7, meas=m.meas, region=m.region)
    soa, w = scenario.clustered_particles(N, z[:max(1, M // 4)], 7, meas=m.meas, sensor=m.sensor_xy,
                                          box=tuple(m.region))
    zd = torch.from_numpy(z).cuda()
    f = phd.Filter(m, stream=stream.cuda_stream)
    ts = []
    for rep in range(5):
        f.set_particles(soa, w, N, stage=phd.STAGE_PREDICTED)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f.update_raw(zd.data_ptr(), M) if hasattr(f, "update_raw") else f.update(z)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    _, summ = f.extract()
    rows.append({"N": N, "M": M, "update_ms": ms, "pairs_per_s": N * M / (ms * 1e-3), "LT": int(summ["LT"])})
    print(json.dumps(rows[-1]), file=sys.stderr)
    f.close()
print(json.dumps({"what": "dense update only (set_particles + update), cfg 5 model, N = 2^22, 1 GPU", "rows": rows},
                 indent=1))
