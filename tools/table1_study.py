"""Table-1-shaped study (NEXT-3) on one B200.

The paper compares, on a bearing/range tracking scenario with 5 tracks over 50
scans and clutter rate r in {0, 10, 20}:
  PHD     the serial particle PHD filter with all N particles,
  DCPPHD  the distributed filter with K = 4 groups of N/4 particles,
  partPHD the serial filter with N/4 particles,
reporting run time and the mean OSPA (p = 1, c = 100).

The paper's scenario is not recoverable (its figures are lost), so this study
uses a synthetic scenario of the same shape: range-bearing sensor
at the origin, region r in [0, 200] m x bearing in [-pi/2, pi/2],
noise stds 5 m / 0.05 rad (PAPER.md:414 read as stds), 5 targets with random
birth and death over 50 scans, R = 200 particles per target per group, K = 4
(PAPER.md:445-447).  DCPPHD runs its 4 groups as 4 rank contexts of an
in-process rank group on the single GPU, so its time is the 4 groups
time-sharing one B200, not a 4-GPU time.  Times are the GPU filter time of one
full run (50 steps, host-synchronous API), median over Monte-Carlo runs.

    python tools/table1_study.py [--runs 10] [--out profiles/r01_table1_study]
"""
import argparse
import json
import math
import os
import sys
import threading
import time
from dataclasses import replace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import scenario  # noqa: E402
from scenario.configs import Config, Model, Scenario, RANGE_BEARING, COUNT_ADAPTIVE, MODE_DCP, MODE_EXACT  # noqa: E402


def paper_config(r, seed, R, J, mode=MODE_EXACT):
    m = Model(meas=RANGE_BEARING, sigma_z=(5.0, 0.05), sensor_xy=(0.0, 0.0),
              region=(0.0, 200.0, -math.pi / 2, math.pi / 2), sigma_a=0.2, p_s=0.99, p_d=0.98,
              clutter_rate=float(r), birth_mass=0.1, birth_sigma_v=1.0, births_per_step=J,
              particles_per_target=R, count_mode=COUNT_ADAPTIVE, capacity=1 << 16, max_meas=256, seed=seed,
              mode=mode)
    s = Scenario(n_targets=5, start_box=(30.0, 150.0, -80.0, 80.0), speed=(0.5, 2.0), steps=50,
                 birth_step_max=20, lifetime=(25, 50), init_box=(0.0, 200.0, -150.0, 150.0), seed=seed)
    return Config("paper_bot_r%d" % r, m, s)


def run_filter(phd, cfg, K, Z, truth):
    from paper_1503_03769_b200.metrics import ospa, positions
    m = cfg.model
    if K > 1:
        # every DCP group is a separate filter of the full intensity:
        # K blocks of m0 R particles, each carrying the full initial mass m0
        big = replace(cfg, model=replace(m, particles_per_target=m.particles_per_target * K))
        soa, w = scenario.initial_population(big, truth)
        w = w * np.float32(K)
    else:
        soa, w = scenario.initial_population(cfg, truth)
    n0 = soa.shape[1]
    grp = phd.LocalGroup(K) if K > 1 else None
    fs = [phd.Filter(m, rank=j, group=grp) for j in range(K)]
    for j, f in enumerate(fs):
        a, b = (n0 * j) // K, (n0 * (j + 1)) // K
        f.set_particles(np.ascontiguousarray(soa[:, a:b]), np.ascontiguousarray(w[a:b]), b - a if K > 1 else n0)
    ospas, card = [], []
    t0 = time.perf_counter()
    gpu_time = 0.0
    for k in range(1, len(Z) + 1):
        z = Z[k - 1]
        t1 = time.perf_counter()
        if K == 1:
            fs[0].step(k, z)
        else:
            th = [threading.Thread(target=lambda f=f: f.step(k, z)) for f in fs]
            [t.start() for t in th]
            [t.join() for t in th]
        gpu_time += time.perf_counter() - t1
        est = fs[0]._estimates()
        tru = truth.states[k][truth.alive[k]][:, [0, 2]]
        ospas.append(ospa(positions(est["states"]), tru, c=100.0, p=1.0))
        card.append((len(est["labels"]), int(truth.alive[k].sum())))
    for f in fs:
        f.close()
    if grp is not None:
        grp.close()
    return {"ospa": float(np.mean(ospas)), "time_s": gpu_time, "card": card}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_table1_study"))
    args = ap.parse_args()
    import paper_1503_03769_b200 as phd
    phd.load()
    K, R = 4, 200
    methods = [("PHD", MODE_EXACT, 1, K * R, K * 100), ("DCPPHD", MODE_DCP, K, R, K * 100),
               ("partPHD", MODE_EXACT, 1, R, 100)]
    rows = []
    for r in (0, 10, 20):
        for name, mode, k_groups, Rm, J in methods:
            res = []
            for run in range(args.runs):
                cfg = paper_config(r, 1000 + run, Rm, J, mode)
                truth = scenario.simulate_truth(cfg)
                Z = scenario.measurements(cfg, truth)
                res.append(run_filter(phd, cfg, k_groups, Z, truth))
            o = np.array([x["ospa"] for x in res])
            t = np.array([x["time_s"] for x in res])
            card_err = np.mean([abs(a - b) for x in res for a, b in x["card"]])
            rows.append({"method": name, "r": r, "groups": k_groups, "particles_per_target_per_group": Rm,
                         "runs": args.runs, "time_s_median": float(np.median(t)), "mean_ospa": float(o.mean()),
                         "std_ospa": float(o.std()), "mean_abs_card_err": float(card_err)})
            print(json.dumps(rows[-1]), flush=True)
    with open(args.out + ".json", "w") as f:
        json.dump(rows, f, indent=1)
    with open(args.out + ".md", "w") as f:
        f.write("Table-1-shaped study on one B200 (tools/table1_study.py): synthetic BOT-like scenario, "
                "5 tracks, 50 scans, R = 200 per target per group, K = 4; DCPPHD's 4 groups time-share the GPU.\n\n")
        f.write("| method | r | time per run (s, median) | mean OSPA (p=1, c=100) | std of OSPA | mean abs cardinality error |\n")
        f.write("|---|---|---|---|---|---|\n")
        for x in rows:
            f.write("| %s | %d | %.4f | %.3f | %.3f | %.3f |\n" % (x["method"], x["r"], x["time_s_median"],
                                                                  x["mean_ospa"], x["std_ospa"],
                                                                  x["mean_abs_card_err"]))
    print(open(args.out + ".md").read())


if __name__ == "__main__":
    main()
