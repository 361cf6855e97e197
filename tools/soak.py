"""Soak run: many full steps of every config through the public API (t = 0 population on
the device), dense, gated and gated with a gate_floor, checking status and finite masses
each step.

    python tools/soak.py [--steps 100]
"""
import argparse
import math
import os
import sys
import time
from dataclasses import replace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    args = ap.parse_args()
    import paper_1503_03769_b200 as phd
    import scenario
    for cname in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        cfg = scenario.get(cname)
        steps = min(args.steps, args.steps if cname in ("cfg1", "cfg2", "cfg3") else max(10, args.steps // 4))
        cfg = replace(cfg, scenario=replace(cfg.scenario, steps=max(cfg.scenario.steps, steps)))
        truth = scenario.simulate_truth(cfg)
        Z = scenario.measurements(cfg, truth)
        ia = scenario.init_args(cfg, truth)
        V = (cfg.model.region[1] - cfg.model.region[0]) * (cfg.model.region[3] - cfg.model.region[2])
        F = max(-126, min(-20, int(math.floor(math.log2(cfg.model.clutter_rate / V))) - 60))
        for gate, floor in ((0, 0), (2, 0), (2, F)):
            f = phd.Filter(replace(cfg.model, gate=gate, gate_floor=floor))
            f.init_population(**ia)
            t0 = time.perf_counter()
            gated = 0
            lts = []
            for k in range(1, steps + 1):
                s = f.step(k, Z[k - 1]).as_dict()
                gated += f.gate_stats()["used"]
                assert math.isfinite(s["W"]) and s["W"] >= 0 and math.isfinite(s["W_pred"]), (cname, k, s)
                lts.append(s["LT"])
            dt = time.perf_counter() - t0
            f.close()
            print("%s gate=%d floor=%d steps=%d gated=%d wall %.2f s  LT last 5 %s"
                  % (cname, gate, floor, steps, gated, dt, lts[-5:]), flush=True)
    print("soak done")


if __name__ == "__main__":
    main()
