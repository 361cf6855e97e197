"""How much of the N x M pair space could exact gating skip?

Runs the filter on a config for a few steps on the GPU, takes the PREDICTED
population of step k (the update's input), and counts the (particle tile,
measurement group) blocks whose largest possible exponent
    E_max = -alpha * dist^2(tile bbox, group bbox) + max_i log2(p_D c w_i)
is below -127, i.e. whose every term 2^E flushes to exactly +0 in the update
kernels.  Tiles are kTileP = 64 consecutive particles in storage order, groups
are runs of G slots of the measurements sorted along a Morton curve.

  python tools/gating_study.py [--config cfg5] [--steps 6]
Position model only.
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def morton_order(x, y, box):
    def q(v, lo, hi):
        return np.clip(((v - lo) / (hi - lo) * 65535.0).astype(np.int64), 0, 65535)
    qx, qy = q(x, box[0], box[1]), q(y, box[2], box[3])

    def spread(v):
        v = (v | (v << 8)) & 0x00FF00FF
        v = (v | (v << 4)) & 0x0F0F0F0F
        v = (v | (v << 2)) & 0x33333333
        v = (v | (v << 1)) & 0x55555555
        return v
    return np.argsort(spread(qx) | (spread(qy) << 1), kind="stable")


def study(soa, w, z, model, tile=64, groups=(256, 2048)):
    sx, sy = model.sigma_z
    assert abs(sx - sy) < 1e-12
    alpha = math.log2(math.e) / (2 * sx * sx)
    c = 1.0 / (2 * math.pi * sx * sy)
    n = soa.shape[1]
    nt = (n + tile - 1) // tile
    pad = nt * tile - n
    x = np.concatenate([soa[0], np.full(pad, np.nan, np.float32)]).reshape(nt, tile).astype(np.float64)
    y = np.concatenate([soa[2], np.full(pad, np.nan, np.float32)]).reshape(nt, tile).astype(np.float64)
    ww = np.concatenate([w, np.zeros(pad, np.float32)]).reshape(nt, tile).astype(np.float64)
    with np.errstate(divide="ignore"):
        lw = np.log2(model.p_d * c * ww)
    tx0, tx1 = np.nanmin(x, 1), np.nanmax(x, 1)
    ty0, ty1 = np.nanmin(y, 1), np.nanmax(y, 1)
    lwm = lw.max(1)
    live = lwm > -np.inf
    order = morton_order(z[:, 0], z[:, 1], model.region)
    zs = z[order].astype(np.float64)
    out = {"tiles": int(nt), "tiles_with_mass": int(live.sum()), "M": int(z.shape[0])}
    for G in groups:
        ng = (len(zs) + G - 1) // G
        kept = 0
        for g in range(ng):
            zz = zs[g * G:(g + 1) * G]
            gx0, gx1, gy0, gy1 = zz[:, 0].min(), zz[:, 0].max(), zz[:, 1].min(), zz[:, 1].max()
            dx = np.maximum(0.0, np.maximum(gx0 - tx1, tx0 - gx1))
            dy = np.maximum(0.0, np.maximum(gy0 - ty1, ty0 - gy1))
            emax = -alpha * (dx * dx + dy * dy) + lwm
            kept += int(np.count_nonzero(emax >= -128.0))
        out["G%d_kept_fraction" % G] = kept / float(nt * ng)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--steps", type=int, default=6)
    args = ap.parse_args()
    import torch  # noqa: F401  (device memory / CUDA context)
    import paper_1503_03769_b200 as phd
    import scenario
    sys.path.insert(0, ROOT)
    from bench import scenario_for
    cfg = scenario_for(args.config, args.steps + 2)
    m = cfg.model
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    soa, w = scenario.initial_population(cfg, truth)
    phd.load(build_if_missing=True)
    f = phd.Filter(m)
    f.set_particles(soa, w, soa.shape[1])
    for k in range(1, args.steps + 1):
        f.predict(k, Z[k - 2] if k >= 2 else None)
        ps, pw, _ = f.get_particles()
        r = study(ps, pw, Z[k - 1], m)
        r["step"] = k
        print(json.dumps(r), flush=True)
        f.update(Z[k - 1])
        f.extract()
        f.resample_exchange(k)


if __name__ == "__main__":
    main()
