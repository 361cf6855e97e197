"""Debug: distribution of the gated path's candidate count per tile (numpy
re-derivation from the predicted particles: cell sort, 512-particle tiles,
bounding boxes, e_max >= -130), next to the library's gate_stats."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import math
import numpy as np, scenario, paper_1503_03769_b200 as phd
from dataclasses import replace

cname = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = scenario.get(cname)
m = replace(cfg.model, gate=1)
truth = scenario.simulate_truth(cfg); Z = scenario.measurements(cfg, truth)
soa, w = scenario.initial_population(cfg, truth)
f = phd.Filter(m); f.set_particles(soa, w, soa.shape[1])
for k in range(1, steps + 1):
    z = Z[k - 1]
    f.predict(k)
    if k == steps:
        ps, pw, _ = f.get_particles()
    f.update(z)
    gs = f.gate_stats()
    f.extract(); f.resample_exchange(k)
x, y = ps[0].astype(np.float64), ps[2].astype(np.float64)
lo0, hi0, lo1, hi1 = m.region
G = 64
c0 = np.clip(np.floor((x - lo0) / ((hi0 - lo0) / G)), 0, G - 1).astype(np.int64)
c1 = np.clip(np.floor((y - lo1) / ((hi1 - lo1) / G)), 0, G - 1).astype(np.int64)
def spread(v):
    v = (v | (v << 8)) & 0x00FF00FF; v = (v | (v << 4)) & 0x0F0F0F0F
    v = (v | (v << 2)) & 0x33333333; return (v | (v << 1)) & 0x55555555
key = spread(c0) | (spread(c1) << 1)
order = np.argsort(key, kind="stable")
x, y, wv = x[order], y[order], pw[order].astype(np.float64)
n = len(x); T = 512; nt = (n + T - 1) // T
pad = nt * T - n
xs = np.concatenate([x, np.full(pad, np.nan)]).reshape(nt, T)
ys = np.concatenate([y, np.full(pad, np.nan)]).reshape(nt, T)
sig = m.sigma_z[0]
cst = m.p_d / (2 * math.pi * sig * sig)
lw = np.log2(np.maximum(cst * wv, 1e-300))
lws = np.concatenate([lw, np.full(pad, -np.inf)]).reshape(nt, T)
bx0, bx1 = np.nanmin(xs, 1), np.nanmax(xs, 1)
by0, by1 = np.nanmin(ys, 1), np.nanmax(ys, 1)
lwm = lws.max(1)
alpha = math.log2(math.e) / (2 * sig * sig)
zz = Z[steps - 1].astype(np.float64)
K = np.zeros(nt, np.int64)
for t0 in range(0, nt, 2048):
    sl = slice(t0, t0 + 2048)
    dx = np.maximum(0, np.maximum(bx0[sl, None] - zz[None, :, 0], zz[None, :, 0] - bx1[sl, None]))
    dy = np.maximum(0, np.maximum(by0[sl, None] - zz[None, :, 1], zz[None, :, 1] - by1[sl, None]))
    K[sl] = (-alpha * (dx * dx + dy * dy) + lwm[sl, None] >= -130).sum(1)
ext = np.maximum(bx1 - bx0, by1 - by0)
print("library gate_stats (used, E, pairs, tiles):", gs)
print("numpy: tiles %d  E %d  mean K %.1f" % (nt, K.sum(), K.mean()))
for q in (50, 75, 90, 95, 99, 99.9, 100):
    print("  K p%-5s %d   tile extent p%-5s %.1f m" % (q, np.percentile(K, q), q, np.percentile(ext, q)))
print("  tiles with K > 512: %d (%.2f%%), their entries %.1f%% of E" % ((K > 512).sum(), 100 * (K > 512).mean(),
      100 * K[K > 512].sum() / max(1, K.sum())))
print("  tiles with K > 256: %d, entries %.1f%% of E" % ((K > 256).sum(), 100 * K[K > 256].sum() / max(1, K.sum())))
# window sizes in cells (the enumeration rounds of k_gate_count / tile_enum) and the fast path
full = np.arange(nt) < n // T
kf = key[order]
kpad = np.concatenate([kf, np.full(pad, -1)]).reshape(nt, T)
cx0 = np.concatenate([c0[order], np.full(pad, -1)]).reshape(nt, T)
cy0 = np.concatenate([c1[order], np.full(pad, -1)]).reshape(nt, T)
fast = full & (kpad[:, 0] == kpad[:, -1]) & (cx0[:, 0] > 0) & (cx0[:, 0] < G - 1) & (cy0[:, 0] > 0) & (cy0[:, 0] < G - 1)
Rw = np.sqrt(np.maximum(lwm + 130, 0) / alpha)
h = (hi0 - lo0) / G
nx = np.floor((bx1 + Rw - lo0) / h).clip(0, G - 1) - np.floor((bx0 - Rw - lo0) / h).clip(0, G - 1) + 1
ny = np.floor((by1 + Rw - lo1) / h).clip(0, G - 1) - np.floor((by0 - Rw - lo1) / h).clip(0, G - 1) + 1
nc = (nx * ny).astype(np.int64)
print("fast-path tiles %.1f%%" % (100 * fast.mean()))
for q in (50, 90, 99, 99.9, 100):
    print("  window cells p%-5s %d  (rounds of 32: %d)" % (q, np.percentile(nc, q), -(-np.percentile(nc, q) // 32)))
print("  tiles with > 1024 window cells: %d" % (nc > 1024).sum())
