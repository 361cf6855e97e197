"""Seeded synthetic inputs for the five workloads (SURVEY.md §8(d) recipe).

Produces, per config: the measurement sets Z_1..Z_K (fp32, shuffled per scan so
labels carry no truth) and the step-0 particle population (fp32 SoA).  Uses
numpy ``PCG64(SeedSequence(seed))`` only.  This module computes no filter
quantity (no likelihood, normaliser, weight or resampling arithmetic); it is
the one module the oracle side and the CUDA side share.

The truth model follows the paper's simulation section:
CV dynamics x' = F x + G w, range-bearing or position sensor, Poisson clutter
uniform over the measurement region.
"""
import math
import numpy as np

from .configs import POSITION, RANGE_BEARING, COUNT_FIXED


def _rng(seed, stream):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), int(stream)])))


class Truth:
    def __init__(self, states, alive):
        self.states = states  # [K+1, n_targets, 4] (x, vx, y, vy); NaN when not alive
        self.alive = alive    # [K+1, n_targets] bool


def simulate_truth(cfg):
    m, s = cfg.model, cfg.scenario
    rng = _rng(s.seed, 11)
    n, K = s.n_targets, s.steps
    x0 = rng.uniform(s.start_box[0], s.start_box[1], n)
    y0 = rng.uniform(s.start_box[2], s.start_box[3], n)
    sp = rng.uniform(s.speed[0], s.speed[1], n)
    hd = rng.uniform(0.0, 2.0 * math.pi, n)
    if s.birth_step_max > 0:
        born = rng.integers(0, s.birth_step_max + 1, n)
    else:
        born = np.zeros(n, dtype=np.int64)
    if s.lifetime[1] > 0:
        life = rng.integers(s.lifetime[0], s.lifetime[1] + 1, n)
    else:
        life = np.full(n, K + 1, dtype=np.int64)
    states = np.full((K + 1, n, 4), np.nan)
    alive = np.zeros((K + 1, n), dtype=bool)
    cur = np.stack([x0, sp * np.cos(hd), y0, sp * np.sin(hd)], axis=1)
    T, sa = m.T, m.sigma_a
    for k in range(K + 1):
        if k > 0:
            w = rng.standard_normal((n, 2)) * sa
            nxt = cur.copy()
            nxt[:, 0] = cur[:, 0] + T * cur[:, 1] + 0.5 * T * T * w[:, 0]
            nxt[:, 1] = cur[:, 1] + T * w[:, 0]
            nxt[:, 2] = cur[:, 2] + T * cur[:, 3] + 0.5 * T * T * w[:, 1]
            nxt[:, 3] = cur[:, 3] + T * w[:, 1]
            # targets not yet born keep their birth state
            nb = k <= born
            nxt[nb] = cur[nb]
            cur = nxt
        a = (born <= k) & (k < born + life)
        alive[k] = a
        states[k, a] = cur[a]
    return Truth(states, alive)


def _sensor(cfg, xy, rng):
    m = cfg.model
    if m.meas == POSITION:
        return xy + rng.standard_normal(xy.shape) * np.array(m.sigma_z)
    dx = xy[:, 0] - m.sensor_xy[0]
    dy = xy[:, 1] - m.sensor_xy[1]
    r = np.hypot(dx, dy) + rng.standard_normal(len(xy)) * m.sigma_z[0]
    th = np.arctan2(dy, dx) + rng.standard_normal(len(xy)) * m.sigma_z[1]
    th = (th + math.pi) % (2.0 * math.pi) - math.pi
    return np.stack([r, th], axis=1)


def measurements(cfg, truth=None):
    """Z_1..Z_K as a list of fp32 arrays [M_k, 2] (index 0 of the list is step 1)."""
    m, s = cfg.model, cfg.scenario
    truth = truth or simulate_truth(cfg)
    rng = _rng(s.seed, 12)
    reg = m.region
    out = []
    for k in range(1, s.steps + 1):
        a = truth.alive[k]
        xy = truth.states[k][a][:, [0, 2]]
        det = rng.uniform(size=len(xy)) < m.p_d
        zt = _sensor(cfg, xy[det], rng) if det.any() else np.zeros((0, 2))
        if s.clutter_fixed_total > 0:
            nc = max(0, s.clutter_fixed_total - len(zt))
        else:
            nc = rng.poisson(m.clutter_rate)
        zc = np.stack([rng.uniform(reg[0], reg[1], nc), rng.uniform(reg[2], reg[3], nc)], axis=1)
        z = np.concatenate([zt, zc], axis=0)
        rng.shuffle(z, axis=0)
        out.append(np.ascontiguousarray(z, dtype=np.float32))
    return out


def initial_count(cfg, truth=None):
    m, s = cfg.model, cfg.scenario
    truth = truth or simulate_truth(cfg)
    m0 = max(int(truth.alive[0].sum()), 1)
    if m.count_mode == COUNT_FIXED:
        return m.fixed_count, m0
    return min(m0 * m.particles_per_target, m.capacity - m.births_per_step), m0


def initial_population(cfg, truth=None, n=None):
    """Step-0 population: y-stratified, x uniform, v ~ U[-20,20]^2, mass m0.

    Returns (soa [4, N] float32 in (x, vx, y, vy) order, w [N] float32).
    """
    m, s = cfg.model, cfg.scenario
    truth = truth or simulate_truth(cfg)
    n0, m0 = initial_count(cfg, truth)
    if n is not None:
        n0 = n
    rng = _rng(s.seed, 13)
    box = s.init_box or (m.region if m.meas == POSITION else (-1000.0, 1000.0, -1000.0, 1000.0))
    i = np.arange(n0, dtype=np.float64)
    y = box[2] + (box[3] - box[2]) * (i + rng.uniform(size=n0)) / n0
    x = rng.uniform(box[0], box[1], n0)
    vx = rng.uniform(-20.0, 20.0, n0)
    vy = rng.uniform(-20.0, 20.0, n0)
    soa = np.stack([x, vx, y, vy]).astype(np.float32)
    if s.init_mass_box is not None:
        b = s.init_mass_box
        xs, ys = soa[0].astype(np.float64), soa[2].astype(np.float64)
        inside = (xs >= b[0]) & (xs <= b[1]) & (ys >= b[2]) & (ys <= b[3])
        w = np.zeros(n0, dtype=np.float32)
        w[inside] = np.float32(m0 / max(int(inside.sum()), 1))
    else:
        w = np.full(n0, np.float32(m0 / n0), dtype=np.float32)
    return np.ascontiguousarray(soa), w


def init_args(cfg, truth=None):
    """Arguments of phd_init_population for a config (the t = 0 population recipe of
    SURVEY.md §8(d); parameters only): total mass m0 = targets alive at step 0 (min 1),
    the Cartesian box, the mass box (cfg 5) and the velocity bound."""
    m, s = cfg.model, cfg.scenario
    truth = truth or simulate_truth(cfg)
    m0 = max(int(truth.alive[0].sum()), 1)
    box = s.init_box or (m.region if m.meas == POSITION else (-1000.0, 1000.0, -1000.0, 1000.0))
    return {"total_mass": float(m0), "box": tuple(float(v) for v in box),
            "mass_box": s.init_mass_box, "v_max": 20.0}


def random_particles(n, seed, box=(-1000.0, 1000.0, -1000.0, 1000.0), vmax=20.0,
                     w_range=(1e-4, 1e-2), stream=21):
    """Generic seeded particle cloud for parity tests (fp32 SoA + fp32 weights)."""
    rng = _rng(seed, stream)
    soa = np.stack([rng.uniform(box[0], box[1], n), rng.uniform(-vmax, vmax, n),
                    rng.uniform(box[2], box[3], n), rng.uniform(-vmax, vmax, n)]).astype(np.float32)
    w = rng.uniform(w_range[0], w_range[1], n).astype(np.float32)
    return np.ascontiguousarray(soa), w


def clustered_particles(n, zs, seed, spread=15.0, vmax=20.0, frac_near=0.7, meas=POSITION,
                        sensor=(0.0, 0.0), box=(-1000.0, 1000.0, -1000.0, 1000.0), stream=22):
    """Particles where a fraction sits near given measurements (so that the
    likelihood sums are dominated by non-negligible terms), the rest uniform."""
    rng = _rng(seed, stream)
    soa, w = random_particles(n, seed, box=box, vmax=vmax, stream=stream + 1)
    zs = np.asarray(zs, dtype=np.float64)
    if len(zs) == 0:
        return soa, w
    k = int(n * frac_near)
    pick = rng.integers(0, len(zs), k)
    if meas == POSITION:
        cx, cy = zs[pick, 0], zs[pick, 1]
    else:
        cx = sensor[0] + zs[pick, 0] * np.cos(zs[pick, 1])
        cy = sensor[1] + zs[pick, 0] * np.sin(zs[pick, 1])
    soa[0, :k] = (cx + rng.standard_normal(k) * spread).astype(np.float32)
    soa[2, :k] = (cy + rng.standard_normal(k) * spread).astype(np.float32)
    perm = rng.permutation(n)
    return np.ascontiguousarray(soa[:, perm]), np.ascontiguousarray(w[perm])


def random_measurements(M, seed, meas=POSITION, region=(-1000.0, 1000.0, -1000.0, 1000.0), stream=31):
    rng = _rng(seed, stream)
    z = np.stack([rng.uniform(region[0], region[1], M), rng.uniform(region[2], region[3], M)], axis=1)
    return np.ascontiguousarray(z, dtype=np.float32)
