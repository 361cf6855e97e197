"""The five BASELINE.json workloads as plain parameter records.

This module holds numbers only (no filter arithmetic); it is shared by the
oracle-side tests and the CUDA-side binding, as DESIGN.md §"Input recipe"
describes.  Every value is either stated by BASELINE.json ``configs[i]`` or is
the SURVEY.md §8(d) reading for a value the config leaves silent.
"""
from dataclasses import dataclass, field, asdict, replace
import math

POSITION = 0
RANGE_BEARING = 1
MODE_EXACT = 0
MODE_DCP = 1
COUNT_ADAPTIVE = 0
COUNT_FIXED = 1


@dataclass(frozen=True)
class Model:
    """Filter model parameters (the fields of ``phd_params`` in include/phd.h)."""
    meas: int = POSITION
    T: float = 1.0                 # CV sampling period
    sigma_a: float = 5.0           # accel-noise std, both axes (BASELINE configs)
    p_s: float = 0.99              # survival e_{k|k-1} (configs override PAPER.md:419)
    p_d: float = 0.98              # detection
    sigma_z: tuple = (10.0, 10.0)  # (sigma, sigma) or (sigma_r, sigma_theta)
    sensor_xy: tuple = (0.0, 0.0)
    region: tuple = (-1000.0, 1000.0, -1000.0, 1000.0)  # xmin,xmax,ymin,ymax | rmin,rmax,thmin,thmax
    clutter_rate: float = 10.0     # lambda (mean clutter count per scan)
    birth_mass: float = 0.1        # gamma (total birth mass per step)
    birth_sigma_v: float = 10.0    # birth velocity std
    births_per_step: int = 200     # J
    particles_per_target: int = 500  # R (adaptive mode)
    fixed_count: int = 0           # N_out (fixed mode)
    count_mode: int = COUNT_ADAPTIVE
    capacity: int = 1 << 16        # max N (global) = max N_out + J
    max_meas: int = 1024
    seed: int = 1
    mode: int = 0                  # 0 exact (global C, exact resampling), 1 DCP (paper-literal groups)
    exchange_count: int = 0        # DCP ring exchange L (0: min_j N_j / 10)
    birth_model: int = 0           # 0: measurement-driven (S10); 1: N(birth_mean, diag(birth_std^2));
                                   # 2: drawn as 0, weighted gamma N(x; birth_mean, Q) / (J p_k(x|Z)) (Eq 6)
    birth_mean: tuple = (0.0, 3.0, 0.0, -3.0)           # x-bar
    birth_std: tuple = (math.sqrt(10.0), 1.0, math.sqrt(10.0), 1.0)  # sqrt(diag Q)
    stphd_all: int = 0             # 1: STPHD state sums for every measurement (not only the index set)
    proposal_scale: float = 1.0    # Eq 5 proposal: CV transition with noise std s sigma_a (1: prior)
    gate: int = 0                  # update: 0 dense, 1 gated (auto fallback), 2 gated when it fits
    gate_floor: int = 0            # gated: 0 exact (skip only exact zeros), else skip terms < 2^gate_floor


@dataclass(frozen=True)
class Scenario:
    """Truth-generation recipe."""
    n_targets: int = 3
    start_box: tuple = (-1000.0, 1000.0, -1000.0, 1000.0)
    speed: tuple = (5.0, 20.0)
    steps: int = 20
    birth_step_max: int = 0        # targets born at U{0..birth_step_max}
    lifetime: tuple = (0, 0)       # (0,0) = alive for the whole run
    clutter_fixed_total: int = 0   # >0: clutter count = total - detections (cfg 5)
    init_box: tuple = None         # Cartesian box of the initial population (None: region box)
    init_mass_box: tuple = None    # only particles inside carry initial mass (cfg 5)
    seed: int = 1


@dataclass(frozen=True)
class Config:
    name: str
    model: Model
    scenario: Scenario
    note: str = ""

    def as_dict(self):
        return {"name": self.name, "model": asdict(self.model), "scenario": asdict(self.scenario)}


def _cfg1():
    m = Model(meas=POSITION, sigma_z=(10.0, 10.0), region=(-1000.0, 1000.0, -1000.0, 1000.0),
              p_d=0.98, p_s=0.99, clutter_rate=10.0, births_per_step=200,
              particles_per_target=500, count_mode=COUNT_ADAPTIVE, capacity=1 << 15, max_meas=256)
    s = Scenario(n_targets=3, steps=20)
    return Config("cfg1_tiny", m, s, "BASELINE.json configs[0]")


def _cfg2():
    m = Model(meas=RANGE_BEARING, sigma_z=(10.0, 0.01), sensor_xy=(0.0, 0.0),
              region=(0.0, 2000.0, -math.pi, math.pi), p_d=0.98, p_s=0.99, clutter_rate=50.0,
              births_per_step=1000, particles_per_target=1000, count_mode=COUNT_ADAPTIVE,
              capacity=1 << 15, max_meas=512)
    s = Scenario(n_targets=10, steps=100, birth_step_max=60, lifetime=(20, 60),
                 init_box=(-1000.0, 1000.0, -1000.0, 1000.0))
    return Config("cfg2_paper_scale", m, s, "BASELINE.json configs[1]")


def _cfg3():
    m = Model(meas=POSITION, sigma_z=(10.0, 10.0), region=(-1000.0, 1000.0, -1000.0, 1000.0),
              p_d=0.95, p_s=0.99, clutter_rate=500.0, births_per_step=14688,
              fixed_count=100000, count_mode=COUNT_FIXED, capacity=114688, max_meas=1024)
    s = Scenario(n_targets=100, steps=50)
    return Config("cfg3_dense", m, s, "BASELINE.json configs[2]")


def _cfg4():
    m = Model(meas=RANGE_BEARING, sigma_z=(10.0, 0.01), sensor_xy=(0.0, 0.0),
              region=(0.0, 2000.0, -math.pi, math.pi), p_d=0.98, p_s=0.99, clutter_rate=2000.0,
              births_per_step=72576, fixed_count=2000000, count_mode=COUNT_FIXED,
              capacity=2072576, max_meas=4096)
    s = Scenario(n_targets=1000, steps=20, init_box=(-1000.0, 1000.0, -1000.0, 1000.0))
    return Config("cfg4_large", m, s, "BASELINE.json configs[3]")


def _cfg5():
    # M = 4096 exactly: 1024 targets detected w.p. 0.98, clutter fills the rest.
    lam = 4096 - 0.98 * 1024
    m = Model(meas=POSITION, sigma_z=(10.0, 10.0), region=(-1000.0, 1000.0, -1000.0, 1000.0),
              p_d=0.98, p_s=0.99, clutter_rate=lam, births_per_step=65536,
              fixed_count=16711680, count_mode=COUNT_FIXED, capacity=1 << 24, max_meas=4096)
    s = Scenario(n_targets=1024, steps=10, start_box=(0.0, 1000.0, 0.0, 1000.0),
                 clutter_fixed_total=4096, init_mass_box=(0.0, 1000.0, 0.0, 1000.0))
    return Config("cfg5_exchange_stress", m, s, "BASELINE.json configs[4]")


CONFIGS = {c.name: c for c in (_cfg1(), _cfg2(), _cfg3(), _cfg4(), _cfg5())}
ORDER = ["cfg1_tiny", "cfg2_paper_scale", "cfg3_dense", "cfg4_large", "cfg5_exchange_stress"]


def get(name):
    if name in CONFIGS:
        return CONFIGS[name]
    for k in ORDER:
        if k.startswith(name):
            return CONFIGS[k]
    raise KeyError(name)


def scaled(cfg, n_out=None, births=None, capacity=None, max_meas=None, steps=None, name=None):
    """A smaller copy of a config (parity-test sizes); only counts change."""
    m = cfg.model
    kw = {}
    if n_out is not None:
        kw["fixed_count"] = n_out
        kw["count_mode"] = COUNT_FIXED
    if births is not None:
        kw["births_per_step"] = births
    if capacity is not None:
        kw["capacity"] = capacity
    if max_meas is not None:
        kw["max_meas"] = max_meas
    m2 = replace(m, **kw)
    s2 = cfg.scenario if steps is None else replace(cfg.scenario, steps=steps)
    return Config(name or (cfg.name + "_scaled"), m2, s2, cfg.note + " (scaled)")
