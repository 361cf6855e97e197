"""TEST INFRASTRUCTURE, NOT PRODUCT CODE: ctypes wrapper of the fp64 oracle.

The oracle (oracle/phd_oracle.c) is a plain single-threaded fp64 reference of
one particle-PHD step written from PAPER.md.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference arm may
import this package; the CUDA product path (paper_1503_03769_b200) never does
and shares no code with it.
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libphd_oracle.so")
SRC = os.path.join(HERE, "phd_oracle.c")
SRC_MT = os.path.join(HERE, "phd_oracle_mt.c")


def build(force=False):
    """Compile the oracle shared library with gcc (plain -O2, no fast-math, no FMA contraction)."""
    srcs = [SRC, SRC_MT, os.path.join(HERE, "phd_oracle.h")]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(f) for f in srcs):
        return LIB
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-pthread",
           "-o", LIB, SRC, SRC_MT, "-lm"]
    subprocess.check_call(cmd, cwd=HERE)
    return LIB


class _Model(ctypes.Structure):
    _fields_ = [("meas", ctypes.c_int32), ("pad_", ctypes.c_int32), ("T", ctypes.c_double),
                ("sigma_a", ctypes.c_double), ("p_s", ctypes.c_double), ("p_d", ctypes.c_double),
                ("sigma_z", ctypes.c_double * 2), ("sensor", ctypes.c_double * 2),
                ("region", ctypes.c_double * 4), ("clutter_rate", ctypes.c_double),
                ("birth_mass", ctypes.c_double), ("birth_sigma_v", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("birth_model", ctypes.c_int32), ("pad2_", ctypes.c_int32),
                ("birth_mean", ctypes.c_double * 4), ("birth_std", ctypes.c_double * 4),
                ("proposal_scale", ctypes.c_double)]


_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_I32 = ctypes.POINTER(ctypes.c_int32)
_U32 = ctypes.POINTER(ctypes.c_uint32)


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        M = ctypes.POINTER(_Model)
        L.orc_philox4x32_10.argtypes = [_U32, _U32, _U32]
        L.orc_conv23.argtypes = [ctypes.c_uint32]
        L.orc_conv23.restype = ctypes.c_double
        L.orc_u52.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.orc_u52.restype = ctypes.c_double
        L.orc_box_muller.argtypes = [ctypes.c_double, ctypes.c_double, _D, _D]
        L.orc_kappa.argtypes = [M]
        L.orc_kappa.restype = ctypes.c_double
        L.orc_likelihood.argtypes = [M, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        L.orc_likelihood.restype = ctypes.c_double
        L.orc_predict.argtypes = [M, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, _D, _D, _D, _D, _D]
        L.orc_births.argtypes = [M, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_int64, _D, ctypes.c_int32, _D, _D, _D, _D, _D]
        L.orc_birth_is_weights.argtypes = [M, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _D,
                                           ctypes.c_int32, _D, _D, _D, _D, _D]
        L.orc_normalizers.argtypes = [M, ctypes.c_int64, _D, _D, _D, _D, ctypes.c_int32, _D]
        L.orc_update.argtypes = [M, ctypes.c_int64, _D, _D, _D, _D, _D, _D, ctypes.c_int32, _D, _D, _D]
        L.orc_normalizers_mt.argtypes = [M, ctypes.c_int64, _D, _D, _D, _D, ctypes.c_int32, _D, ctypes.c_int32]
        L.orc_update_mt.argtypes = [M, ctypes.c_int64, _D, _D, _D, _D, _D, _D, ctypes.c_int32, _D, _D, _D,
                                    ctypes.c_int32]
        L.orc_extract.argtypes = [M, ctypes.c_int32, _D, ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                  _I32, _D, _D, _I64, _I32, _D]
        L.orc_extract.restype = ctypes.c_int32
        L.orc_init_population.argtypes = [M, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _D, ctypes.c_double,
                                          ctypes.c_double, _D, _D, _D, _D, _D, _D]
        L.orc_init_population.restype = ctypes.c_int64
        L.orc_resample_U.argtypes = [ctypes.c_uint64, ctypes.c_int32]
        L.orc_resample_U.restype = ctypes.c_double
        L.orc_resample.argtypes = [ctypes.c_int64, _D, ctypes.c_double, ctypes.c_int64, _I64]
        L.orc_resample.restype = ctypes.c_double
        _lib = L
    return _lib


def model(m):
    """orc_model from a scenario.configs.Model (or any object with the same fields)."""
    om = _Model()
    om.meas = int(m.meas)
    om.T, om.sigma_a, om.p_s, om.p_d = float(m.T), float(m.sigma_a), float(m.p_s), float(m.p_d)
    om.sigma_z[0], om.sigma_z[1] = float(m.sigma_z[0]), float(m.sigma_z[1])
    om.sensor[0], om.sensor[1] = float(m.sensor_xy[0]), float(m.sensor_xy[1])
    for i in range(4):
        om.region[i] = float(m.region[i])
    om.clutter_rate = float(m.clutter_rate)
    om.birth_mass = float(m.birth_mass)
    om.birth_sigma_v = float(m.birth_sigma_v)
    om.seed = int(m.seed)
    om.birth_model = int(getattr(m, "birth_model", 0))
    for i in range(4):
        om.birth_mean[i] = float(getattr(m, "birth_mean", (0.0, 0.0, 0.0, 0.0))[i])
        om.birth_std[i] = float(getattr(m, "birth_std", (0.0, 0.0, 0.0, 0.0))[i])
    om.proposal_scale = float(getattr(m, "proposal_scale", 1.0))
    return om


def _d(a):
    return a.ctypes.data_as(_D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return [int(o[i]) for i in range(4)]


def conv23(w):
    return lib().orc_conv23(int(w))


def u52(w0, w1):
    return lib().orc_u52(int(w0), int(w1))


def box_muller(u1, u2):
    a, b = ctypes.c_double(), ctypes.c_double()
    lib().orc_box_muller(float(u1), float(u2), ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def init_population(m, n_out, box, v_max, total_mass, mass_box=None, g_lo=0, g_hi=None):
    """t = 0 population (S23): particles g_lo .. g_hi-1 of n_out.
    Returns (soa [4, n] fp64 in (x, vx, y, vy) order, holding fp32 values; w [n]; inside count)."""
    g_hi = n_out if g_hi is None else g_hi
    n = g_hi - g_lo
    x, vx, y, vy, w = (np.zeros(max(n, 1)) for _ in range(5))
    b = _f64(box)
    mb = _f64(mass_box) if mass_box is not None else None
    inside = lib().orc_init_population(ctypes.byref(model(m)), int(n_out), int(g_lo), int(g_hi), _d(b), float(v_max),
                                       float(total_mass), _d(mb) if mb is not None else None, _d(x), _d(vx), _d(y),
                                       _d(vy), _d(w))
    return np.stack([x[:n], vx[:n], y[:n], vy[:n]]), w[:n], int(inside)


def kappa(m):
    return lib().orc_kappa(ctypes.byref(model(m)))


def likelihood(m, z, xy):
    return lib().orc_likelihood(ctypes.byref(model(m)), float(z[0]), float(z[1]), float(xy[0]), float(xy[1]))


def predict(m, k, soa, w, g0=0):
    """Eq 5 survivors; soa [4, n] (x, vx, y, vy), w [n]; returns fp64 copies."""
    s = _f64(soa).copy()
    ww = _f64(w).copy()
    n = s.shape[1]
    x, vx, y, vy = [np.ascontiguousarray(s[i]) for i in range(4)]
    lib().orc_predict(ctypes.byref(model(m)), int(k), n, int(g0), _d(x), _d(vx), _d(y), _d(vy), _d(ww))
    return np.stack([x, vx, y, vy]), ww


def births(m, k, n_out, J, zprev, b0=0, nb=None, blo=0):
    """Eq 6: births b0 .. b0+nb-1 of this filter's J (global slots n_out + b).
    birth_model 2 weights them by the full ratio over the filter's births [blo, blo+J)."""
    nb = J - b0 if nb is None else nb
    zp = _f64(np.zeros((0, 2)) if zprev is None else zprev).reshape(-1, 2)
    out = [np.zeros(nb) for _ in range(5)]
    om = model(m)
    lib().orc_births(ctypes.byref(om), int(k), int(n_out), int(J), int(b0), int(nb),
                     _d(zp), int(len(zp)), *[_d(a) for a in out])
    if om.birth_model == 2:
        lib().orc_birth_is_weights(ctypes.byref(om), int(J), int(blo), int(nb), _d(zp), int(len(zp)),
                                   *[_d(a) for a in out])
    return np.stack(out[:4]), out[4]


def normalizers(m, soa, w, z):
    s = _f64(soa)
    x, y = np.ascontiguousarray(s[0]), np.ascontiguousarray(s[2])
    ww = _f64(w)
    zz = _f64(z).reshape(-1, 2)
    C = np.zeros(len(zz))
    lib().orc_normalizers(ctypes.byref(model(m)), len(ww), _d(x), _d(y), _d(ww), _d(zz), len(zz), _d(C))
    return C


def update(m, soa, w, z, C):
    s = _f64(soa)
    x, vx, y, vy = [np.ascontiguousarray(s[i]) for i in range(4)]
    ww = _f64(w)
    zz = _f64(z).reshape(-1, 2)
    CC = _f64(C)
    wo = np.zeros(len(ww))
    acc = np.zeros((len(zz), 5))
    lib().orc_update(ctypes.byref(model(m)), len(ww), _d(x), _d(vx), _d(y), _d(vy), _d(ww),
                     _d(zz), len(zz), _d(CC), _d(wo), _d(acc))
    return wo, acc


def normalizers_mt(m, soa, w, z, nthreads):
    """normalizers() split over particles across threads (all-core CPU baseline; timing)."""
    s = _f64(soa)
    x, y = np.ascontiguousarray(s[0]), np.ascontiguousarray(s[2])
    ww = _f64(w)
    zz = _f64(z).reshape(-1, 2)
    C = np.zeros(len(zz))
    lib().orc_normalizers_mt(ctypes.byref(model(m)), len(ww), _d(x), _d(y), _d(ww), _d(zz), len(zz), _d(C),
                             int(nthreads))
    return C


def update_mt(m, soa, w, z, C, nthreads):
    """update() split over particles across threads (all-core CPU baseline; timing)."""
    s = _f64(soa)
    x, vx, y, vy = [np.ascontiguousarray(s[i]) for i in range(4)]
    ww = _f64(w)
    zz = _f64(z).reshape(-1, 2)
    CC = _f64(C)
    wo = np.zeros(len(ww))
    acc = np.zeros((len(zz), 5))
    lib().orc_update_mt(ctypes.byref(model(m)), len(ww), _d(x), _d(vx), _d(y), _d(vy), _d(ww),
                        _d(zz), len(zz), _d(CC), _d(wo), _d(acc), int(nthreads))
    return wo, acc


def extract(m, acc, W, W_pred, cap=None):
    acc = _f64(acc).reshape(-1, 5)
    nz = len(acc)
    cap = max(nz, 1) if cap is None else cap
    labels = np.zeros(cap, dtype=np.int32)
    states = np.zeros((cap, 4))
    mass = np.zeros(cap)
    LT = ctypes.c_int64()
    clamped = ctypes.c_int32()
    und = ctypes.c_double()
    n = lib().orc_extract(ctypes.byref(model(m)), nz, _d(acc), float(W), float(W_pred), cap,
                          labels.ctypes.data_as(_I32), _d(states), _d(mass), ctypes.byref(LT),
                          ctypes.byref(clamped), ctypes.byref(und))
    return {"labels": labels[:n].copy(), "states": states[:n].copy(), "mass": mass[:n].copy(),
            "LT": LT.value, "lt_clamped": clamped.value, "undetected_mass": und.value}


def resample_U(seed, k):
    return lib().orc_resample_U(int(seed), int(k))


def resample(w, U, n_out):
    ww = _f64(w)
    anc = np.zeros(n_out, dtype=np.int64)
    W = lib().orc_resample(len(ww), _d(ww), float(U), int(n_out), anc.ctypes.data_as(_I64))
    return anc, W


def round_half_away(W):
    import math
    return int(math.floor(W + 0.5)) if W >= 0 else -int(math.floor(-W + 0.5))


def step(m, k, soa, w, z, zprev, n_out_next, births_J):
    """One serial step in the paper's order: predict, births,
    normalisers, update, local estimate, resample.  Returns a dict of every
    intermediate (fp64)."""
    n_surv = soa.shape[1]
    ps, pw = predict(m, k, soa, w)
    bs, bw = births(m, k, n_surv, births_J, zprev)
    xs = np.concatenate([ps, bs], axis=1)
    ws = np.concatenate([pw, bw])
    C = normalizers(m, xs, ws, z)
    w_new, acc = update(m, xs, ws, z, C)
    # N_k = sum_j w_j: sequential fp64 (done inside orc_resample as well)
    Wseq = 0.0
    for v in w_new.tolist():
        Wseq += v
    W_pred = 0.0
    for v in ws.tolist():
        W_pred += v
    est = extract(m, acc, Wseq, W_pred)
    U = resample_U(m.seed, k)
    n_out = n_out_next(est["LT"]) if callable(n_out_next) else int(n_out_next)
    anc, _ = resample(w_new, U, n_out)
    off = xs[:, anc]
    return {"pred": xs, "w_pred": ws, "C": C, "w_upd": w_new, "acc": acc, "W": Wseq, "W_pred": W_pred,
            "est": est, "U": U, "n_out": n_out, "anc": anc, "offspring": off,
            "w_off": np.full(n_out, Wseq / n_out if n_out else 0.0)}
