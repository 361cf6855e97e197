"""Thin ctypes binding of include/phd.h (argument marshalling only).

Every step of the filter runs in the CUDA kernels of libphd.so; this module
only converts numpy / torch arrays to pointers.  There is no fallback: if the
library is missing or no CUDA device is present, the calls fail loudly.
"""
import ctypes
import os

import numpy as np

from . import build as _build

ABI_VERSION = 3
STAGE_RESAMPLED = 0
STAGE_PREDICTED = 1

STATUS = {0: "PHD_OK", 1: "PHD_EINVAL", 2: "PHD_ESTATE", 3: "PHD_ECAPACITY", 4: "PHD_EMODEL",
          5: "PHD_ENOMEM", 6: "PHD_ECUDA", 7: "PHD_ENCCL", 8: "PHD_ENODEV"}


class PhdError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class Params(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("meas", ctypes.c_int32), ("T", ctypes.c_double),
                ("sigma_a", ctypes.c_double), ("p_s", ctypes.c_double), ("p_d", ctypes.c_double),
                ("sigma_z", ctypes.c_double * 2), ("sensor_xy", ctypes.c_double * 2),
                ("region", ctypes.c_double * 4), ("clutter_rate", ctypes.c_double),
                ("birth_mass", ctypes.c_double), ("birth_sigma_v", ctypes.c_double),
                ("births_per_step", ctypes.c_int64), ("particles_per_target", ctypes.c_int64),
                ("fixed_count", ctypes.c_int64), ("count_mode", ctypes.c_int32), ("max_meas", ctypes.c_int32),
                ("capacity", ctypes.c_int64), ("seed", ctypes.c_uint64), ("mode", ctypes.c_int32),
                ("reserved0", ctypes.c_int32), ("exchange_count", ctypes.c_int64), ("birth_model", ctypes.c_int32),
                ("gate_floor", ctypes.c_int32), ("birth_mean", ctypes.c_double * 4), ("birth_std", ctypes.c_double * 4),
                ("stphd_all", ctypes.c_int32), ("gate", ctypes.c_int32), ("proposal_scale", ctypes.c_double)]


_AR_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_size_t)
_AG_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)


class HostTransport(ctypes.Structure):
    _fields_ = [("user", ctypes.c_void_p), ("allreduce_f64", _AR_FN), ("allgather_bytes", _AG_FN)]


def host_transport(allreduce, allgather):
    """phd_host_transport from two Python collectives on host data (test infrastructure):
    allreduce(list of float) -> list of float summed over the ranks in rank order;
    allgather(bytes) -> list of bytes, one per rank."""
    def ar(_user, buf, n):
        try:
            vals = allreduce([buf[i] for i in range(n)])
            for i in range(n):
                buf[i] = vals[i]
            return 0
        except Exception:  # pragma: no cover
            return 1

    def ag(_user, send, recv, nbytes):
        try:
            parts = allgather(ctypes.string_at(send, nbytes))
            ctypes.memmove(recv, b"".join(parts), nbytes * len(parts))
            return 0
        except Exception:  # pragma: no cover
            return 1

    t = HostTransport(None, _AR_FN(ar), _AG_FN(ag))
    t._keep = (t.allreduce_f64, t.allgather_bytes)
    return t


class Estimate(ctypes.Structure):
    _fields_ = [("label", ctypes.c_int32), ("state", ctypes.c_float * 4), ("mass", ctypes.c_float)]


class Summary(ctypes.Structure):
    _fields_ = [("W", ctypes.c_double), ("W_pred", ctypes.c_double), ("undetected_mass", ctypes.c_double),
                ("LT", ctypes.c_int64), ("N", ctypes.c_int64), ("N_out", ctypes.c_int64), ("M", ctypes.c_int32),
                ("n_est", ctypes.c_int32), ("lt_clamped", ctypes.c_int32), ("count_clamped", ctypes.c_int32),
                ("zero_mass", ctypes.c_int32), ("near_half", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = ["phd_abi_version", "phd_status_str", "phd_last_error", "phd_nccl_unique_id", "phd_workspace_size",
           "phd_create", "phd_destroy", "phd_set_particles", "phd_get_particles", "phd_predict", "phd_update",
           "phd_extract", "phd_resample_exchange", "phd_step", "phd_get_normalizers", "phd_get_accumulators",
           "phd_get_ancestors", "phd_get_resample_meta", "phd_launch_count", "phd_set_timing", "phd_get_timing",
           "phd_philox4x32_10", "phd_rank_block", "phd_resample_bounds", "phd_plan_exchange",
           "phd_group_create", "phd_group_destroy", "phd_create_in_group", "phd_get_local_estimates",
           "phd_get_gate_stats", "phd_exchange_path", "phd_set_retained_measurements", "phd_init_population",
           "phd_philox4x32_10_device", "phd_create_with_transport", "phd_get_graph_stats"]

_lib = None
_P = ctypes.c_void_p
_F = ctypes.POINTER(ctypes.c_float)
_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_I32 = ctypes.POINTER(ctypes.c_int32)
_U32 = ctypes.POINTER(ctypes.c_uint32)


def lib_path():
    return _build.LIB


def load(build_if_missing=True):
    """Load libphd.so (building it when missing and nvcc is available)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("PHD_LIB") or _build.LIB  # PHD_LIB: an alternate build (tuning experiments)
    if build_if_missing and path == _build.LIB:
        _build.build()
    if not os.path.exists(path):
        raise OSError("libphd.so not built (%s); run __graft_entry__.build()" % path)
    L = ctypes.CDLL(path)
    L.phd_abi_version.restype = ctypes.c_int32
    L.phd_status_str.restype = ctypes.c_char_p
    L.phd_status_str.argtypes = [ctypes.c_int]
    L.phd_last_error.restype = ctypes.c_char_p
    L.phd_last_error.argtypes = [_P]
    L.phd_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.phd_workspace_size.argtypes = [ctypes.POINTER(Params), ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]
    L.phd_create.argtypes = [ctypes.POINTER(Params), ctypes.c_int32, ctypes.c_int32, ctypes.c_char_p,
                             ctypes.c_int32, _P, _P, ctypes.POINTER(_P)]
    L.phd_create_in_group.argtypes = [ctypes.POINTER(Params), _P, ctypes.c_int32, ctypes.c_int32, _P, _P,
                                      ctypes.POINTER(_P)]
    L.phd_create_with_transport.argtypes = [ctypes.POINTER(Params), ctypes.c_int32, ctypes.c_int32,
                                            ctypes.POINTER(HostTransport), ctypes.c_int32, _P, _P, ctypes.POINTER(_P)]
    L.phd_group_create.argtypes = [ctypes.c_int32, ctypes.POINTER(_P)]
    L.phd_group_destroy.argtypes = [_P]
    L.phd_group_destroy.restype = None
    L.phd_destroy.argtypes = [_P]
    L.phd_destroy.restype = None
    L.phd_set_particles.argtypes = [_P, _P, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_int32]
    L.phd_get_particles.argtypes = [_P, _F, _F, ctypes.c_int64, _I64, _I64]
    L.phd_predict.argtypes = [_P, ctypes.c_int32, _P, ctypes.c_int32]
    L.phd_update.argtypes = [_P, _P, ctypes.c_int32]
    L.phd_extract.argtypes = [_P, ctypes.POINTER(Estimate), ctypes.c_int32, _I32, ctypes.POINTER(Summary)]
    L.phd_resample_exchange.argtypes = [_P, ctypes.c_int32]
    L.phd_step.argtypes = [_P, ctypes.c_int32, _P, ctypes.c_int32, ctypes.POINTER(Estimate), ctypes.c_int32,
                           _I32, ctypes.POINTER(Summary)]
    L.phd_get_normalizers.argtypes = [_P, _D, ctypes.c_int32]
    L.phd_get_accumulators.argtypes = [_P, _D, ctypes.c_int32]
    L.phd_get_ancestors.argtypes = [_P, _I32, ctypes.c_int64, _I64, _I64]
    L.phd_get_local_estimates.argtypes = [_P, ctypes.POINTER(Estimate), ctypes.c_int32, _I32]
    L.phd_get_resample_meta.argtypes = [_P, _D, _D, _I64, _D]
    L.phd_get_gate_stats.argtypes = [_P, _I64]
    L.phd_set_retained_measurements.argtypes = [_P, _P, ctypes.c_int32]
    L.phd_init_population.argtypes = [_P, ctypes.c_double, _D, _D, ctypes.c_double]
    L.phd_philox4x32_10_device.argtypes = [ctypes.c_uint64, _P, ctypes.c_int64, _P, _P]
    L.phd_get_graph_stats.argtypes = [_P, _I64, _I64]
    L.phd_exchange_path.argtypes = [_P]
    L.phd_exchange_path.restype = ctypes.c_int32
    L.phd_launch_count.argtypes = [_P]
    L.phd_launch_count.restype = ctypes.c_int64
    L.phd_set_timing.argtypes = [_P, ctypes.c_int32]
    L.phd_get_timing.argtypes = [_P, _F]
    L.phd_philox4x32_10.argtypes = [_U32, _U32, _U32]
    L.phd_philox4x32_10.restype = None
    L.phd_rank_block.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _I64, _I64]
    L.phd_resample_bounds.argtypes = [ctypes.c_int32, _D, ctypes.c_int64, ctypes.c_double, _I64, _D]
    L.phd_plan_exchange.argtypes = [ctypes.c_int32, ctypes.c_int32, _I64, ctypes.c_int64, ctypes.c_int64,
                                    _I64, _I64, _I64, _I64]
    _lib = L
    return L


def params_from(model):
    """phd_params from a scenario.configs.Model-like object."""
    p = Params()
    p.abi_version = ABI_VERSION
    p.meas = int(model.meas)
    p.T, p.sigma_a, p.p_s, p.p_d = float(model.T), float(model.sigma_a), float(model.p_s), float(model.p_d)
    p.sigma_z[0], p.sigma_z[1] = float(model.sigma_z[0]), float(model.sigma_z[1])
    p.sensor_xy[0], p.sensor_xy[1] = float(model.sensor_xy[0]), float(model.sensor_xy[1])
    for i in range(4):
        p.region[i] = float(model.region[i])
    p.clutter_rate = float(model.clutter_rate)
    p.birth_mass = float(model.birth_mass)
    p.birth_sigma_v = float(model.birth_sigma_v)
    p.births_per_step = int(model.births_per_step)
    p.particles_per_target = int(model.particles_per_target)
    p.fixed_count = int(model.fixed_count)
    p.count_mode = int(model.count_mode)
    p.max_meas = int(model.max_meas)
    p.capacity = int(model.capacity)
    p.seed = int(model.seed)
    p.mode = int(getattr(model, "mode", 0))
    p.reserved0 = 0
    p.exchange_count = int(getattr(model, "exchange_count", 0))
    p.birth_model = int(getattr(model, "birth_model", 0))
    p.gate_floor = int(getattr(model, "gate_floor", 0))
    for i in range(4):
        p.birth_mean[i] = float(getattr(model, "birth_mean", (0.0, 0.0, 0.0, 0.0))[i])
        p.birth_std[i] = float(getattr(model, "birth_std", (0.0, 0.0, 0.0, 0.0))[i])
    p.stphd_all = int(getattr(model, "stphd_all", 0))
    p.gate = int(getattr(model, "gate", 0))
    p.proposal_scale = float(getattr(model, "proposal_scale", 1.0))
    return p


def _ptr(a):
    """Raw pointer of a contiguous numpy array or torch tensor (host or device)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous()
        return a.data_ptr()
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _f32(a):
    if a is None or hasattr(a, "data_ptr"):
        return a
    return np.ascontiguousarray(a, dtype=np.float32)


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    st = load().phd_nccl_unique_id(buf)
    if st != 0:
        raise PhdError(st, "ncclGetUniqueId failed")
    return buf.raw


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    load().phd_philox4x32_10(c, k, o)
    return [int(o[i]) for i in range(4)]


def philox_device(seed, ctr, out):
    """The kernels' Philox on n counters: ctr and out are device buffers of n x 4 uint32
    (e.g. torch int32 CUDA tensors of shape [n, 4]); synchronous."""
    n = int(ctr.shape[0])
    st = load().phd_philox4x32_10_device(int(seed), ctypes.c_void_p(ctr.data_ptr()), n,
                                         ctypes.c_void_p(out.data_ptr()), None)
    if st != 0:
        raise PhdError(st, "phd_philox4x32_10_device")


def rank_block(n, world, rank):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    st = load().phd_rank_block(int(n), int(world), int(rank), ctypes.byref(lo), ctypes.byref(hi))
    if st != 0:
        raise PhdError(st, "phd_rank_block")
    return lo.value, hi.value


def resample_bounds(W_r, n_out, U):
    W_r = np.ascontiguousarray(W_r, dtype=np.float64)
    b = np.zeros(len(W_r) + 1, dtype=np.int64)
    W = ctypes.c_double()
    st = load().phd_resample_bounds(len(W_r), W_r.ctypes.data_as(_D), int(n_out), float(U),
                                    b.ctypes.data_as(_I64), ctypes.byref(W))
    if st != 0:
        raise PhdError(st, "phd_resample_bounds")
    return b, W.value


def plan_exchange(world, rank, bounds, n_out, J):
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    arrs = [np.zeros(world, dtype=np.int64) for _ in range(4)]
    st = load().phd_plan_exchange(int(world), int(rank), bounds.ctypes.data_as(_I64), int(n_out), int(J),
                                  *[a.ctypes.data_as(_I64) for a in arrs])
    if st != 0:
        raise PhdError(st, "phd_plan_exchange")
    return tuple(arrs)


def workspace_size(model, world=1):
    p = params_from(model)
    n = ctypes.c_size_t()
    st = load().phd_workspace_size(ctypes.byref(p), int(world), ctypes.byref(n))
    if st != 0:
        raise PhdError(st, "phd_workspace_size")
    return n.value


class LocalGroup:
    """In-process rank group (phd_group): run `world` Filter contexts of one
    process (one thread per rank) through the multi-rank path without NCCL."""

    def __init__(self, world):
        self.L = load()
        h = _P()
        st = self.L.phd_group_create(int(world), ctypes.byref(h))
        if st != 0:
            raise PhdError(st, "phd_group_create")
        self.h, self.world = h, world

    def close(self):
        if getattr(self, "h", None):
            self.L.phd_group_destroy(self.h)
            self.h = None


class Filter:
    """One rank's filter context (phd_ctx)."""

    def __init__(self, model, rank=0, world=1, nccl_id=None, device=0, stream=None, workspace=None, group=None,
                 transport=None):
        self.L = load()
        self.model = model
        self.params = params_from(model)
        self.rank, self.world = rank, (group.world if group is not None else world)
        self._ws = workspace  # keep the caller's buffer alive
        self._group = group
        h = _P()
        self._transport = transport
        if group is not None:
            st = self.L.phd_create_in_group(ctypes.byref(self.params), group.h, int(rank), int(device), stream,
                                            _ptr(workspace), ctypes.byref(h))
        elif transport is not None:
            st = self.L.phd_create_with_transport(ctypes.byref(self.params), int(rank), int(world),
                                                  ctypes.byref(transport), int(device), stream, _ptr(workspace),
                                                  ctypes.byref(h))
        else:
            st = self.L.phd_create(ctypes.byref(self.params), int(rank), int(world), nccl_id, int(device),
                                   stream, _ptr(workspace), ctypes.byref(h))
        if st != 0:
            raise PhdError(st, "phd_create failed (see stderr)")
        self.h = h
        self.cap = int(model.max_meas)
        self._est = (Estimate * max(1, self.cap))()
        self._sum = Summary()
        self._n = ctypes.c_int32()

    def close(self):
        if getattr(self, "h", None):
            self.L.phd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != 0:
            msg = self.L.phd_last_error(self.h)
            raise PhdError(st, "%s: %s" % (what, msg.decode() if msg else ""))

    # ---- population ----
    def set_particles(self, soa4, w, n_global, stage=STAGE_RESAMPLED, mass=0.0):
        soa4 = _f32(soa4)
        w = _f32(w)
        n_local = soa4.shape[1] if hasattr(soa4, "shape") else 0
        self._keep = (soa4, w)
        self._check(self.L.phd_set_particles(self.h, _ptr(soa4), _ptr(w), int(n_local), int(n_global),
                                             float(mass), int(stage)), "phd_set_particles")

    def init_population(self, total_mass, box=None, mass_box=None, v_max=20.0):
        """t = 0 population on the device: y-stratified over box, total mass
        total_mass (only inside mass_box when given).  Collective."""
        b = None if box is None else (ctypes.c_double * 4)(*[float(v) for v in box])
        mb = None if mass_box is None else (ctypes.c_double * 4)(*[float(v) for v in mass_box])
        self._check(self.L.phd_init_population(self.h, float(total_mass), b, mb, float(v_max)),
                    "phd_init_population")

    def get_particles(self, cap=None):
        n = ctypes.c_int64()
        g0 = ctypes.c_int64()
        self.L.phd_get_particles(self.h, None, None, 0, ctypes.byref(n), ctypes.byref(g0))
        nn = n.value
        soa = np.zeros((4, nn), dtype=np.float32)
        w = np.zeros(nn, dtype=np.float32)
        self._check(self.L.phd_get_particles(self.h, soa.ctypes.data_as(_F), w.ctypes.data_as(_F), nn,
                                             ctypes.byref(n), ctypes.byref(g0)), "phd_get_particles")
        return soa, w, g0.value

    # ---- the step ----
    def predict(self, k, z_prev=None):
        zp = _f32(z_prev)
        m = 0 if zp is None else int(zp.shape[0])
        self._check(self.L.phd_predict(self.h, int(k), _ptr(zp), m), "phd_predict")

    def update(self, z):
        z = _f32(z)
        self._zkeep = z
        self._check(self.L.phd_update(self.h, _ptr(z), int(z.shape[0])), "phd_update")

    def extract(self):
        self._check(self.L.phd_extract(self.h, self._est, self.cap, ctypes.byref(self._n), ctypes.byref(self._sum)),
                    "phd_extract")
        return self._estimates(), self._sum.as_dict()

    def estimates(self):
        """Estimates of the last extract / step: labels, states (x, vx, y, vy), masses."""
        return self._estimates()

    def _estimates(self):
        n = self._n.value
        labels = np.array([self._est[i].label for i in range(n)], dtype=np.int32)
        states = np.array([list(self._est[i].state) for i in range(n)], dtype=np.float32).reshape(n, 4)
        mass = np.array([self._est[i].mass for i in range(n)], dtype=np.float32)
        return {"labels": labels, "states": states, "mass": mass}

    def resample_exchange(self, k):
        self._check(self.L.phd_resample_exchange(self.h, int(k)), "phd_resample_exchange")

    def step(self, k, z):
        z = _f32(z)
        self._zkeep = z
        self._check(self.L.phd_step(self.h, int(k), _ptr(z), int(z.shape[0]), self._est, self.cap,
                                    ctypes.byref(self._n), ctypes.byref(self._sum)), "phd_step")
        return self._sum

    def step_raw(self, k, zptr, M):
        """phd_step with a raw (host or device) measurement pointer; returns n_est."""
        st = self.L.phd_step(self.h, int(k), zptr, int(M), self._est, self.cap, ctypes.byref(self._n),
                             ctypes.byref(self._sum))
        self._check(st, "phd_step")
        return self._n.value

    # ---- introspection ----
    def normalizers(self, M):
        C = np.zeros(max(M, 1))
        self._check(self.L.phd_get_normalizers(self.h, C.ctypes.data_as(_D), len(C)), "phd_get_normalizers")
        return C[:M]

    def accumulators(self, M):
        a = np.zeros((max(M, 1), 5))
        self._check(self.L.phd_get_accumulators(self.h, a.ctypes.data_as(_D), len(a)), "phd_get_accumulators")
        return a[:M]

    def ancestors(self):
        n = ctypes.c_int64()
        first = ctypes.c_int64()
        self.L.phd_get_ancestors(self.h, (ctypes.c_int32 * 1)(), 0, ctypes.byref(n), ctypes.byref(first))
        a = np.zeros(max(n.value, 1), dtype=np.int32)
        self._check(self.L.phd_get_ancestors(self.h, a.ctypes.data_as(_I32), len(a), ctypes.byref(n),
                                             ctypes.byref(first)), "phd_get_ancestors")
        return a[:n.value], first.value

    def local_estimates(self):
        """DCP mode: this rank's pre-fusion estimates of the last extract."""
        n = ctypes.c_int32()
        buf = (Estimate * max(1, self.cap))()
        self._check(self.L.phd_get_local_estimates(self.h, buf, self.cap, ctypes.byref(n)), "phd_get_local_estimates")
        k = n.value
        return {"labels": np.array([buf[i].label for i in range(k)], dtype=np.int32),
                "states": np.array([list(buf[i].state) for i in range(k)], dtype=np.float32).reshape(k, 4),
                "mass": np.array([buf[i].mass for i in range(k)], dtype=np.float32)}

    def resample_meta(self):
        W, U = ctypes.c_double(), ctypes.c_double()
        n = ctypes.c_int64()
        Wr = np.zeros(self.world)
        self._check(self.L.phd_get_resample_meta(self.h, ctypes.byref(W), ctypes.byref(U), ctypes.byref(n),
                                                 Wr.ctypes.data_as(_D)), "phd_get_resample_meta")
        return {"W": W.value, "U": U.value, "N_out": n.value, "W_r": Wr}

    def gate_stats(self):
        """(used, entries, pairs evaluated, tiles) of the last update's gated path."""
        out = np.zeros(4, dtype=np.int64)
        self._check(self.L.phd_get_gate_stats(self.h, out.ctypes.data_as(_I64)), "phd_get_gate_stats")
        return {"used": int(out[0]), "entries": int(out[1]), "pairs": int(out[2]), "tiles": int(out[3])}

    def set_retained_measurements(self, z):
        """Z_{k-1} for the births of the next predict/step (checkpoint resume)."""
        z = _f32(z)
        self._zkeep = z
        self._check(self.L.phd_set_retained_measurements(self.h, _ptr(z), int(z.shape[0])),
                    "phd_set_retained_measurements")

    def checkpoint(self, path, k, z):
        """Save this rank's resampled population after step k with Z_k (which the
        births of step k + 1 are drawn around): an npz that restore() resumes from
        exactly (counter-based noise)."""
        soa, w, g0 = self.get_particles()
        meta = self.resample_meta()
        np.savez(path, soa=soa, w=w, g0=g0, k=int(k), n_out=int(meta["N_out"]), z=_f32(z), rank=self.rank,
                 world=self.world)

    def restore(self, path):
        """Load a checkpoint() of this rank; returns the step k it was taken after."""
        d = np.load(path)
        if int(d["rank"]) != self.rank or int(d["world"]) != self.world:
            raise ValueError("checkpoint of rank %d/%d, filter is %d/%d" % (int(d["rank"]), int(d["world"]),
                                                                         self.rank, self.world))
        self.set_particles(np.ascontiguousarray(d["soa"]), np.ascontiguousarray(d["w"]), int(d["n_out"]))
        self.set_retained_measurements(d["z"])
        return int(d["k"])

    def graph_stats(self):
        """(graphs captured, replays) of phd_step's CUDA-graph path."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.L.phd_get_graph_stats(self.h, ctypes.byref(a), ctypes.byref(b)), "phd_get_graph_stats")
        return a.value, b.value

    def exchange_path(self):
        """0 none, 1 send/recv, 2 fused gather + exchange over peer memory."""
        return int(self.L.phd_exchange_path(self.h))

    def launch_count(self):
        return self.L.phd_launch_count(self.h)

    def set_timing(self, on=True):
        self._check(self.L.phd_set_timing(self.h, 1 if on else 0), "phd_set_timing")

    def timing(self):
        ms = (ctypes.c_float * 8)()
        self._check(self.L.phd_get_timing(self.h, ms), "phd_get_timing")
        keys = ["predict", "pass1", "pass2", "update", "extract", "resample", "exchange", "step"]
        return dict(zip(keys, [float(v) for v in ms]))
