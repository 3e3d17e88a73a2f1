"""ctypes binding of the CPU ORACLE (libvpetabc_oracle.so) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module.  It shares no code with the product package
(paper_2603_14859_b200); the Python API mirrors the product binding so that a test can
build both from the same keyword arguments.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

MAX_P = 8
MAX_MODELS = 4
KINDS = {"2TCM_IRR": 0, "2TCM_REV": 1, "MRTM": 2, "LPNTPET": 3}
DISTANCES = {"L1": 1, "WL2": 2}
ACCEPTS = {"TOPN": 0, "EPS": 1}
INPUTS = {"PWL": 0, "FENG": 1}
STATUS = {0: "OK", 1: "E_ARG", 2: "E_STATE", 3: "E_NOMEM", 4: "E_CUDA", 5: "E_UNSUPPORTED"}


class ModelSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved0", C.c_uint32), ("n_draws", C.c_uint64),
                ("lo", C.c_float * MAX_P), ("hi", C.c_float * MAX_P)]


class Config(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("n_models", C.c_uint32), ("seed", C.c_uint64),
                ("device", C.c_int32), ("distance", C.c_int32), ("accept", C.c_int32),
                ("n_accept", C.c_uint32), ("epsilon", C.c_double), ("lpnt_step_min", C.c_double),
                ("flags", C.c_uint32), ("reserved1", C.c_uint32), ("model", ModelSpec * MAX_MODELS)]


class Result(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("prob", "preferred", "count", "mean", "sd", "q", "ki_mean",
                                           "ki_sd", "ki_q", "acc_idx", "acc_dist")]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = _build.build()
        L = C.CDLL(path)
        vp = C.c_void_p
        L.abc_init.argtypes = [C.POINTER(Config), C.POINTER(vp)]
        L.abc_set_input_function.argtypes = [vp, C.c_int32, vp, vp, C.c_uint32]
        L.abc_set_frames.argtypes = [vp, vp, vp, vp, C.c_uint32]
        L.abc_run_voxels.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.POINTER(Result)]
        L.abc_model_select.argtypes = [vp, vp, C.c_uint64, C.c_uint32, vp, vp]
        L.abc_set_sim_noise.argtypes = [vp, C.c_double, C.c_double]
        L.abc_patlak.argtypes = [vp, vp, C.c_uint64, C.c_double, C.c_uint32, vp, vp]
        L.oracle_std_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32]
        L.oracle_std_normal.restype = C.c_double
        L.abc_response_envelope.argtypes = [vp, vp, C.c_uint64, C.c_uint32, vp, C.c_uint32, C.c_uint32, vp]
        L.abc_last_error.argtypes = [vp]
        L.abc_last_error.restype = C.c_char_p
        L.abc_destroy.argtypes = [vp]
        L.abc_destroy.restype = None
        L.oracle_set_threads.argtypes = [C.c_int]
        L.oracle_set_threads.restype = None
        L.oracle_get_threads.restype = C.c_int
        L.oracle_philox4x32_10.argtypes = [vp, vp, vp]
        L.oracle_philox4x32_10.restype = None
        L.oracle_uniform.argtypes = [C.c_uint32]
        L.oracle_uniform.restype = C.c_float
        L.oracle_draw.argtypes = [vp, C.c_uint64, vp, vp]
        L.oracle_simulate.argtypes = [vp, C.c_int32, vp, vp]
        L.oracle_bank.argtypes = [vp, vp]
        L.oracle_distance.argtypes = [C.c_int32, vp, vp, vp, C.c_uint32]
        L.oracle_distance.restype = C.c_double
        L.oracle_gamma_variate.argtypes = [C.c_double] * 4
        L.oracle_gamma_variate.restype = C.c_double
        L.oracle_feng.argtypes = [vp, C.c_double]
        L.oracle_feng.restype = C.c_double
        L.oracle_quantile7.argtypes = [vp, C.c_uint32, C.c_double]
        L.oracle_quantile7.restype = C.c_double
        L.oracle_family_width.argtypes = [C.c_int32]
        L.oracle_family_width.restype = C.c_uint32
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


def family_width(kind: str) -> int:
    return int(lib().oracle_family_width(KINDS[kind]))


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def uniform(x: int) -> float:
    return float(lib().oracle_uniform(int(x) & 0xFFFFFFFF))


def distance(dist: str, y, s, w=None) -> float:
    y = np.ascontiguousarray(y, dtype=np.float32)
    s = np.ascontiguousarray(s, dtype=np.float32)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
    return float(lib().oracle_distance(DISTANCES[dist], _ptr(y), _ptr(s), _ptr(w), len(y)))


def gamma_variate(tD, tP, alpha, t) -> float:
    return float(lib().oracle_gamma_variate(tD, tP, alpha, t))


def feng(params, t) -> float:
    p = np.ascontiguousarray(params, dtype=np.float64)
    return float(lib().oracle_feng(_ptr(p), t))


def std_normal(seed: int, i: int, f: int) -> float:
    return float(lib().oracle_std_normal(seed, i, f))


def quantile7(sorted_x, q) -> float:
    x = np.ascontiguousarray(sorted_x, dtype=np.float64)
    return float(lib().oracle_quantile7(_ptr(x), len(x), q))


def make_config(models, seed=2026, distance="WL2", accept="TOPN", n_accept=1, epsilon=0.0,
                lpnt_step_min=0.05, flags=0, device=0) -> Config:
    cfg = Config()
    cfg.struct_size = C.sizeof(Config)
    cfg.n_models = len(models)
    cfg.seed = int(seed)
    cfg.device = int(device)
    cfg.distance = DISTANCES[distance]
    cfg.accept = ACCEPTS[accept]
    cfg.n_accept = int(n_accept)
    cfg.epsilon = float(epsilon)
    cfg.lpnt_step_min = float(lpnt_step_min)
    cfg.flags = int(flags)
    for m, spec in enumerate(models):
        ms = cfg.model[m]
        ms.kind = KINDS[spec["kind"]]
        ms.n_draws = int(spec["n_draws"])
        lo = list(spec["lo"]) + [0.0] * (MAX_P - len(spec["lo"]))
        hi = list(spec["hi"]) + [0.0] * (MAX_P - len(spec["hi"]))
        for k in range(MAX_P):
            ms.lo[k] = lo[k]
            ms.hi[k] = hi[k]
    return cfg


class OracleContext:
    """Mirror of paper_2603_14859_b200.AbcContext, computed by the CPU oracle."""

    def __init__(self, models, **kw):
        self.models = [dict(m) for m in models]
        self.kw = kw
        self.cfg = make_config(self.models, **kw)
        h = C.c_void_p()
        st = lib().abc_init(C.byref(self.cfg), C.byref(h))
        if st != 0:
            raise OracleError(st, "abc_init rejected the configuration")
        self._h = h
        self.M = len(models)
        self.P = family_width(models[0]["kind"])
        self.N = sum(int(m["n_draws"]) for m in models)
        self.L = None

    def _check(self, st):
        if st != 0:
            raise OracleError(st, lib().abc_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            lib().abc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_input_function(self, kind, value, t=None):
        v = np.ascontiguousarray(value, dtype=np.float64)
        tt = None if t is None else np.ascontiguousarray(t, dtype=np.float64)
        self._check(lib().abc_set_input_function(self._h, INPUTS[kind], _ptr(tt), _ptr(v), len(v)))

    def set_frames(self, start, dur, weight=None):
        s = np.ascontiguousarray(start, dtype=np.float64)
        d = np.ascontiguousarray(dur, dtype=np.float64)
        w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float32)
        self._check(lib().abc_set_frames(self._h, _ptr(s), _ptr(d), _ptr(w), len(s)))
        self.L = len(s)

    def draw(self, i):
        m = np.zeros(1, dtype=np.int32)
        th = np.zeros(MAX_P, dtype=np.float32)
        self._check(lib().oracle_draw(self._h, int(i), _ptr(m), _ptr(th)))
        return int(m[0]), th[: self.P].copy()

    def simulate(self, kind, theta):
        th = np.zeros(MAX_P, dtype=np.float32)
        th[: len(theta)] = np.asarray(theta, dtype=np.float32)
        out = np.zeros(self.L, dtype=np.float64)
        self._check(lib().oracle_simulate(self._h, KINDS[kind], _ptr(th), _ptr(out)))
        return out

    def patlak(self, tacs, t_star):
        """(K_i, intercept) per voxel: OLS Patlak line over frames with mid-time >= t_star."""
        y = np.ascontiguousarray(tacs, dtype=np.float32)
        J = y.shape[0]
        ki = np.zeros(J, dtype=np.float32)
        v0 = np.zeros(J, dtype=np.float32)
        self._check(lib().abc_patlak(self._h, _ptr(y), J, float(t_star), 0, _ptr(ki), _ptr(v0)))
        return ki, v0

    def set_sim_noise(self, ell, half_life_min=float("inf")):
        self._check(lib().abc_set_sim_noise(self._h, float(ell), float(half_life_min)))

    def response_envelope(self, acc_idx, t):
        """J x T x 3 (2.5/50/97.5 %) of 1 + gamma/k2a g(t) over accepted lp-ntPET draws."""
        idx = np.ascontiguousarray(acc_idx, dtype=np.uint64)
        tt = np.ascontiguousarray(t, dtype=np.float64)
        J, n = idx.shape
        out = np.zeros((J, tt.size, 3), dtype=np.float32)
        self._check(lib().abc_response_envelope(self._h, _ptr(idx), J, n, _ptr(tt), tt.size, 0, _ptr(out)))
        return out

    def bank(self):
        out = np.zeros((self.N, self.L), dtype=np.float32)
        self._check(lib().oracle_bank(self._h, _ptr(out)))
        return out

    def run_voxels(self, tacs, want=("prob", "preferred", "count", "mean", "sd", "q", "ki_mean",
                                     "ki_sd", "ki_q", "acc_idx", "acc_dist")):
        y = np.ascontiguousarray(tacs, dtype=np.float32)
        J = y.shape[0]
        M, P = self.M, self.P
        topn = self.kw.get("accept", "TOPN") == "TOPN"
        n = int(self.kw.get("n_accept", 1))
        shapes = {"prob": ((J, M), np.float32), "preferred": ((J,), np.int32), "count": ((J, M), np.uint32),
                  "mean": ((J, P), np.float32), "sd": ((J, P), np.float32), "q": ((J, P, 3), np.float32),
                  "ki_mean": ((J,), np.float32), "ki_sd": ((J,), np.float32), "ki_q": ((J, 3), np.float32),
                  "acc_idx": ((J, n), np.uint64), "acc_dist": ((J, n), np.float64)}
        out = {}
        r = Result()
        for name in want:
            if name in ("acc_idx", "acc_dist") and not topn:
                continue
            shp, dt = shapes[name]
            out[name] = np.zeros(shp, dtype=dt)
            setattr(r, name, out[name].ctypes.data)
        self._check(lib().abc_run_voxels(self._h, _ptr(y) if J else None, J, 0, C.byref(r)))
        return out
