"""ctypes binding of libvpetabc.so (include/vpetabc.h): argument marshalling only.

Every step of the hot path runs in the CUDA library; this module only converts Python
arguments to the C structs and pointers.  There is no CPU fallback: if the library is
missing or cannot be loaded, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VPET_LIB") or os.path.join(_HERE, "libvpetabc.so")  # VPET_LIB: tuning builds only

ABI_VERSION = 2  # include/vpetabc.h VPETABC_ABI_VERSION
MAX_P = 8
MAX_MODELS = 4
MAX_L = 128
KINDS = {"2TCM_IRR": 0, "2TCM_REV": 1, "MRTM": 2, "LPNTPET": 3}
DISTANCES = {"L1": 1, "WL2": 2}
ACCEPTS = {"TOPN": 0, "EPS": 1}
INPUTS = {"PWL": 0, "FENG": 1}
FLAG_TIMING, FLAG_EXACT, FLAG_COUNT_WORK, FLAG_NO_PRUNE, FLAG_NO_REORDER, FLAG_NO_TREE = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
FLAG_DENSE_TC = 0x40
FLAG_FORCE_FALLBACK = 0x80
PTR_TACS_DEVICE, PTR_OUT_DEVICE = 0x1, 0x2
STATUS = {0: "OK", 1: "E_ARG", 2: "E_STATE", 3: "E_NOMEM", 4: "E_CUDA", 5: "E_UNSUPPORTED"}

SYMBOLS = ("abc_init", "abc_set_input_function", "abc_set_frames", "abc_run_voxels", "abc_model_select",
           "abc_set_stream", "abc_sync", "abc_get_stats", "abc_get_bank", "abc_last_error", "abc_destroy",
           "abc_abi_version", "abc_response_envelope",
           "abc_set_sim_noise", "abc_patlak", "abc_reduce_accepted")


class ModelSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved0", C.c_uint32), ("n_draws", C.c_uint64),
                ("lo", C.c_float * MAX_P), ("hi", C.c_float * MAX_P)]


class Config(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("n_models", C.c_uint32), ("seed", C.c_uint64),
                ("device", C.c_int32), ("distance", C.c_int32), ("accept", C.c_int32),
                ("n_accept", C.c_uint32), ("epsilon", C.c_double), ("lpnt_step_min", C.c_double),
                ("flags", C.c_uint32), ("reserved1", C.c_uint32), ("model", ModelSpec * MAX_MODELS)]


RESULT_FIELDS = ("prob", "preferred", "count", "mean", "sd", "q", "ki_mean", "ki_sd", "ki_q", "acc_idx", "acc_dist")


class Result(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in RESULT_FIELDS]


class Stats(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("gpu_launches", C.c_uint32), ("n_voxels", C.c_uint64),
                ("n_draws", C.c_uint64), ("n_fallback", C.c_uint64), ("n_fallback_exact", C.c_uint64),
                ("frame_updates", C.c_uint64),
                ("bound_updates", C.c_uint64),
                ("lp", C.c_uint32), ("heap_k", C.c_uint32),
                ("ms_h2d", C.c_double), ("ms_bank", C.c_double), ("ms_order", C.c_double),
                ("ms_scan", C.c_double), ("ms_certify", C.c_double), ("ms_fallback", C.c_double),
                ("ms_d2h", C.c_double), ("ms_total", C.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "struct_size"}


class AbcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libvpetabc.so; raise if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(the CUDA library is required; there is no CPU fallback)")
    L = C.CDLL(path)
    vp = C.c_void_p
    L.abc_init.argtypes = [C.POINTER(Config), C.POINTER(vp)]
    L.abc_set_input_function.argtypes = [vp, C.c_int32, vp, vp, C.c_uint32]
    L.abc_set_frames.argtypes = [vp, vp, vp, vp, C.c_uint32]
    L.abc_run_voxels.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.POINTER(Result)]
    L.abc_model_select.argtypes = [vp, vp, C.c_uint64, C.c_uint32, vp, vp]
    L.abc_set_sim_noise.argtypes = [vp, C.c_double, C.c_double]
    L.abc_patlak.argtypes = [vp, vp, C.c_uint64, C.c_double, C.c_uint32, vp, vp]
    L.abc_response_envelope.argtypes = [vp, vp, C.c_uint64, C.c_uint32, vp, C.c_uint32, C.c_uint32, vp]
    L.abc_reduce_accepted.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(Result)]
    L.abc_set_stream.argtypes = [vp, vp]
    L.abc_sync.argtypes = [vp]
    L.abc_get_stats.argtypes = [vp, C.POINTER(Stats)]
    L.abc_get_bank.argtypes = [vp, vp, C.c_uint64, C.c_uint64]
    L.abc_last_error.argtypes = [vp]
    L.abc_last_error.restype = C.c_char_p
    L.abc_destroy.argtypes = [vp]
    L.abc_destroy.restype = None
    L.abc_abi_version.restype = C.c_uint32
    assert C.sizeof(Config) == 376, C.sizeof(Config)
    if L.abc_abi_version() != ABI_VERSION:
        raise RuntimeError(f"{path}: ABI version {L.abc_abi_version()} != {ABI_VERSION} of this binding (rebuild)")
    _lib = L
    return L


def make_config(models, seed=2026, distance="WL2", accept="TOPN", n_accept=1, epsilon=0.0,
                lpnt_step_min=0.05, flags=0, device=0) -> Config:
    cfg = Config()
    cfg.struct_size = C.sizeof(Config)
    cfg.n_models = len(models)
    cfg.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
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


def host_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)
