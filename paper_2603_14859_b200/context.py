"""AbcContext: thin Python wrapper over one abc_ctx (one device)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A


def family_width(kind: str) -> int:
    """Parameter columns of a model family: 5 (2TCM: K1,k2,k3,k4,Vb), 7 (RT: R1,k2,k2a,gamma,tD,tP,alpha)."""
    return 7 if kind in ("MRTM", "LPNTPET") else 5


_DTYPES = {"prob": np.float32, "preferred": np.int32, "count": np.uint32, "mean": np.float32, "sd": np.float32,
           "q": np.float32, "ki_mean": np.float32, "ki_sd": np.float32, "ki_q": np.float32, "acc_idx": np.uint64,
           "acc_dist": np.float64}
ALL_OUTPUTS = tuple(_DTYPES)


class AbcContext:
    def __init__(self, models, seed=2026, distance="WL2", accept="TOPN", n_accept=1, epsilon=0.0,
                 lpnt_step_min=0.05, flags=0, device=0):
        self._lib = A.load_library()
        self.models = [dict(m) for m in models]
        self.accept = accept
        self.n_accept = int(n_accept)
        self.device = int(device)
        self.cfg = A.make_config(self.models, seed=seed, distance=distance, accept=accept, n_accept=n_accept,
                                 epsilon=epsilon, lpnt_step_min=lpnt_step_min, flags=flags, device=device)
        h = C.c_void_p()
        st = self._lib.abc_init(C.byref(self.cfg), C.byref(h))
        if st != 0:
            raise A.AbcError(st, "abc_init rejected the configuration")
        self._h = h
        self.M = len(self.models)
        self.P = family_width(self.models[0]["kind"])
        self.N = sum(int(m["n_draws"]) for m in self.models)
        self.L = None

    # -- lifecycle --
    def close(self):
        if getattr(self, "_h", None):
            self._lib.abc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != 0:
            raise A.AbcError(st, self._lib.abc_last_error(self._h).decode())

    # -- configuration --
    def set_input_function(self, kind, value, t=None):
        v = np.ascontiguousarray(value, dtype=np.float64)
        tt = None if t is None else np.ascontiguousarray(t, dtype=np.float64)
        self._check(self._lib.abc_set_input_function(self._h, A.INPUTS[kind], None if tt is None else A.host_ptr(tt),
                                                     A.host_ptr(v), len(v)))

    def set_frames(self, start, dur, weight=None):
        s = np.ascontiguousarray(start, dtype=np.float64)
        d = np.ascontiguousarray(dur, dtype=np.float64)
        w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float32)
        self._check(self._lib.abc_set_frames(self._h, A.host_ptr(s), A.host_ptr(d),
                                             None if w is None else A.host_ptr(w), len(s)))
        self.L = len(s)

    def set_stream(self, stream_handle):
        """Order the context's work on a CUDA stream handle (e.g. torch.cuda.current_stream().cuda_stream)."""
        self._check(self._lib.abc_set_stream(self._h, C.c_void_p(stream_handle) if stream_handle else None))

    def sync(self):
        self._check(self._lib.abc_sync(self._h))

    def stats(self) -> dict:
        s = A.Stats()
        s.struct_size = C.sizeof(A.Stats)
        self._check(self._lib.abc_get_stats(self._h, C.byref(s)))
        return s.as_dict()

    def bank(self, first=0, count=None):
        """Rows of the last run's simulation bank (N x L, FP32) -- diagnostic copy to host."""
        count = self.N - first if count is None else count
        out = np.empty((count, self.L), dtype=np.float32)
        self._check(self._lib.abc_get_bank(self._h, A.host_ptr(out), int(first), int(count)))
        return out

    # -- run --
    def shapes(self, J):
        M, P, n = self.M, self.P, self.n_accept
        return {"prob": (J, M), "preferred": (J,), "count": (J, M), "mean": (J, P), "sd": (J, P), "q": (J, P, 3),
                "ki_mean": (J,), "ki_sd": (J,), "ki_q": (J, 3), "acc_idx": (J, n), "acc_dist": (J, n)}

    def run_voxels(self, tacs, want=ALL_OUTPUTS, out=None):
        """Run Alg. 1 on a J x L float32 array.

        tacs: numpy array (host) or torch CUDA tensor (device).  Outputs are numpy arrays for host
        input and torch CUDA tensors for device input, unless `out` (dict of preallocated arrays /
        tensors, all host or all device) is given.
        """
        is_torch = type(tacs).__module__.startswith("torch")
        flags = 0
        if is_torch:
            import torch
            if tacs.dtype != torch.float32 or not tacs.is_contiguous() or tacs.dim() != 2:
                raise ValueError("tacs must be a contiguous 2-D float32 tensor")
            J = int(tacs.shape[0])
            tptr = C.c_void_p(tacs.data_ptr()) if J else None
            if tacs.is_cuda:
                flags |= A.PTR_TACS_DEVICE
        else:
            y = np.ascontiguousarray(tacs, dtype=np.float32)
            if y.ndim != 2:
                raise ValueError("tacs must be J x L")
            J = y.shape[0]
            tptr = A.host_ptr(y) if J else None
        shapes = self.shapes(J)
        want = [w for w in want if not (self.accept == "EPS" and w in ("acc_idx", "acc_dist"))]
        res = {}
        if out is not None:
            res = dict(out)
        elif is_torch and tacs.is_cuda:
            import torch
            tdt = {np.float32: torch.float32, np.int32: torch.int32, np.uint32: torch.int32,
                   np.uint64: torch.int64, np.float64: torch.float64}
            for name in want:
                res[name] = torch.empty(shapes[name], dtype=tdt[_DTYPES[name]], device=tacs.device)
        else:
            for name in want:
                res[name] = np.empty(shapes[name], dtype=_DTYPES[name])
        r = A.Result()
        dev_out = None
        for name, arr in res.items():
            if type(arr).__module__.startswith("torch"):
                ptr = arr.data_ptr()
                d = bool(arr.is_cuda)
            else:
                ptr = arr.ctypes.data
                d = False
            if dev_out is None:
                dev_out = d
            elif dev_out != d:
                raise ValueError("outputs must be all host or all device")
            setattr(r, name, ptr)
        if dev_out:
            flags |= A.PTR_OUT_DEVICE
        self._check(self._lib.abc_run_voxels(self._h, tptr, J, flags, C.byref(r)))
        return res

    def reduce_accepted(self, acc_idx, n_use, want=("prob", "preferred", "count", "mean", "sd", "q", "ki_mean",
                                                    "ki_sd", "ki_q")):
        """Posterior summaries of the first n_use accepted draws of each row of acc_idx (J x n_acc)
        through abc_reduce_accepted: for a sorted top-n list this is the top-n_use result of the same
        run (SURVEY §8f-3 pilot sweep by truncation).  numpy in -> numpy out; torch CUDA in -> torch
        CUDA out."""
        shapes = self.shapes(0)
        if type(acc_idx).__module__.startswith("torch") and acc_idx.is_cuda:
            import torch
            idx = acc_idx.to(torch.int64).contiguous()
            J, n_acc = int(idx.shape[0]), int(idx.shape[1])
            tdt = {np.float32: torch.float32, np.int32: torch.int32, np.uint32: torch.int32, np.uint64: torch.int64}
            res = {}
            for name in want:
                shp = (J, int(n_use)) if name == "acc_idx" else (J,) + shapes[name][1:]
                res[name] = torch.empty(shp, dtype=tdt[_DTYPES[name]], device=idx.device)
            r = A.Result()
            for name, arr in res.items():
                setattr(r, name, arr.data_ptr())
            self._check(self._lib.abc_reduce_accepted(self._h, C.c_void_p(idx.data_ptr()), J, n_acc, int(n_use),
                                                      A.PTR_TACS_DEVICE | A.PTR_OUT_DEVICE, C.byref(r)))
            return res
        idx = np.ascontiguousarray(acc_idx, dtype=np.uint64)
        J, n_acc = idx.shape
        res = {}
        for name in want:
            shp = (J, int(n_use)) if name == "acc_idx" else (J,) + shapes[name][1:]
            res[name] = np.empty(shp, dtype=_DTYPES[name])
        r = A.Result()
        for name, arr in res.items():
            setattr(r, name, arr.ctypes.data)
        self._check(self._lib.abc_reduce_accepted(self._h, idx.ctypes.data if J else None, J, n_acc, int(n_use), 0,
                                                  C.byref(r)))
        return res

    def model_select(self, tacs):
        """Model probabilities (J x M) and preferred model (J) through abc_model_select (P:109-114,
        P:282).  numpy host array in -> numpy out; torch CUDA tensor in -> torch CUDA tensors out."""
        if type(tacs).__module__.startswith("torch") and tacs.is_cuda:
            import torch
            if tacs.dtype != torch.float32 or not tacs.is_contiguous() or tacs.dim() != 2:
                raise ValueError("tacs must be a contiguous 2-D float32 tensor")
            J = int(tacs.shape[0])
            prob = torch.empty((J, self.M), dtype=torch.float32, device=tacs.device)
            pref = torch.empty(J, dtype=torch.int32, device=tacs.device)
            self._check(self._lib.abc_model_select(self._h, C.c_void_p(tacs.data_ptr()) if J else None, J,
                                                   A.PTR_TACS_DEVICE | A.PTR_OUT_DEVICE, C.c_void_p(prob.data_ptr()),
                                                   C.c_void_p(pref.data_ptr())))
            return {"prob": prob, "preferred": pref}
        y = np.ascontiguousarray(tacs, dtype=np.float32)
        J = y.shape[0]
        prob = np.empty((J, self.M), dtype=np.float32)
        pref = np.empty(J, dtype=np.int32)
        self._check(self._lib.abc_model_select(self._h, A.host_ptr(y) if J else None, J, 0, prob.ctypes.data,
                                               pref.ctypes.data))
        return {"prob": prob, "preferred": pref}

    def patlak(self, tacs, t_star):
        """(K_i, intercept) per voxel: least-squares Patlak line over the frames with mid-time >=
        t_star (abc_patlak).  numpy host arrays, or a torch CUDA tensor (device outputs)."""
        if type(tacs).__module__.startswith("torch") and tacs.is_cuda:
            import torch
            J = int(tacs.shape[0])
            ki = torch.empty(J, dtype=torch.float32, device=tacs.device)
            v0 = torch.empty(J, dtype=torch.float32, device=tacs.device)
            self._check(self._lib.abc_patlak(self._h, C.c_void_p(tacs.data_ptr()), J, float(t_star),
                                             A.PTR_TACS_DEVICE | A.PTR_OUT_DEVICE, C.c_void_p(ki.data_ptr()),
                                             C.c_void_p(v0.data_ptr())))
            return ki, v0
        y = np.ascontiguousarray(tacs, dtype=np.float32)
        J = y.shape[0]
        ki = np.zeros(J, dtype=np.float32)
        v0 = np.zeros(J, dtype=np.float32)
        self._check(self._lib.abc_patlak(self._h, y.ctypes.data, J, float(t_star), 0, ki.ctypes.data, v0.ctypes.data))
        return ki, v0

    def set_sim_noise(self, ell, half_life_min=float("inf")):
        """Gaussian noise on the simulated draws (P:218-220 model, abc_set_sim_noise); ell = 0: none."""
        self._check(self._lib.abc_set_sim_noise(self._h, float(ell), float(half_life_min)))

    def response_envelope(self, acc_idx, t):
        """J x T x 3 (2.5/50/97.5 %) quantiles of 1 + gamma/k2a g(t) over each voxel's accepted
        lp-ntPET draws (Fig. 1).  acc_idx: J x n uint64 (numpy, or a torch CUDA tensor:
        the result is then a torch CUDA tensor); t: times in minutes."""
        tt = np.ascontiguousarray(t, dtype=np.float64)
        T = int(tt.size)
        if type(acc_idx).__module__.startswith("torch") and acc_idx.is_cuda:
            import torch
            idx = acc_idx.to(torch.int64).contiguous()
            J, n = int(idx.shape[0]), int(idx.shape[1])
            out = torch.empty((J, T, 3), dtype=torch.float32, device=idx.device)
            self._check(self._lib.abc_response_envelope(self._h, C.c_void_p(idx.data_ptr()), J, n, tt.ctypes.data, T,
                                                        A.PTR_TACS_DEVICE | A.PTR_OUT_DEVICE,
                                                        C.c_void_p(out.data_ptr())))
            return out
        idx = np.ascontiguousarray(acc_idx, dtype=np.uint64)
        J, n = idx.shape
        out = np.zeros((J, T, 3), dtype=np.float32)
        self._check(self._lib.abc_response_envelope(self._h, idx.ctypes.data, J, n, tt.ctypes.data, T, 0,
                                                    out.ctypes.data))
        return out
