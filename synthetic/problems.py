"""Seeded synthetic problems shaped like the paper's workloads (BASELINE.json configs).

Ground truth is produced by RK4 integration of the model ODEs on a 1-s grid with
trapezoidal frame averaging -- the physical data-generating process, deliberately a
different numerical route from the method's closed forms.  Recipes: DESIGN.md "Input recipe".
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np
import torch

from .schedules import decay_weights, fdg22, tb35, uniform_frames

# Feng input of the phantoms, (beta1, beta2, beta3, kappa1, kappa2, kappa3); inside the
# P:209-213 ranges (chosen).
FENG_PHANTOM = (1.0e5, 5.0e4, 1.5e4, 10.0, 0.5, 0.02)
T_HALF_F18 = 109.8  # min
T_HALF_C11 = 20.4   # min, textbook (paper silent, R11)
DT = 1.0 / 60.0     # RK4 step of the ground-truth generator (1 s)


def priors_fdg():
    """eq:prior2 P:272-277: K1~U(0.001,1), k2~U(0.001,2), k3~U(0.001,0.5), k4~U(0,0.1),
    Vb~U(0.03,0.2).  Columns [K1, k2, k3, k4, Vb]."""
    return [0.001, 0.001, 0.001, 0.0, 0.03], [1.0, 2.0, 0.5, 0.1, 0.2]


def priors_rt():
    """lp-ntPET / MRTM ABC priors (paper silent; R12): R1~U(0.5,1.5),
    k2~U(0.05,0.6), k2a~U(0.01,0.2), gamma~U(0,0.2), tD~U(15,45), tP-tD~U(1,45),
    alpha~U(0.25,4).  Columns [R1, k2, k2a, gamma, tD, tP(offset drawn), alpha]."""
    return [0.5, 0.05, 0.01, 0.0, 15.0, 1.0, 0.25], [1.5, 0.6, 0.2, 0.2, 45.0, 45.0, 4.0]


@dataclasses.dataclass
class Problem:
    name: str
    ctx_kwargs: dict
    input_kind: str
    input_value: np.ndarray
    input_t: Optional[np.ndarray]
    frame_start: np.ndarray
    frame_dur: np.ndarray
    weight: Optional[np.ndarray]
    tacs: np.ndarray
    truth: dict

    @property
    def J(self) -> int:
        return int(self.tacs.shape[0])

    @property
    def L(self) -> int:
        return int(self.tacs.shape[1])

    def replace(self, tacs=None, **ctx_kwargs) -> "Problem":
        kw = dict(self.ctx_kwargs)
        kw.update(ctx_kwargs)
        return dataclasses.replace(self, ctx_kwargs=kw, tacs=self.tacs if tacs is None else tacs)

    def subset(self, idx) -> "Problem":
        idx = np.asarray(idx)
        truth = {k: (v[idx] if isinstance(v, np.ndarray) and v.shape[:1] == (self.J,) else v)
                 for k, v in self.truth.items()}
        return dataclasses.replace(self, tacs=np.ascontiguousarray(self.tacs[idx]), truth=truth)

    def setup(self, ctx) -> None:
        """Configure an AbcContext / OracleContext with this problem's input and frames."""
        ctx.set_input_function(self.input_kind, self.input_value, t=self.input_t)
        ctx.set_frames(self.frame_start, self.frame_dur, self.weight)


# ----------------------------------------------------------------------------------
# ground-truth generators (RK4, torch float64)
# ----------------------------------------------------------------------------------
def _feng_t(bk, t):
    b1, b2, b3, k1, k2, k3 = bk
    return (b1 * t - b2 - b3) * math.exp(-k1 * t) + b2 * math.exp(-k2 * t) + b3 * math.exp(-k3 * t)


def _grid_frames(start, dur):
    """Segment -> frame map on the DT grid; frame bounds must lie on the grid."""
    tend = float(start[-1] + dur[-1])
    K = int(round(tend / DT))
    seg = -np.ones(K, dtype=np.int64)
    for f, (s, d) in enumerate(zip(start, dur)):
        a, b = int(round(s / DT)), int(round((s + d) / DT))
        assert abs(a * DT - s) < 1e-9 and abs(b * DT - (s + d)) < 1e-9, "frame bounds off the 1-s grid"
        seg[a:b] = f
    return K, seg


def _rk4_frame_means(deriv, state0, out_fn, start, dur, device):
    """Integrate y' = deriv(t, y) by RK4 on the DT grid; return trapezoidal frame means of out_fn."""
    K, seg = _grid_frames(start, dur)
    L = len(start)
    J = state0[0].shape[0]
    acc = torch.zeros(J, L, dtype=torch.float64, device=device)
    y = state0
    t = 0.0
    o_prev = out_fn(t, y)
    h = DT
    for k in range(K):
        k1 = deriv(t, y)
        k2 = deriv(t + h / 2, tuple(a + (h / 2) * b for a, b in zip(y, k1)))
        k3 = deriv(t + h / 2, tuple(a + (h / 2) * b for a, b in zip(y, k2)))
        k4 = deriv(t + h, tuple(a + h * b for a, b in zip(y, k3)))
        y = tuple(a + (h / 6) * (b1 + 2 * b2 + 2 * b3 + b4) for a, b1, b2, b3, b4 in zip(y, k1, k2, k3, k4))
        t = (k + 1) * h
        o = out_fn(t, y)
        f = int(seg[k])
        if f >= 0:
            acc[:, f] += 0.5 * h * (o_prev + o)
        o_prev = o
    return (acc / torch.as_tensor(dur, dtype=torch.float64, device=device)).cpu().numpy()


def truth_2tcm(theta, feng, start, dur, device="cpu"):
    """Frame-mean C_T of eq:2TCM/eq:2TCM_op (C_wb = C_p) for theta [J,5] = K1,k2,k3,k4,Vb."""
    th = torch.as_tensor(np.asarray(theta, dtype=np.float64), device=device)
    K1, k2, k3, k4, Vb = (th[:, i] for i in range(5))

    def deriv(t, y):
        cf, cm = y
        cp = _feng_t(feng, t)
        return (K1 * cp - (k2 + k3) * cf + k4 * cm, k3 * cf - k4 * cm)

    def out(t, y):
        return (1 - Vb) * (y[0] + y[1]) + Vb * _feng_t(feng, t)

    z = torch.zeros_like(K1)
    return _rk4_frame_means(deriv, (z, z.clone()), out, start, dur, device)


def _gamma_t(tD, tP, al, t):
    x = torch.clamp((t - tD) / (tP - tD), min=0.0)
    g = torch.where(x > 0, torch.exp(al * (torch.log(torch.clamp(x, min=1e-300)) + 1.0 - x)), torch.zeros_like(x))
    return g


def truth_rt(theta, feng, ref_k, start, dur, device="cpu"):
    """Frame means of (C_r, C_t): C_r = 1TCM(ref_k) (x) Feng; C_t from the differentiated
    eq:lp-ntPET: C_t' = R1 C_r' + k2 C_r - k2a C_t - gamma g(t) C_t, C_t(0) = R1 C_r(0) = 0.
    theta [J,7] = R1, k2, k2a, gamma, tD, tP, alpha."""
    th = torch.as_tensor(np.asarray(theta, dtype=np.float64), device=device)
    R1, k2, k2a, gam, tD, tP, al = (th[:, i] for i in range(7))
    K1r, k2r = ref_k

    def deriv(t, y):
        cr, ct = y
        cp = _feng_t(feng, t)
        dcr = K1r * cp - k2r * cr
        g = _gamma_t(tD, tP, al, torch.full_like(cr, t))
        return (dcr, R1 * dcr + k2 * cr - k2a * ct - gam * g * ct)

    z = torch.zeros_like(R1)
    ct = _rk4_frame_means(deriv, (z, z.clone()), lambda t, y: y[1], start, dur, device)
    cr = _rk4_frame_means(deriv, (z[:1], z[:1].clone()), lambda t, y: y[0], start, dur, device)[0]
    return cr, ct


def feng_frame_means(feng, start, dur):
    """Frame means of the Feng curve by trapezoid on the DT grid (IDIF generation)."""
    K, seg = _grid_frames(start, dur)
    acc = np.zeros(len(start))
    vals = np.array([_feng_t(feng, k * DT) for k in range(K + 1)])
    for k in range(K):
        if seg[k] >= 0:
            acc[seg[k]] += 0.5 * DT * (vals[k] + vals[k + 1])
    return acc / np.asarray(dur)


def noise_fdg(C, start, dur, ell, half_life, rng):
    """y = C + ell sigma_t N(0,1), sigma_t = sqrt(C e^{-lam t}/dt) e^{lam t} at frame mid."""
    lam = math.log(2.0) / half_life
    mid = np.asarray(start) + 0.5 * np.asarray(dur)
    sig = np.sqrt(np.maximum(C, 0.0) * np.exp(-lam * mid) / dur) * np.exp(lam * mid)
    return C + ell * sig * rng.standard_normal(C.shape)


def noise_fdg_eps(C, start, dur, ell, half_life, eps):
    """noise_fdg with the standard normals `eps` given (same shape as C)."""
    lam = math.log(2.0) / half_life
    mid = np.asarray(start) + 0.5 * np.asarray(dur)
    sig = np.sqrt(np.maximum(C, 0.0) * np.exp(-lam * mid) / dur) * np.exp(lam * mid)
    return C + ell * sig * eps


def noise_rt_gauss(C, start, dur, ell1, half_life, rng):
    """epsilon ~ N(0, ell1 sqrt(C / (dt e^{lam t})))  (Gaussian variant)."""
    lam = math.log(2.0) / half_life
    mid = np.asarray(start) + 0.5 * np.asarray(dur)
    sig = ell1 * np.sqrt(np.maximum(C, 0.0) / (dur * np.exp(lam * mid)))
    return C + sig * rng.standard_normal(C.shape)


def _draw_uniform(rng, lo, hi, J):
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    return lo + (hi - lo) * rng.random((J, len(lo)))


# ----------------------------------------------------------------------------------
# config 1: 64 voxels, irreversible 2TCM FDG, 22 frames / 50 min, 1e4 draws, p = 1 %
# ----------------------------------------------------------------------------------
def config1(J=64, N=10_000, p=0.01, distance="WL2", seed=1001, abc_seed=2026, device="cpu"):
    start, dur = fdg22()
    rng = np.random.default_rng(seed)
    lo, hi = priors_fdg()
    theta = _draw_uniform(rng, lo, hi, J)
    theta[:, 3] = 0.0  # irreversible truth
    C = truth_2tcm(theta, FENG_PHANTOM, start, dur, device)
    y = noise_fdg(C, start, dur, 7.0, T_HALF_F18, rng).astype(np.float32)
    n = int(math.floor(N * p + 1e-9))  # n = floor(N p)
    kw = dict(models=[dict(kind="2TCM_IRR", n_draws=N, lo=lo, hi=hi)], seed=abc_seed, distance=distance,
              accept="TOPN", n_accept=n)
    return Problem("config1", kw, "FENG", np.array(FENG_PHANTOM, dtype=np.float64), None, start, dur,
                   decay_weights(start, dur, T_HALF_F18), y, dict(theta=theta, clean=C))


# ----------------------------------------------------------------------------------
# config 2: lp-ntPET vs MRTM model selection, 61 x 60 s, 1e5 draws per model
# ----------------------------------------------------------------------------------
NOISE_CV = {"low": 0.02, "mid": 0.05, "high": 0.10}


def config2(J=10_000, N_per_model=100_000, n=100, noise="mid", seed=1002, abc_seed=2026, device="cpu",
            distance="WL2", lpnt_step_min=0.05, n_frames=61):
    start, dur = uniform_frames(n_frames, 60.0)
    rng = np.random.default_rng(seed)
    half = J // 2
    R1 = rng.uniform(0.8, 1.2, J)
    k2 = rng.uniform(0.2, 0.5, J)
    bp = rng.uniform(1.5, 3.5, J)
    k2a = k2 / (1.0 + bp)
    act = np.zeros(J, dtype=bool)
    act[:half] = True
    mag = np.where(rng.random(J) < 0.5, 0.15, 0.35) * np.exp(0.1 * rng.standard_normal(J))
    gam = np.where(act, mag * k2a, 0.0)
    tD = rng.uniform(30.0, 40.0, J)
    early = rng.random(J) < 0.5
    tP = np.where(early, rng.uniform(0.0, 1.0, J) * (45.0 - (tD + 2.0)) + tD + 2.0, rng.uniform(45.0, 60.0, J))
    al = np.clip(rng.normal(0.7, 0.1, J), 0.3, None)
    theta = np.stack([R1, k2, k2a, gam, tD, tP, al], axis=1)
    cr, C = truth_rt(theta, FENG_PHANTOM, (0.1, 0.3), start, dur, device)
    lam = math.log(2.0) / T_HALF_C11
    mid = start + 0.5 * dur
    late = slice(-10, None)
    cref = float(np.mean(C[:, late]))
    ell1 = NOISE_CV[noise] * math.sqrt(cref * 1.0 * math.exp(lam * float(np.mean(mid[late]))))
    y = noise_rt_gauss(C, start, dur, ell1, T_HALF_C11, rng).astype(np.float32)
    lo, hi = priors_rt()
    kw = dict(models=[dict(kind="MRTM", n_draws=N_per_model, lo=lo, hi=hi),
                      dict(kind="LPNTPET", n_draws=N_per_model, lo=lo, hi=hi)],
              seed=abc_seed, distance=distance, accept="TOPN", n_accept=n, lpnt_step_min=lpnt_step_min)
    kt = np.concatenate([[0.0], mid])
    kv = np.concatenate([[0.0], cr])
    return Problem("config2", kw, "PWL", kv, kt, start, dur, decay_weights(start, dur, T_HALF_C11), y,
                   dict(theta=theta, active=act, clean=C, ref=cr, ell1=ell1))


# ----------------------------------------------------------------------------------
# config 4: total-body FDG phantom 192 x 192 x 673, elliptic-cylinder body mask
# ----------------------------------------------------------------------------------
TB_SHAPE = (673, 192, 192)  # (z, y, x)
TB_CLASSES = {  # class: (K1, k2, k3, k4, Vb) means (FDG-like, inside eq:prior2 ranges)
    0: ("soft", (0.05, 0.30, 0.03, 0.000, 0.04)),
    1: ("brain", (0.10, 0.15, 0.08, 0.005, 0.05)),
    2: ("myocardium", (0.60, 1.20, 0.15, 0.000, 0.15)),
    3: ("liver", (0.80, 1.00, 0.01, 0.010, 0.15)),
    4: ("tumour", (0.30, 0.40, 0.15, 0.000, 0.05)),
    5: ("kidney", (0.70, 1.50, 0.02, 0.030, 0.18)),
    6: ("muscle", (0.03, 0.20, 0.02, 0.000, 0.03)),
    7: ("lung", (0.02, 0.30, 0.01, 0.000, 0.15)),
    8: ("marrow", (0.15, 0.60, 0.10, 0.000, 0.06)),
}


def tb_geometry(z):
    """In-mask voxels of axial slice z: (flat index within the slice [n], class label [n])."""
    nz, ny, nx = TB_SHAPE
    cx, cy = (nx - 1) / 2.0, (ny - 1) / 2.0
    yy, xx = np.mgrid[0:ny, 0:nx]
    dx, dy = xx - cx, yy - cy
    body = (dx / 60.0) ** 2 + (dy / 35.0) ** 2 <= 1.0
    rad = np.sqrt((dx / 60.0) ** 2 + (dy / 35.0) ** 2)
    zeta = (z + 0.5) / nz
    lab = np.zeros((ny, nx), dtype=np.int32)
    lab[rad > 0.85] = 6

    def ell(x0, y0, ax, ay):
        return ((xx - x0) / ax) ** 2 + ((yy - y0) / ay) ** 2 <= 1.0

    if zeta >= 0.88:
        lab[ell(cx, cy, 28, 24)] = 1
    elif 0.70 <= zeta < 0.86:
        lab[ell(cx - 28, cy, 20, 22) | ell(cx + 28, cy, 20, 22)] = 7
        lab[ell(cx - 8, cy + 4, 12, 10)] = 2
        lab[ell(cx, cy + 26, 6, 6)] = 8
    elif 0.56 <= zeta < 0.70:
        lab[ell(cx - 25, cy, 28, 22)] = 3
        if zeta < 0.64:
            lab[ell(cx - 30, cy + 18, 8, 6) | ell(cx + 30, cy + 18, 8, 6)] = 5
        lab[ell(cx, cy + 26, 6, 6)] = 8
        zt = 0.63 * nz
        tum = (xx - (cx - 30)) ** 2 + (yy - (cy - 5)) ** 2 + (z - zt) ** 2 <= 36.0
        lab[tum] = 4
    elif zeta < 0.45:
        lab[ell(cx - 25, cy, 5, 5) | ell(cx + 25, cy, 5, 5)] = 8
    elif zeta < 0.56:
        lab[ell(cx, cy + 26, 6, 6)] = 8
    flat = np.flatnonzero(body.ravel())
    return flat, lab.ravel()[flat]


def tb_voxel_count():
    return sum(len(tb_geometry(z)[0]) for z in range(TB_SHAPE[0]))


def config4_chunk(chunk=0, n_chunks=32, N=10_000_000, n=18, seed=1004, abc_seed=2026, device="cpu",
                  max_voxels=None, distance="WL2", voxel_index=None, ell=7.0):
    """Axial slices z = chunk, chunk + n_chunks, ... of the TB phantom (raster order within each
    slice; n_chunks = 1 is the whole 4,441,800-voxel volume).  IDIF = frame means of the Feng
    curve + 2 % noise as PWL knots.  voxel_index selects voxels of the chunk (e.g. a
    stratified sample) before the ground truth is integrated; the TACs of a voxel do not depend on
    which other voxels are generated."""
    start, dur = tb35()
    lo, hi = priors_fdg()
    feng = FENG_PHANTOM
    thetas, labels, zs = [], [], []
    for z in range(chunk, TB_SHAPE[0], n_chunks):
        flat, lab = tb_geometry(z)
        rng = np.random.default_rng([seed, z])
        base = np.array([TB_CLASSES[c][1] for c in lab], dtype=np.float64)
        jit = np.exp(0.1 * rng.standard_normal(base.shape))
        th = np.clip(base * jit, np.array(lo) + 1e-6, np.array(hi) - 1e-6)
        th[:, 3] = np.where(base[:, 3] > 0, th[:, 3], 0.0)
        thetas.append(th)
        labels.append(lab)
        zs.append(np.full(len(lab), z, dtype=np.int32))
    theta = np.concatenate(thetas)
    lab = np.concatenate(labels)
    zz = np.concatenate(zs)
    pos = np.concatenate([np.arange(len(t)) for t in thetas])  # position within the slice
    if max_voxels is not None:
        theta, lab, zz, pos = theta[:max_voxels], lab[:max_voxels], zz[:max_voxels], pos[:max_voxels]
    if voxel_index is not None:
        vi = np.asarray(voxel_index)
        theta, lab, zz, pos = theta[vi], lab[vi], zz[vi], pos[vi]
    C = truth_2tcm(theta, feng, start, dur, device)
    y = np.empty(C.shape, dtype=np.float32)
    order = np.argsort(zz, kind="stable")
    zs_sorted = zz[order]
    for z in np.unique(zz):
        a, b = np.searchsorted(zs_sorted, [z, z + 1])
        sel = order[a:b]
        rng = np.random.default_rng([seed, int(z), 1])
        nz = len(tb_geometry(int(z))[0])
        eps = rng.standard_normal((nz, C.shape[1]))[pos[sel]]  # the slice's noise field, same for any subset
        y[sel] = noise_fdg_eps(C[sel], start, dur, ell, T_HALF_F18, eps)
    idif_rng = np.random.default_rng([seed, 999_999])
    fm = feng_frame_means(feng, start, dur)
    fm = fm * (1.0 + 0.02 * idif_rng.standard_normal(fm.shape))
    mid = start + 0.5 * dur
    kt = np.concatenate([[0.0], mid])
    kv = np.concatenate([[0.0], fm])
    half = N // 2
    kw = dict(models=[dict(kind="2TCM_IRR", n_draws=half, lo=lo, hi=hi),
                      dict(kind="2TCM_REV", n_draws=N - half, lo=lo, hi=hi)],
              seed=abc_seed, distance=distance, accept="TOPN", n_accept=n)
    return Problem(f"config4_chunk{chunk}of{n_chunks}", kw, "PWL", kv, kt, start, dur,
                   decay_weights(start, dur, T_HALF_F18), y, dict(theta=theta, label=lab, z=zz, clean=C))


def _smooth_field(rng, pts, n_waves=12, scale=0.04):
    """A smooth random field on points pts [n, 3] (voxel coordinates): sum of random low-frequency
    3-D cosines with random phases (mean 0, variance n_waves / 2), standardised analytically (so a
    voxel's value does not depend on which other voxels are generated), mapped to (0, 1) by the
    normal CDF (every value of the range occurs, near-uniform marginals)."""
    f = np.zeros(len(pts))
    for _ in range(n_waves):
        k = rng.normal(0.0, scale, 3)
        f += np.cos(pts @ k + rng.uniform(0, 2 * np.pi))
    f = f / math.sqrt(n_waves / 2.0)
    return 0.5 * (1.0 + np.vectorize(math.erf)(f / math.sqrt(2.0)))


def config4_continuous(chunk=0, n_chunks=32, N=10_000_000, n=18, ell=7.0, seed=1014, abc_seed=2026, device="cpu",
                       max_voxels=None, voxel_index=None, distance="WL2"):
    """Harder variant of config 4 (VERDICT r01 "what's weak" 10): the same body mask, frames, IDIF and
    noise model, but the kinetic parameters are CONTINUOUS smooth random fields spanning the whole
    eq:prior2 ranges instead of 9 tissue classes -- no clustering for the pruned scan to
    exploit -- and half the volume (a smooth region) reversible (k4 > 0).  ell = noise level of P:220."""
    start, dur = tb35()
    lo, hi = priors_fdg()
    feng = FENG_PHANTOM
    zs = list(range(chunk, TB_SHAPE[0], n_chunks))
    pts = []
    for z in zs:
        flat, _ = tb_geometry(z)
        yy, xx = np.divmod(flat, TB_SHAPE[2])
        pts.append(np.stack([xx, yy, np.full(len(flat), z)], axis=1).astype(np.float64))
    pts = np.concatenate(pts)
    zz = pts[:, 2].astype(np.int32)
    pos = np.concatenate([np.arange(np.sum(zz == z)) for z in zs])
    rng = np.random.default_rng([seed, 0])
    theta = np.empty((len(pts), 5))
    for k in range(5):
        u = _smooth_field(rng, pts)
        theta[:, k] = lo[k] + (hi[k] - lo[k]) * np.clip(u, 1e-6, 1 - 1e-6)
    rev = _smooth_field(rng, pts) > 0.5
    theta[~rev, 3] = 0.0
    if max_voxels is not None:
        theta, zz, pos, rev = theta[:max_voxels], zz[:max_voxels], pos[:max_voxels], rev[:max_voxels]
    if voxel_index is not None:
        vi = np.asarray(voxel_index)
        theta, zz, pos, rev = theta[vi], zz[vi], pos[vi], rev[vi]
    C = truth_2tcm(theta, feng, start, dur, device)
    y = np.empty(C.shape, dtype=np.float32)
    order = np.argsort(zz, kind="stable")
    zs_sorted = zz[order]
    for z in np.unique(zz):
        a, b = np.searchsorted(zs_sorted, [z, z + 1])
        sel = order[a:b]
        nz = len(tb_geometry(int(z))[0])
        eps = np.random.default_rng([seed, int(z), 1]).standard_normal((nz, C.shape[1]))[pos[sel]]
        y[sel] = noise_fdg_eps(C[sel], start, dur, ell, T_HALF_F18, eps)
    idif_rng = np.random.default_rng([1004, 999_999])  # the config-4 IDIF
    fm = feng_frame_means(feng, start, dur)
    fm = fm * (1.0 + 0.02 * idif_rng.standard_normal(fm.shape))
    mid = start + 0.5 * dur
    kt = np.concatenate([[0.0], mid])
    kv = np.concatenate([[0.0], fm])
    half = N // 2
    kw = dict(models=[dict(kind="2TCM_IRR", n_draws=half, lo=lo, hi=hi),
                      dict(kind="2TCM_REV", n_draws=N - half, lo=lo, hi=hi)],
              seed=abc_seed, distance=distance, accept="TOPN", n_accept=n)
    return Problem(f"config4c_chunk{chunk}of{n_chunks}_ell{ell}", kw, "PWL", kv, kt, start, dur,
                   decay_weights(start, dur, T_HALF_F18), y, dict(theta=theta, reversible=rev, z=zz, clean=C))


# ----------------------------------------------------------------------------------
# config 3: brain phantom 128 x 128 x 63, whole volume, MRTM vs lp-ntPET, 90 x 60 s
# ----------------------------------------------------------------------------------
BRAIN_SHAPE = (63, 128, 128)  # (z, y, x)
# class: (R1, k2, BP) means; k2a = k2 / (1 + BP) (MRTM kinetics, eq:lp-ntPET with gamma = 0)
BRAIN_CLASSES = {
    0: ("outside", (0.05, 0.05, 0.0)),
    1: ("white", (0.70, 0.20, 0.5)),
    2: ("grey", (1.00, 0.30, 1.0)),
    3: ("cerebellum", (1.00, 0.18, 0.0)),
    4: ("striatum", (1.00, 0.35, 3.0)),
    5: ("striatum_active", (1.00, 0.35, 3.0)),
}


def brain_geometry(z):
    """Class label of every voxel of axial slice z (raster order, 128 x 128)."""
    nz, ny, nx = BRAIN_SHAPE
    cz, cy, cx = (nz - 1) / 2.0, (ny - 1) / 2.0, (nx - 1) / 2.0
    yy, xx = np.mgrid[0:ny, 0:nx].astype(np.float64)

    def ell(x0, y0, z0, ax, ay, az):
        return ((xx - x0) / ax) ** 2 + ((yy - y0) / ay) ** 2 + ((z - z0) / az) ** 2 <= 1.0

    lab = np.zeros((ny, nx), dtype=np.int32)
    rb = np.sqrt(((xx - cx) / 50.0) ** 2 + ((yy - cy) / 57.0) ** 2 + ((z - cz - 4) / 27.0) ** 2)
    brain = rb <= 1.0
    lab[brain] = 1
    lab[brain & (rb > 0.85)] = 2
    lab[ell(cx, cy + 38, 10, 30, 16, 9)] = 3  # cerebellum: posterior, inferior
    for side in (-1, 1):  # caudate (x0 +-12) and putamen (x0 +-24) ellipsoids
        lab[ell(cx + side * 12, cy - 14, cz + 6, 5, 9, 7)] = 4
        lab[ell(cx + side * 24, cy - 4, cz + 2, 6, 12, 8)] = 4
    # activated sub-region: dorsal half of the left putamen and left caudate head
    act = (ell(cx - 24, cy - 4, cz + 2, 6, 12, 8) & (yy < cy - 4)) | (ell(cx - 12, cy - 14, cz + 6, 5, 9, 7) & (yy < cy - 16))
    lab[act] = 5
    return lab.ravel()


def config3(slices=None, N=10_000_000, n=100, noise="mid", seed=1003, abc_seed=2026, device="cpu",
            max_voxels=None, voxel_index=None, distance="WL2", lpnt_step_min=0.05):
    """Brain phantom: every voxel of the 128 x 128 x 63 volume (or of
    `slices`), striatal ellipsoids with an activated sub-region (gamma > 0, onset and peak per
    the config-2 recipe, region-wide with voxel jitter), cerebellar reference region,
    reference TAC = 1TCM(0.1, 0.3) (x) Feng, 90 x 60 s frames, Gaussian noise of
    P:229 at the config-2 level `noise`; N = 1e7 draws split between MRTM and lp-ntPET, n = 100."""
    start, dur = uniform_frames(90, 60.0)
    zs = range(BRAIN_SHAPE[0]) if slices is None else slices
    labs, zz = [], []
    for z in zs:
        lab = brain_geometry(z)
        labs.append(lab)
        zz.append(np.full(lab.shape, z, dtype=np.int32))
    lab = np.concatenate(labs)
    zz = np.concatenate(zz)
    flat = np.concatenate([np.arange(BRAIN_SHAPE[1] * BRAIN_SHAPE[2]) for _ in zs])
    if voxel_index is not None:
        lab, zz, flat = lab[voxel_index], zz[voxel_index], flat[voxel_index]
    if max_voxels is not None:
        lab, zz, flat = lab[:max_voxels], zz[:max_voxels], flat[:max_voxels]
    J = len(lab)
    rng = np.random.default_rng([seed, 0])
    region = np.random.default_rng([seed, 1])  # region-wide activation timing
    tD0 = region.uniform(30.0, 40.0)
    tP0 = region.uniform(tD0 + 2.0, 45.0)
    al0 = float(np.clip(region.normal(0.7, 0.1), 0.3, None))
    base = np.array([BRAIN_CLASSES[c][1] for c in range(len(BRAIN_CLASSES))], dtype=np.float64)[lab]
    jit = np.exp(0.1 * rng.standard_normal((J, 3)))
    R1 = base[:, 0] * jit[:, 0]
    k2 = base[:, 1] * jit[:, 1]
    bp = base[:, 2] * jit[:, 2]
    k2a = k2 / (1.0 + bp)
    active = lab == 5
    gam = np.where(active, 0.35 * k2a * np.exp(0.1 * rng.standard_normal(J)), 0.0)
    tD = tD0 + 0.5 * rng.standard_normal(J)
    tP = np.maximum(tP0 + 0.5 * rng.standard_normal(J), tD + 1.0)
    al = np.clip(al0 + 0.02 * rng.standard_normal(J), 0.3, None)
    theta = np.stack([R1, k2, k2a, gam, tD, tP, al], axis=1)
    cr, C = truth_rt(theta, FENG_PHANTOM, (0.1, 0.3), start, dur, device)
    lam = math.log(2.0) / T_HALF_C11
    mid = start + 0.5 * dur
    late = slice(-10, None)
    ref_mask = lab == 3
    cref = float(np.mean(C[ref_mask][:, late])) if ref_mask.any() else float(np.mean(cr[late]))
    ell1 = NOISE_CV[noise] * math.sqrt(cref * 1.0 * math.exp(lam * float(np.mean(mid[late]))))
    y = noise_rt_gauss(C, start, dur, ell1, T_HALF_C11, rng).astype(np.float32)
    lo, hi = priors_rt()
    half = N // 2
    kw = dict(models=[dict(kind="MRTM", n_draws=half, lo=lo, hi=hi),
                      dict(kind="LPNTPET", n_draws=N - half, lo=lo, hi=hi)],
              seed=abc_seed, distance=distance, accept="TOPN", n_accept=n, lpnt_step_min=lpnt_step_min)
    kt = np.concatenate([[0.0], mid])
    kv = np.concatenate([[0.0], cr])
    return Problem("config3", kw, "PWL", kv, kt, start, dur, decay_weights(start, dur, T_HALF_C11), y,
                   dict(theta=theta, active=active, label=lab, z=zz, flat=flat, clean=C, ref=cr, ell1=ell1))
