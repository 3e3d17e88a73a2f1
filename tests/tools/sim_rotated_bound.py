"""Offline estimate (CPU, numpy): row work of the FP32 scan with boxes in the frame basis (the
current kernel) vs boxes in a PCA-rotated basis with a per-tile tail bound for early row exit.

Both schemes use the final per-voxel threshold tau_v (the K-th smallest D, exact) for every
decision, tiles of 32 rows in a Morton order of the first 4 principal projections, and warps of
64 voxels consecutive in a Morton order of the voxels' first 3 principal projections.  Counts per
voxel: row coordinate updates (a warp evaluates a tile's rows for all its voxels once the tile is
alive for one) and tile-bound coordinate updates.

python tests/tools/sim_rotated_bound.py [--draws 1000000] [--warps 8] [--head 8]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import synthetic as S  # noqa: E402
from oracle import oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--draws", type=int, default=1_000_000)
ap.add_argument("--warps", type=int, default=8)
ap.add_argument("--head", type=int, nargs="+", default=[4, 8, 12])
ap.add_argument("--K", type=int, default=22)
ap.add_argument("--pool", type=int, default=20000, help="voxels sampled to form the voxel order")
a = ap.parse_args()

T = 32
p = S.config4_chunk(chunk=0, n_chunks=32, N=a.draws, n=18, max_voxels=a.pool)
ctx = O.OracleContext(**p.ctx_kwargs)
p.setup(ctx)
bank = ctx.bank().astype(np.float64)  # (N, L)
N, L = bank.shape
w = np.ones(L) if p.weight is None else np.asarray(p.weight, dtype=np.float64)
sw = np.sqrt(w)
X = bank * sw
Y = p.tacs.astype(np.float64) * sw

# principal axes of the scaled bank
mu = X.mean(0)
C = np.cov((X - mu).T)
ev, U = np.linalg.eigh(C)
U = U[:, ::-1]
ev = ev[::-1]
print("bank variance in the first 4 / 8 / 12 PCs: %.4f %.4f %.4f" % tuple(ev[:k].sum() / ev.sum() for k in (4, 8, 12)))


def morton(P, bits=10):
    q = np.clip(((P - P.min(0)) / (np.ptp(P, 0) + 1e-30) * ((1 << bits) - 1)).astype(np.int64), 0, (1 << bits) - 1)
    key = np.zeros(len(P), dtype=np.int64)
    d = P.shape[1]
    for b in range(bits):
        for j in range(d):
            key |= ((q[:, j] >> b) & 1) << (b * d + j)
    return np.argsort(key, kind="stable")


order = morton((X - mu) @ U[:, :4], bits=12)
X = X[order]
Xr = X @ U  # rotated rows (orthonormal: distances preserved)
nt = N // T
X = X[:nt * T]
Xr = Xr[:nt * T]
# frame basis: frames in descending spread order (as the kernel)
fperm = np.argsort(-X.var(0))
Xf = X[:, fperm]


def boxes(Z):
    Zt = Z.reshape(nt, T, -1)
    return Zt.min(1), Zt.max(1)


flo, fhi = boxes(Xf)
rlo, rhi = boxes(Xr)

# voxel order and warps
vo = morton((Y - mu) @ U[:, :3], bits=10)
rng = np.random.default_rng(5)
starts = rng.choice(len(vo) // 64, a.warps, replace=False) * 64
tot = {"frame": [0.0, 0.0]}
for m in a.head:
    tot[f"rot_h{m}"] = [0.0, 0.0, 0.0]
nvox = 0
for s0 in starts:
    vids = vo[s0:s0 + 64]
    yf = Y[vids][:, fperm]
    yr = Y[vids] @ U
    # exact final thresholds (K-th smallest D)
    D = (yf ** 2).sum(1)[:, None] - 2.0 * yf @ Xf.T + (Xf ** 2).sum(1)[None, :]
    tau = np.partition(D, a.K - 1, axis=1)[:, a.K - 1]
    # frame basis: tile alive for voxel v if box LB < tau
    gap = np.maximum(np.maximum(flo[None] - yf[:, None], yf[:, None] - fhi[None]), 0.0)
    lbf = (gap ** 2).sum(-1)  # (64, nt)
    alive_any = (lbf < tau[:, None]).any(0)
    rows = alive_any.sum() * T * L  # per voxel: every row of an alive tile, all L frames
    tot["frame"][0] += rows * 64
    tot["frame"][1] += nt * L * 64  # tile bounds (upper bound: every tile checked)
    gr = np.maximum(np.maximum(rlo[None] - yr[:, None], yr[:, None] - rhi[None]), 0.0) ** 2
    lbr = gr.sum(-1)
    alive_r = (lbr < tau[:, None]).any(0)
    tiles = np.flatnonzero(alive_r)
    Dr_rows = Xr.reshape(nt, T, L)[tiles]  # (na, T, L)
    for m in a.head:
        tail = gr[:, tiles, m:].sum(-1)  # (64, na)
        dh = ((Dr_rows[None, :, :, :m] - yr[:, None, None, :m]) ** 2).sum(-1)  # (64, na, T)
        surv = (dh + tail[:, :, None] < tau[:, None, None]).any(0)  # (na, T) any voxel
        work = len(tiles) * T * m + surv.sum() * (L - m)
        tot[f"rot_h{m}"][0] += work * 64
        tot[f"rot_h{m}"][1] += nt * L * 64
        tot[f"rot_h{m}"][2] += surv.mean() if len(tiles) else 0.0
    nvox += 64
    print(f"warp at {s0}: tau median {np.median(tau):.3g}; frame alive tiles {alive_any.sum()}, rotated {alive_r.sum()}",
          flush=True)
print(f"N = {N}, {nvox} voxels")
for k, v in tot.items():
    extra = f", rows needing the full evaluation {v[2] / len(starts):.3f}" if len(v) > 2 else ""
    print(f"{k:10s}: row coordinate updates per voxel {v[0] / nvox / 1e6:.3f} M{extra}")
