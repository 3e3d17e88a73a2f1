"""Tightness study of tile lower bounds (analysis tool, runs on the GPU box with torch).

For a sample of config-4 voxels and the bank of N draws (taken from the product via
AbcContext.bank()), order the prescaled bank like order.cu (Morton code of the 4-PC projection),
cut it into tiles, and count per voxel the tiles whose lower bound is below the final
threshold tau_j (the n-th smallest D) for
  * the per-frame box bound used by the scan (sum_f dist(y_f, [lo_f, hi_f])^2),
  * a principal-subspace box bound: sum_k dist(p_k(y), [lo_k, hi_k])^2 + dist(r_y, [r_lo, r_hi])^2
    with p = projection on the top-K principal axes and r = norm of the residual,
  * the max of the two.
python tools/bound_study.py [--N 1000000] [--voxels 256] [--tile 32]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2603_14859_b200 import AbcContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1_000_000)
ap.add_argument("--voxels", type=int, default=256)
ap.add_argument("--tile", type=int, default=32)
ap.add_argument("--n", type=int, default=18)
a = ap.parse_args()
dev = "cuda"
p = S.config4_chunk(chunk=0, n_chunks=32, N=a.N, n=a.n, device=dev)
sel = np.linspace(0, p.J - 1, a.voxels).astype(np.int64)
ctx = AbcContext(**p.ctx_kwargs)
p.setup(ctx)
r = ctx.run_voxels(p.tacs[sel])
tau = torch.as_tensor(r["acc_dist"][:, -1].astype(np.float64), device=dev)
bank = torch.as_tensor(ctx.bank(), device=dev, dtype=torch.float64)[:, :p.L]
w = torch.as_tensor(p.weight.astype(np.float64), device=dev)
sw = w.sqrt()
X = bank * sw
Y = torch.as_tensor(p.tacs[sel].astype(np.float64), device=dev) * sw
mu = X.mean(0)
Xc = X - mu
cov = Xc.T @ Xc / X.shape[0]
ev, V = torch.linalg.eigh(cov)
V = V.flip(1)
ev = ev.flip(0)
print("explained variance (first 8):", (ev[:8] / ev.sum()).cpu().numpy().round(5))
P4 = Xc @ V[:, :4]
lo4 = P4.min(0).values
q = ((P4 - lo4) * (32767.0 / (P4.max(0).values - lo4).max())).clamp(0, 32767).long()


def spread4(v):
    out = torch.zeros_like(v)
    for b in range(15):
        out |= ((v >> b) & 1) << (4 * b)
    return out


key = sum(spread4(q[:, c]) << c for c in range(4))
order = torch.argsort(key)
Xo = X[order]
T = a.tile
nt = Xo.shape[0] // T
Xt = Xo[: nt * T].view(nt, T, -1)
lo, hi = Xt.min(1).values, Xt.max(1).values  # [nt, L]


def frame_box(yv):
    d = torch.clamp(torch.maximum(lo - yv, yv - hi), min=0)
    return (d * d).sum(1)


res = {}
for K in (4, 8, 12, 16):
    Pk = (Xo[: nt * T] - mu) @ V[:, :K]
    rs = ((Xo[: nt * T] - mu) - Pk @ V[:, :K].T).norm(dim=1)
    Pt = Pk.view(nt, T, K)
    plo, phi = Pt.min(1).values, Pt.max(1).values
    rt = rs.view(nt, T)
    rlo, rhi = rt.min(1).values, rt.max(1).values
    cnt_f, cnt_p, cnt_b, cnt_pair = [], [], [], []
    for j in range(len(sel)):
        yv = Y[j]
        bf = frame_box(yv)
        py = (yv - mu) @ V[:, :K]
        ry = ((yv - mu) - py @ V[:, :K].T).norm()
        d = torch.clamp(torch.maximum(plo - py, py - phi), min=0)
        dr = torch.clamp(torch.maximum(rlo - ry, ry - rhi), min=0)
        bp = (d * d).sum(1) + dr * dr
        cnt_f.append(int((bf < tau[j]).sum()))
        cnt_p.append(int((bp < tau[j]).sum()))
        cnt_b.append(int((torch.maximum(bf, bp) < tau[j]).sum()))
        # exact: draws with D < tau (lower limit of any method)
        if K == 4:
            D = ((Xo - yv) ** 2).sum(1)
            cnt_pair.append(int((D <= tau[j]).sum()))
    res[K] = (np.mean(cnt_f), np.mean(cnt_p), np.mean(cnt_b))
    print(f"K={K:2d}: tiles alive at final tau per voxel: frame box {res[K][0]:.1f}  subspace box {res[K][1]:.1f}  "
          f"max {res[K][2]:.1f}  (of {nt})", flush=True)
    if K == 4:
        print(f"draws with D <= tau per voxel: {np.mean(cnt_pair):.1f}")
