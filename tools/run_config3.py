"""Config 3: the 128 x 128 x 63 brain phantom, whole volume (1,032,192 voxels),
MRTM vs lp-ntPET, 90 x 60 s frames, N = 1e7 draws, n = 100, one B200.  Reports the stage times
of the hot path, the voxel and pair rates, and the activation detection rates (activated
striatum with P(lp-ntPET) > 0.5; non-activated striatum with P(MRTM) >= 0.5) -- the quantities
of Table III on this synthetic phantom (qualitative only).

python tools/run_config3.py [--N 10000000] [--slices 0:63] [--batch 0]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2603_14859_b200 import FLAG_TIMING, AbcContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=10_000_000)
ap.add_argument("--n", type=int, default=100)
ap.add_argument("--slices", default="0:63")
ap.add_argument("--batch", type=int, default=0, help="voxels per abc_run_voxels call (0 = all)")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
z0, z1 = (int(v) for v in a.slices.split(":"))
t0 = time.time()
p = S.config3(slices=range(z0, z1), N=a.N, n=a.n, device="cuda")
gen = time.time() - t0
print(f"generated {p.J} voxels x {p.L} frames in {gen:.1f} s", flush=True)
ctx = AbcContext(**dict(p.ctx_kwargs, flags=FLAG_TIMING))
p.setup(ctx)
B = a.batch or p.J
for rep in range(a.reps):
    t = time.time()
    parts, agg = [], {}
    for s in range(0, p.J, B):
        parts.append(ctx.run_voxels(p.tacs[s:s + B]))
        st = ctx.stats()
        for k in ("ms_total", "ms_bank", "ms_order", "ms_scan", "ms_certify"):
            agg[k] = agg.get(k, 0.0) + st[k]
        agg["n_fallback"] = agg.get("n_fallback", 0) + st["n_fallback"]
    wall = time.time() - t
    print(f"rep {rep}: wall {wall:.2f} s", json.dumps({k: round(v, 2) for k, v in agg.items()}), flush=True)
prob = np.concatenate([r["prob"] for r in parts])
lab = p.truth["label"]
act = lab == 5
stri = lab == 4
out = {"J": p.J, "N": ctx.N, "n": a.n, "L": p.L, "wall_s": wall, **agg,
       "voxels_per_s": p.J / (agg["ms_total"] / 1e3), "pairs_per_s": p.J * ctx.N / (agg["ms_total"] / 1e3),
       "sensitivity_active": float(np.mean(prob[act, 1] > 0.5)) if act.any() else None,
       "specificity_striatum": float(np.mean(prob[stri, 1] <= 0.5)) if stri.any() else None,
       "p_lp_by_class": {S.problems.BRAIN_CLASSES[c][0]: float(np.mean(prob[lab == c, 1])) for c in np.unique(lab)}}
print(json.dumps(out))
