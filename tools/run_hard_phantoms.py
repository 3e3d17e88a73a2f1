"""Does the speed survive harder data?  (VERDICT r01 "what's weak" 10 / "next" 5.)

The pruned FP32 pass is exact for any data, but its SPEED depends on how clusterable the TACs are.
This runs the config-4 setup (N = 1e7, n = 18, L = 35, IRR vs REV) on
  * the 9-class TB phantom (10 % log-normal jitter around class means) and
  * a CONTINUOUS phantom: every kinetic parameter a smooth random field spanning the whole
    eq:prior2 range, half the volume reversible (synthetic.config4_continuous),
each at noise levels ell in {3.5, 7, 14} (the paper's TB study uses ell = 7), on the same
axial slab set, and reports per-stage device times, the executed fraction of the dense J N L frame
updates, the ALU roofline fraction of the scan and the number of uncertified voxels.

python tools/run_hard_phantoms.py [--chunks 16] [--out f.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2603_14859_b200 import FLAG_COUNT_WORK, FLAG_TIMING, AbcContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--chunks", type=int, default=16)
ap.add_argument("--draws", type=int, default=10_000_000)
ap.add_argument("--ells", default="3.5,7,14")
ap.add_argument("--out", default=None)
a = ap.parse_args()
rows = []
for phantom in ("classes", "continuous"):
    for ell in [float(x) for x in a.ells.split(",")]:
        t0 = time.time()
        gen = S.config4_chunk if phantom == "classes" else S.config4_continuous
        p = gen(chunk=0, n_chunks=a.chunks, N=a.draws, n=18, ell=ell, device="cuda")
        gen_s = time.time() - t0
        y = torch.from_numpy(p.tacs).cuda()
        ctx = AbcContext(**dict(p.ctx_kwargs, flags=FLAG_TIMING))
        p.setup(ctx)
        sts = []
        for _ in range(3):
            ctx.run_voxels(y, want=("prob", "ki_mean", "ki_sd"))
            sts.append(ctx.stats())
        st = {k: float(np.median([s[k] for s in sts[1:]])) for k in
              ("ms_total", "ms_bank", "ms_order", "ms_scan", "ms_certify", "ms_fallback")}
        cctx = AbcContext(**dict(p.ctx_kwargs, flags=FLAG_TIMING | FLAG_COUNT_WORK))
        p.setup(cctx)
        cctx.run_voxels(y, want=("prob",))
        cs = cctx.stats()
        J, N, L = p.J, ctx.N, p.L
        ops = 2.0 * cs["frame_updates"] + 4.0 * cs["bound_updates"]
        row = {"phantom": phantom, "ell": ell, "J": J, "N": N, **st, "n_fallback": int(sts[-1]["n_fallback"]),
               "pairs_per_s": J * N / (st["ms_total"] / 1e3), "voxels_per_s": J / (st["ms_total"] / 1e3),
               "executed_fraction_of_dense": cs["frame_updates"] / float(J * N * L),
               "scan_alu_frac": ops / (st["ms_scan"] / 1e3) / (148 * 128 * 1.965e9),
               "projected_whole_volume_s": 4_441_800 / (J / (st["ms_total"] / 1e3)), "gen_s": gen_s}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del ctx, cctx, y
        torch.cuda.empty_cache()
res = json.dumps({"hard_phantoms": rows}, indent=1)
print(res)
if a.out:
    open(a.out, "w").write(res)
