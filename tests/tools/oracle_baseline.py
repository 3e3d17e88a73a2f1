"""The CPU oracle at the bench's full draw budget (SURVEY §8(d) "Oracle timing"): a seeded random
voxel subset of the whole TB volume at N = 1e7, the oracle's FP64 bank build timed separately, the
per-voxel time extrapolated to the 4,441,800-voxel volume.  The oracle is test infrastructure and
runs here as it stands (never tuned); this is a reported baseline, not a target.

python tests/tools/oracle_baseline.py [--voxels 1024] [--draws 10000000] [--out f.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

import synthetic as S  # noqa: E402
from oracle import oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--voxels", type=int, default=1024)
ap.add_argument("--draws", type=int, default=10_000_000)
ap.add_argument("--out", default=None)
a = ap.parse_args()
J_total = S.tb_voxel_count()
idx = np.sort(np.random.default_rng(2026).choice(J_total, a.voxels, replace=False))
t = time.perf_counter()
p = S.config4_chunk(chunk=0, n_chunks=1, N=a.draws, n=18, voxel_index=idx)
gen_s = time.perf_counter() - t
ctx = O.OracleContext(**p.ctx_kwargs)
p.setup(ctx)
t = time.perf_counter()
ctx.bank()
bank_s = time.perf_counter() - t
t = time.perf_counter()
ctx.run_voxels(p.tacs)
run_s = time.perf_counter() - t
vox_s = max(run_s - bank_s, 1e-9)  # run_voxels rebuilds the bank
per_voxel = vox_s / p.J
res = {"oracle_baseline": {
    "workload": f"config 4, {p.J} voxels drawn at random (seed 2026) from the 4,441,800-voxel volume, N = {ctx.N}, "
                "n = 18, L = 35, IRR vs REV",
    "threads": O.get_threads(), "bank_s": bank_s, "run_s": run_s, "voxel_loop_s": vox_s,
    "core_s_per_voxel": per_voxel * O.get_threads(), "pairs_per_s": p.J * ctx.N / vox_s,
    "projected_whole_volume_s": bank_s + J_total * per_voxel,
    "projected_whole_volume_h": (bank_s + J_total * per_voxel) / 3600.0, "input_generation_s": gen_s}}
print(json.dumps(res, indent=1))
if a.out:
    open(a.out, "w").write(json.dumps(res, indent=1))
