"""Run the bench workload (config-4 batch, N = 1e7) for a few steps -- the command profiled by ncu.

python tools/profile_step.py --save /tmp/p.pkl            # generate inputs once (RK4 phantom on GPU)
python tools/profile_step.py --load /tmp/p.pkl --steps 2  # run (no input generation: ncu-friendly)
"""
import argparse
import os
import pickle
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--max-voxels", type=int, default=None)
ap.add_argument("--draws", type=int, default=10_000_000)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--save", default=None)
ap.add_argument("--chunks", type=int, default=32, help="1 = the whole 4.44M-voxel volume (the bench workload)")
ap.add_argument("--device-tacs", action="store_true", help="TACs resident on the device (as bench.py times)")
ap.add_argument("--load", default=None)
ap.add_argument("--digest", action="store_true", help="print a hash of the output maps (compare variants)")
a = ap.parse_args()
if a.load:
    prob = pickle.load(open(a.load, "rb"))
else:
    import synthetic as S
    prob = S.config4_chunk(chunk=0, n_chunks=a.chunks, N=a.draws, n=18, device="cuda", max_voxels=a.max_voxels)
    prob.truth.pop("clean", None)
    if a.save:
        pickle.dump(prob, open(a.save, "wb"))
        print("saved", a.save, prob.tacs.shape)
        sys.exit(0)
from paper_2603_14859_b200 import FLAG_TIMING, AbcContext  # noqa: E402

ctx = AbcContext(**dict(prob.ctx_kwargs, flags=FLAG_TIMING | a.flags))
prob.setup(ctx)
y = np.ascontiguousarray(prob.tacs)
if a.device_tacs:
    import torch
    y = torch.from_numpy(y).cuda()
for s in range(a.steps):
    t = time.time()
    r = ctx.run_voxels(y, want=("prob", "preferred", "count", "mean", "sd", "q", "ki_mean", "ki_sd", "ki_q"))
    st = ctx.stats()
    print(f"step {s}: {time.time() - t:.3f} s  scan {st['ms_scan']:.1f} ms  order {st['ms_order']:.1f} ms  "
          f"bank {st['ms_bank']:.1f} ms  certify {st['ms_certify']:.2f} ms  fb+reduce {st['ms_fallback']:.2f} ms  "
          f"total {st['ms_total']:.2f} ms  fallback voxels {st['n_fallback']}  "
          f"launches {st['gpu_launches']}" + (f"  frame_updates {st['frame_updates']}  bound_updates {st['bound_updates']}"
                                              if a.flags & 4 else ""), flush=True)
if a.digest:
    import hashlib
    h = hashlib.sha256()
    for k in sorted(r):
        v = r[k]
        h.update((v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)).tobytes())
    print("digest", h.hexdigest()[:16], flush=True)
