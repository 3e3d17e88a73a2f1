"""Per-tissue-class cost of the FP32 pass: runs 10 CTAs worth of voxels of each class."""
import pickle
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_14859_b200 import AbcContext  # noqa: E402
from synthetic.problems import TB_CLASSES  # noqa: E402

p = pickle.load(open(sys.argv[1], "rb"))
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lab = p.truth["label"]
for c, (name, _) in TB_CLASSES.items():
    idx = np.flatnonzero(lab == c)[:5120]
    if len(idx) == 0:
        continue
    sub = p.subset(idx)
    ctx = AbcContext(**dict(sub.ctx_kwargs, flags=1 | 4 | flags))
    sub.setup(ctx)
    ctx.run_voxels(sub.tacs)
    ctx.run_voxels(sub.tacs)
    s = ctx.stats()
    y = sub.tacs
    print(f"{name:11s} J={len(idx):5d} scan {s['ms_scan']:8.1f} ms  frame_upd/vox {s['frame_updates'] / len(idx):.3e} "
          f"bound_upd/vox {s['bound_updates'] / len(idx):.3e}  mean late TAC {y[:, -5:].mean():.0f}", flush=True)
