"""Config 2 (BASELINE.json configs[1]): lp-ntPET vs MRTM model selection, 1e4 noisy TACs, 61 x 60 s
frames, 1e5 draws per model, at three noise levels.  Reports the step time of the hot path and the
detection rates (activated TACs with P(lp-ntPET) > 0.5, null TACs with P(MRTM) >= 0.5) -- the
quantities of Table II on this synthetic population (qualitative comparison only).

python tools/run_config2.py [--n 100] [--J 10000]
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
ap.add_argument("--J", type=int, default=10_000)
ap.add_argument("--n", type=int, default=100)
ap.add_argument("--per-model", type=int, default=100_000)
a = ap.parse_args()
out = {}
for noise in ("low", "mid", "high"):
    t0 = time.time()
    p = S.config2(J=a.J, N_per_model=a.per_model, n=a.n, noise=noise, device="cuda")
    gen = time.time() - t0
    ctx = AbcContext(**dict(p.ctx_kwargs, flags=FLAG_TIMING))
    p.setup(ctx)
    ctx.run_voxels(p.tacs)
    r = ctx.run_voxels(p.tacs)
    st = ctx.stats()
    act = p.truth["active"]
    p_lp = r["prob"][:, 1]
    sens = float(np.mean(p_lp[act] > 0.5))
    spec = float(np.mean(p_lp[~act] <= 0.5))
    out[noise] = {"sensitivity": sens, "specificity": spec, "ms_total": st["ms_total"], "ms_bank": st["ms_bank"],
                  "ms_scan": st["ms_scan"], "ms_certify": st["ms_certify"], "n_fallback": st["n_fallback"],
                  "pairs_per_s": p.J * ctx.N / (st["ms_total"] / 1e3), "gen_s": gen}
    print(noise, json.dumps(out[noise]), flush=True)
print(json.dumps({"config2": out, "J": a.J, "N": 2 * a.per_model, "n": a.n}))
