"""Config 5 (BASELINE.json configs[4]): scaling sweep over prior draws N x acceptance quantile p on a
J = 2^17 subset of the config-4 TB phantom, default bound-pruned FP32 path vs the dense shared-bank
tensor-core distance (ABC_FLAG_DENSE_TC).  Both give the same certified results (checked here on
the accepted-index arrays); the sweep reports per-stage device times (CUDA events, median of
--reps warm runs) and the pairs/s of each mode.

python tools/run_config5.py [--J 131072] [--draws 10000,100000,1000000] [--p 0.001,0.01]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2603_14859_b200 import FLAG_DENSE_TC, FLAG_TIMING, AbcContext, AbcError  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--J", type=int, default=1 << 17)
ap.add_argument("--draws", default="10000,100000,1000000")
ap.add_argument("--p", default="0.001,0.01")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--modes", default="fp32,dense")
ap.add_argument("--out", default=None)
a = ap.parse_args()

base = S.config4_chunk(chunk=0, n_chunks=32, N=10_000, n=18, max_voxels=a.J, device="cuda")
rows = []
for N in [int(x) for x in a.draws.split(",")]:
    for p in [float(x) for x in a.p.split(",")]:
        n = int(np.floor(N * p))
        if n < 1 or n > 15360:
            continue
        models = [dict(m, n_draws=N // 2) for m in base.ctx_kwargs["models"]]
        prob = base.replace(models=models, n_accept=n)
        ref = None
        for mode in a.modes.split(","):
            flags = FLAG_TIMING | (FLAG_DENSE_TC if mode == "dense" else 0)
            ctx = AbcContext(**dict(prob.ctx_kwargs, flags=flags))
            prob.setup(ctx)
            sts, res = [], None
            try:
                for _ in range(max(1, a.reps) + 1):
                    res = ctx.run_voxels(prob.tacs, want=("acc_idx", "prob"))
                    sts.append(ctx.stats())
            except AbcError as e:  # e.g. the dense mode's candidate band exceeds its capacity at large n
                row = {"N": N, "p": p, "n": n, "J": prob.J, "mode": mode, "unsupported": str(e)}
                rows.append(row)
                print(json.dumps(row), flush=True)
                ctx.close()
                continue
            sts = sts[1:]
            med = {k: float(np.median([s[k] for s in sts])) for k in ("ms_total", "ms_bank", "ms_order", "ms_scan",
                                                                      "ms_certify", "ms_fallback")}
            same = None
            acc = res["acc_idx"]
            acc = acc.cpu().numpy() if hasattr(acc, "cpu") else np.asarray(acc)
            if ref is None:
                ref = acc.copy()
            else:
                same = bool(np.array_equal(ref, acc))
            row = {"N": N, "p": p, "n": n, "J": prob.J, "mode": mode, **med, "n_fallback": int(sts[-1]["n_fallback"]),
                   "pairs_per_s": prob.J * N / (med["ms_total"] / 1e3), "identical_to_fp32": same}
            rows.append(row)
            print(json.dumps(row), flush=True)
            ctx.close()
print(json.dumps({"config5": rows}))
if a.out:
    open(a.out, "w").write(json.dumps({"config5": rows}, indent=1))
