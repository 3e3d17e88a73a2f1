"""Pilot calibration of the number of accepted draws n.

(i) Parameter accuracy: on config-4-shaped simulation data with known truth, for a grid of
    n, the MSE of the posterior-mean K_i against the true K_i; a quadratic in log n is fitted and
    its minimum reported (the U-shaped MSE curve, P:173 (ii)-(iii)).
(ii) Model selection: on config-2-shaped lp-ntPET / MRTM data, for a grid of n, accuracy,
    sensitivity, specificity of "P(lp-ntPET | y) > 0.5" and the ROC AUC of P(lp-ntPET | y).
Every run is the full hot path through the C ABI (one abc_run_voxels per n).

python tools/pilot_calibration.py [--tb-voxels 8000] [--tb-draws 1000000] [--rt-J 4000]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2603_14859_b200 import FLAG_TIMING, AbcContext  # noqa: E402


def auc(score, label):
    """ROC AUC by the rank-sum (Mann-Whitney) formula, ties counted half."""
    pos, neg = score[label], score[~label]
    if len(pos) == 0 or len(neg) == 0:
        return float("nan")
    allv = np.concatenate([pos, neg])
    order = np.argsort(allv, kind="mergesort")
    ranks = np.empty(len(allv))
    sv = allv[order]
    i = 0
    while i < len(sv):
        j = i
        while j + 1 < len(sv) and sv[j + 1] == sv[i]:
            j += 1
        ranks[order[i:j + 1]] = 0.5 * (i + j) + 1.0
        i = j + 1
    return float((ranks[: len(pos)].sum() - len(pos) * (len(pos) + 1) / 2) / (len(pos) * len(neg)))


ap = argparse.ArgumentParser()
ap.add_argument("--tb-voxels", type=int, default=8000)
ap.add_argument("--tb-draws", type=int, default=1_000_000)
ap.add_argument("--tb-n", default="1,2,3,5,8,12,18,27,40,60,90,135,200")
ap.add_argument("--rt-J", type=int, default=4000)
ap.add_argument("--rt-per-model", type=int, default=100_000)
ap.add_argument("--rt-n", default="15,25,50,100,150,200")
a = ap.parse_args()
out = {}

# (i) parameter accuracy on the TB phantom (truth known)
tb = S.config4_chunk(chunk=5, n_chunks=32, N=a.tb_draws, n=18, max_voxels=a.tb_voxels)
th = tb.truth["theta"]
ki_true = th[:, 0] * th[:, 2] / (th[:, 1] + th[:, 2])
rows = []
for n in [int(x) for x in a.tb_n.split(",")]:
    ctx = AbcContext(**dict(tb.ctx_kwargs, n_accept=n, flags=FLAG_TIMING))
    tb.setup(ctx)
    r = ctx.run_voxels(tb.tacs, want=("ki_mean", "prob"))
    est = r["ki_mean"].astype(np.float64)
    ok = np.isfinite(est)
    err = est[ok] - ki_true[ok]
    rows.append({"n": n, "mse_ki": float(np.mean(err ** 2)), "bias_ki": float(np.mean(err)),
                 "var_ki": float(np.var(err)), "ms_total": ctx.stats()["ms_total"]})
    print(json.dumps(rows[-1]), flush=True)
    ctx.close()
ln = np.log([r["n"] for r in rows])
mse = np.array([r["mse_ki"] for r in rows])
c2, c1, c0 = np.polyfit(ln, mse, 2)
n_opt = float(np.exp(-c1 / (2 * c2))) if c2 > 0 else float("nan")
out["parameter_accuracy"] = {"data": f"config-4 TB phantom, {tb.J} voxels, N = {a.tb_draws}, IRR vs REV",
                             "target": "K_i = K1 k3/(k2+k3), posterior mean (P:282)", "rows": rows,
                             "quadratic_fit_log_n": [float(c2), float(c1), float(c0)], "n_at_fitted_min": n_opt,
                             "n_at_observed_min": rows[int(np.argmin(mse))]["n"]}

# (ii) model selection on lp-ntPET / MRTM simulation data
rt_rows = []
for noise in ("low", "mid", "high"):
    rt = S.config2(J=a.rt_J, N_per_model=a.rt_per_model, n=100, noise=noise)
    act = rt.truth["active"]
    for n in [int(x) for x in a.rt_n.split(",")]:
        ctx = AbcContext(**dict(rt.ctx_kwargs, n_accept=n, flags=FLAG_TIMING))
        rt.setup(ctx)
        r = ctx.run_voxels(rt.tacs, want=("prob",))
        p_lp = r["prob"][:, 1].astype(np.float64)
        call = p_lp > 0.5
        row = {"noise": noise, "n": n, "sensitivity": float(np.mean(call[act])), "specificity": float(np.mean(~call[~act])),
               "accuracy": float(np.mean(call == act)), "auc": auc(p_lp, act), "ms_total": ctx.stats()["ms_total"]}
        rt_rows.append(row)
        print(json.dumps(row), flush=True)
        ctx.close()
out["model_selection"] = {"data": f"config-2 lp-ntPET vs MRTM, J = {a.rt_J}, {a.rt_per_model} draws per model",
                          "rows": rt_rows}
print(json.dumps({"pilot_calibration": out}))
