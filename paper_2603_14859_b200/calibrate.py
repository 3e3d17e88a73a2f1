"""Pilot calibration of the acceptance rule (§II-D "Threshold h").

The paper tunes h, p and n with a short pilot on simulated data of known truth:
  parameter accuracy: (i) for a small grid of n compute the posterior mean of a target
      parameter and its MSE; (ii) the MSE-vs-n curve is U-shaped; (iii) fit a smooth curve and take
      the n at its minimum;
  model selection: (i) simulate from each model; (ii) over a grid of n compute accuracy and
      ROC AUC of the model probabilities; (iii) choose a working point on the elbow.

Everything that touches the draws runs in the CUDA library: ONE top-n run at the largest n of the
grid (abc_run_voxels), then the summaries of every smaller n by truncation of its sorted accepted
lists (abc_reduce_accepted: the prefix of length n' of a list sorted by (D, i) IS the top-n' set).
This module only does the host-side statistics of the pilot outputs (MSE, curve fit, ROC) and the
mapping from a pilot to an epsilon for eps mode: with a fixed budget N, accepting the
n nearest draws is accepting D <= D_(n), so the eps that accepts n draws in a
typical voxel is a quantile over voxels of the pilot's n-th smallest discrepancy.
"""
from __future__ import annotations

from typing import Dict, Iterable, Optional

import numpy as np


def pilot_sweep(ctx, tacs, n_grid: Iterable[int], want=("prob", "preferred", "count", "mean", "sd", "ki_mean",
                                                          "ki_sd")) -> Dict[int, dict]:
    """Summaries for every n of `n_grid` from ONE run at max(n_grid) (ctx.n_accept must be >= it).

    Returns {n: outputs}; outputs[max] also carries the run's acc_idx / acc_dist."""
    grid = sorted({int(n) for n in n_grid})
    if grid[-1] > ctx.n_accept:
        raise ValueError(f"the context accepts n = {ctx.n_accept} < max(n_grid) = {grid[-1]}")
    full = ctx.run_voxels(tacs)
    out = {}
    for n in grid:
        if n == ctx.n_accept:
            out[n] = full
        else:
            out[n] = ctx.reduce_accepted(full["acc_idx"], n, want=want)
    return out


def epsilon_from_pilot(acc_dist, n: int, q: float = 0.5) -> float:
    """eps such that a fraction q of the pilot voxels accept at least n draws in eps mode.

    acc_dist: J x n_max sorted FP64 discrepancies of a top-n_max pilot run (n <= n_max).  A voxel
    accepts >= n draws under D <= eps iff its n-th smallest D is <= eps, so eps = the q-quantile
    over voxels of D_(n) (type 7)."""
    d = np.asarray(acc_dist, dtype=np.float64)
    if not 1 <= n <= d.shape[1]:
        raise ValueError("need 1 <= n <= n_max of the pilot")
    return float(np.quantile(d[:, n - 1], q, method="linear"))


def mse_curve(post_means: Dict[int, np.ndarray], truth: np.ndarray, mask: Optional[np.ndarray] = None):
    """(ns, mse): mean squared error of the posterior mean of the target parameter per n (P:173 (i))."""
    ns = np.array(sorted(post_means), dtype=np.float64)
    t = np.asarray(truth, dtype=np.float64)
    m = np.ones(t.shape, dtype=bool) if mask is None else np.asarray(mask, dtype=bool)
    mse = np.array([np.mean((np.asarray(post_means[int(n)], dtype=np.float64)[m] - t[m]) ** 2) for n in ns])
    return ns, mse


def fit_u_curve(ns, mse) -> dict:
    """Least-squares quadratic in log n through the MSE curve and the n at its minimum (P:173 (iii)).

    Returns {"n_opt", "coef" (c0, c1, c2 of c0 + c1 x + c2 x^2, x = ln n), "u_shaped"}.  If the fit is
    not convex (no interior minimum), n_opt is the grid point with the smallest MSE."""
    x = np.log(np.asarray(ns, dtype=np.float64))
    y = np.asarray(mse, dtype=np.float64)
    A = np.stack([np.ones_like(x), x, x * x], axis=1)
    coef, *_ = np.linalg.lstsq(A, y, rcond=None)
    c0, c1, c2 = coef
    if c2 > 0:
        xo = -c1 / (2 * c2)
        u = bool(x.min() < xo < x.max())
        n_opt = float(np.exp(np.clip(xo, x.min(), x.max())))
    else:
        u = False
        n_opt = float(np.asarray(ns)[int(np.argmin(y))])
    return {"n_opt": n_opt, "coef": [float(c0), float(c1), float(c2)], "u_shaped": u}


def roc_auc(score, label) -> float:
    """Area under the ROC curve of `score` for the positive class (label True): the Mann-Whitney
    probability P(score_pos > score_neg) + 1/2 P(tie) (P:175 (ii))."""
    s = np.asarray(score, dtype=np.float64)
    y = np.asarray(label, dtype=bool)
    pos, neg = s[y], s[~y]
    if len(pos) == 0 or len(neg) == 0:
        return float("nan")
    allv = np.concatenate([pos, neg])
    order = np.argsort(allv, kind="mergesort")
    ranks = np.empty(len(allv), dtype=np.float64)
    sv = allv[order]
    i = 0
    while i < len(sv):  # average ranks of ties
        j = i
        while j + 1 < len(sv) and sv[j + 1] == sv[i]:
            j += 1
        ranks[order[i:j + 1]] = 0.5 * (i + j) + 1.0
        i = j + 1
    r_pos = ranks[: len(pos)].sum()
    return float((r_pos - len(pos) * (len(pos) + 1) / 2.0) / (len(pos) * len(neg)))


def sens_spec(prob_complex, label, threshold: float = 0.5) -> tuple:
    """Sensitivity and specificity of the '> threshold' model-selection rule for the
    complex model (label True = data simulated from it)."""
    p = np.asarray(prob_complex, dtype=np.float64)
    y = np.asarray(label, dtype=bool)
    call = p > threshold
    sens = float(np.mean(call[y])) if y.any() else float("nan")
    spec = float(np.mean(~call[~y])) if (~y).any() else float("nan")
    return sens, spec
