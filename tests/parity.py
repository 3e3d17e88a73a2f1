"""Parity helpers: run the CUDA path (through the C ABI) and the CPU oracle on the same seeded
inputs and compare element by element with the tolerances of BASELINE.json's north star:
  * accepted-index sets bit-exact, except draws whose discrepancy lies within 1e-6 relative of
    the acceptance boundary (such voxels are counted separately);
  * posterior means and SDs within 1e-4 relative; model probabilities within 1e-3 absolute
    (on voxels whose accepted sets match).
"""
from __future__ import annotations

import numpy as np

BOUNDARY_REL = 1e-6
MOMENT_RTOL = 1e-4
PROB_ATOL = 1e-3


def run_gpu(problem, tacs=None, **overrides):
    from paper_2603_14859_b200 import AbcContext
    kw = dict(problem.ctx_kwargs)
    kw.update(overrides)
    ctx = AbcContext(**kw)
    problem.setup(ctx)
    res = ctx.run_voxels(problem.tacs if tacs is None else tacs)
    return res, ctx


def run_oracle(problem, tacs=None, **overrides):
    from oracle import oracle as O
    kw = dict(problem.ctx_kwargs)
    kw.update(overrides)
    kw.pop("flags", None)
    ctx = O.OracleContext(**kw)
    problem.setup(ctx)
    return ctx.run_voxels(problem.tacs if tacs is None else tacs), ctx


def _close(a, b, rtol, atol=0.0):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nan_a, nan_b = np.isnan(a), np.isnan(b)
    if not np.array_equal(nan_a, nan_b):
        return False
    m = ~nan_a
    return bool(np.all(np.abs(a[m] - b[m]) <= atol + rtol * np.abs(b[m])))


def compare(gpu: dict, ora: dict, topn: bool = True, max_exempt_frac: float = 0.05):
    """Return a report dict; raise AssertionError on any violation."""
    J = len(ora["preferred"])
    same = np.ones(J, dtype=bool)
    exempt = 0
    if topn:
        gi, oi = gpu["acc_idx"].astype(np.int64), ora["acc_idx"].astype(np.int64)
        gd, od = gpu["acc_dist"], ora["acc_dist"]
        for j in range(J):
            if np.array_equal(gi[j], oi[j]):
                # identical indices: identical FP64 distances up to RN32 flips in the bank
                assert np.allclose(gd[j], od[j], rtol=1e-9, atol=0), (j, gd[j], od[j])
                continue
            tau = od[j, -1]
            sg, so = set(gi[j].tolist()), set(oi[j].tolist())
            dist = {int(i): float(d) for i, d in zip(gi[j], gd[j])}
            dist.update({int(i): float(d) for i, d in zip(oi[j], od[j])})
            for i in sg ^ so:
                assert abs(dist[i] - tau) <= BOUNDARY_REL * abs(tau), (j, i, dist[i], tau)
            if sg == so:  # same set, order differs only among boundary-equal distances
                same[j] = True
                continue
            same[j] = False
            exempt += 1
            # a voxel whose accepted set differs only by boundary swaps still obeys
            # |P_gpu(m) - P_oracle(m)| <= (#swaps)/n and |count_gpu - count_oracle| <= #swaps
            swaps = len(sg - so)
            n = gi.shape[1]
            assert np.all(np.abs(gpu["count"][j].astype(np.int64) - ora["count"][j].astype(np.int64)) <= swaps), j
            assert np.all(np.abs(gpu["prob"][j].astype(np.float64) - ora["prob"][j]) <= swaps / n + PROB_ATOL), j
        assert exempt <= max(1, max_exempt_frac * J), f"{exempt} of {J} voxels differ at the boundary"
    else:
        same = np.all(gpu["count"] == ora["count"], axis=1)
    s = same
    assert np.array_equal(gpu["preferred"][s], ora["preferred"][s])
    assert np.array_equal(gpu["count"][s], ora["count"][s])
    assert _close(gpu["prob"][s], ora["prob"][s], 0.0, PROB_ATOL)
    for k in ("mean", "ki_mean"):
        assert _close(gpu[k][s], ora[k][s], MOMENT_RTOL, 1e-12), k
    for k in ("sd", "ki_sd"):
        assert _close(gpu[k][s], ora[k][s], MOMENT_RTOL, 1e-9), k
    for k in ("q", "ki_q"):
        assert _close(gpu[k][s], ora[k][s], MOMENT_RTOL, 1e-12), k
    return {"J": J, "boundary_exempt": exempt, "matched": int(s.sum())}
