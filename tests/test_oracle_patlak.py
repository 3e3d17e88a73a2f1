"""Pins of the oracle's Patlak K_i map (P:282's clinical reference, Patlak 1983; SURVEY §8f-4;
DESIGN.md R18): exact recovery of a line built from independently integrated input curves, the
Patlak limit of the irreversible 2TCM (slope -> K_i = K1 k3/(k2+k3)), and the degenerate cases."""
import math

import numpy as np
import pytest
from scipy import integrate

import synthetic as S
from oracle import oracle as O

FENG = [1.0e5, 5.0e4, 1.5e4, 10.0, 0.5, 0.02]


def feng(t):
    b1, b2, b3, k1, k2, k3 = FENG
    return (b1 * t - b2 - b3) * math.exp(-k1 * t) + b2 * math.exp(-k2 * t) + b3 * math.exp(-k3 * t)


def ctx_feng(start, dur):
    c = O.OracleContext([dict(kind="2TCM_IRR", n_draws=4, lo=[0.1, 0.1, 0.05, 0, 0.05], hi=[0.1, 0.1, 0.05, 0, 0.05])])
    c.set_input_function("FENG", np.array(FENG))
    c.set_frames(start, dur)
    return c


def test_exact_line_is_recovered():
    """y_f = K X_f + V Cp_f with X, Cp from adaptive quadrature of the Feng curve."""
    start, dur = S.fdg22()
    c = ctx_feng(start, dur)
    mid = start + 0.5 * dur
    cp = np.array([integrate.quad(feng, s, s + d, epsabs=0, epsrel=1e-13, limit=200)[0] / d for s, d in zip(start, dur)])
    X = np.array([integrate.quad(feng, 0, t, epsabs=0, epsrel=1e-13, limit=400, points=[0.1, 0.5, 1.0])[0] for t in mid])
    K, V = 0.0123, 0.37
    y = (K * X + V * cp).astype(np.float32)[None, :]
    ki, v0 = c.patlak(y, 10.0)
    assert ki[0] == pytest.approx(K, rel=2e-6)
    assert v0[0] == pytest.approx(V, rel=2e-5)


def test_patlak_limit_of_irreversible_2tcm_step_input():
    """Step input C_p = c: the irreversible 2TCM TAC becomes linear in t = X/Cp at late times with
    slope K_i = K1 k3/(k2+k3) (eq:2TCM_op P:75-80, k4 = 0)."""
    th = [0.2, 0.3, 0.1, 0.0, 0.0]
    c = O.OracleContext([dict(kind="2TCM_IRR", n_draws=2, lo=th, hi=th)])
    c.set_input_function("PWL", np.array([50.0, 50.0]), t=np.array([0.0, 500.0]))
    start = np.arange(0, 120, 4.0)
    dur = np.full(start.size, 4.0)
    c.set_frames(start, dur)
    y = c.simulate("2TCM_IRR", th).astype(np.float32)[None, :]
    ki, _ = c.patlak(y, 60.0)
    assert ki[0] == pytest.approx(0.2 * 0.1 / (0.3 + 0.1), rel=2e-3)


def test_degenerate_cases():
    start, dur = np.array([0.0, 5.0, 10.0]), np.array([5.0, 5.0, 5.0])
    c = ctx_feng(start, dur)
    y = np.ones((2, 3), dtype=np.float32)
    ki, v0 = c.patlak(y, 12.0)  # one frame with mid >= 12: no line
    assert np.all(np.isnan(ki)) and np.all(np.isnan(v0))
    ki2, _ = c.patlak(np.zeros((1, 3), dtype=np.float32), 0.0)
    assert ki2[0] == 0.0
