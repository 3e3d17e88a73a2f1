"""Pins of the oracle's simulated-draw noise (abc_set_sim_noise, the P:218-220
observation model applied to the draws as S:301 does; R17).  Box-Muller is checked against
its textbook definition on the Random123-pinned Philox words, the normals against N(0, 1), and the
bank's noise against the variance the P:220 model fixes, ell^2 sigma_f^2 with
sigma_f = sqrt(C e^{-lambda t}/dt) e^{lambda t}."""
import math

import numpy as np
import pytest
from scipy import stats

import synthetic as S
from oracle import oracle as O

SEED = 2026


def bm(seed, i, f):
    x = [int(w) for w in O.philox([i & 0xffffffff, i >> 32, 2 + f // 2, 0x56504554], [seed & 0xffffffff, seed >> 32])]
    ua = ((((x[0] << 32) | x[1]) >> 11) + 0.5) * 2.0 ** -53
    ub = ((((x[2] << 32) | x[3]) >> 11) + 0.5) * 2.0 ** -53
    r = math.sqrt(-2.0 * math.log(ua))
    return r * (math.sin(2 * math.pi * ub) if f & 1 else math.cos(2 * math.pi * ub))


def test_box_muller_definition():
    for i, f in [(0, 0), (0, 1), (1, 0), (12345, 7), (2**33 + 5, 34), (999, 121)]:
        assert O.std_normal(SEED, i, f) == pytest.approx(bm(SEED, i, f), rel=1e-14, abs=1e-15)


def test_normals_are_standard_and_pairwise_uncorrelated():
    z = np.array([[O.std_normal(SEED, i, f) for f in range(4)] for i in range(20000)])
    flat = z.ravel()
    assert abs(flat.mean()) < 4 / math.sqrt(flat.size)
    assert abs(flat.var() - 1.0) < 6 * math.sqrt(2.0 / flat.size)
    assert stats.kstest(flat, "norm").pvalue > 1e-3
    for a, b in [(0, 1), (0, 2), (1, 3)]:  # cos/sin of one pair, and across pairs
        assert abs(np.corrcoef(z[:, a], z[:, b])[0, 1]) < 5 / math.sqrt(z.shape[0])


def fixed_problem(N):
    th = [0.1, 0.2, 0.05, 0.0, 0.05]
    p = S.config1(J=2, N=N)
    return p.replace(models=[dict(kind="2TCM_IRR", n_draws=N, lo=th, hi=th)], n_accept=1), th


def test_zero_noise_is_the_noise_free_bank():
    p, _ = fixed_problem(64)
    c = O.OracleContext(**p.ctx_kwargs)
    p.setup(c)
    b0 = c.bank()
    c.set_sim_noise(0.0, 109.8)
    assert np.array_equal(c.bank(), b0)


def test_bank_noise_follows_the_p220_model():
    """Fixed parameters: every draw has the same noise-free TAC v, so the bank's per-frame spread
    across draws must be ell sigma_f with the P:220 sigma, and each value must be
    RN32(v + ell sigma z_if)."""
    N, ell, thalf = 4000, 3.0, 109.8
    p, th = fixed_problem(N)
    c = O.OracleContext(**p.ctx_kwargs)
    p.setup(c)
    v = c.simulate("2TCM_IRR", np.array(th, dtype=np.float32))
    c.set_sim_noise(ell, thalf)
    b = c.bank().astype(np.float64)
    lam = math.log(2.0) / thalf
    t = p.frame_start + 0.5 * p.frame_dur
    sig = np.sqrt(np.maximum(v, 0) * np.exp(-lam * t) / p.frame_dur) * np.exp(lam * t)
    sd = b.std(axis=0, ddof=1)
    # sample SD within 5 standard errors (sd / sqrt(2(N-1)))
    assert np.all(np.abs(sd - ell * sig) < 5 * ell * sig / math.sqrt(2 * (N - 1)))
    for i in (0, 1, 777, N - 1):
        for f in (0, 5, 21):
            want = np.float32(v[f] + ell * sig[f] * O.std_normal(SEED, i, f))
            assert abs(b[i, f] - float(want)) <= abs(float(want)) * 2.0 ** -23, (i, f)


def test_noise_arguments():
    p, _ = fixed_problem(8)
    c = O.OracleContext(**p.ctx_kwargs)
    for ell, th in [(-1.0, 100.0), (float("nan"), 100.0), (1.0, 0.0), (1.0, -5.0)]:
        with pytest.raises(O.OracleError):
            c.set_sim_noise(ell, th)
    c.set_sim_noise(1.0, float("inf"))  # no decay correction
