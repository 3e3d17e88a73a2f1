"""Pins of the oracle's response-function credible envelope (Fig. 1):
r(t) = k2a(t)/k2a = 1 + (gamma/k2a) g(t), quantiles over a voxel's accepted lp-ntPET draws.
Pinned against values the definition fixes: r = 1 before onset and for gamma = 0, the closed form
r(tP) = 1 + gamma/k2a (g peaks at 1 at tP, eq:Bt P:90-94 with the S:70 normalisation), NaN without
lp-ntPET draws, and numpy's linear-interpolation quantiles of a brute-force evaluation."""
import math

import numpy as np
import pytest

from oracle import oracle as O

LO = [0.5, 0.05, 0.01, 0.0, 15, 1, 0.25]
HI = [1.5, 0.6, 0.2, 0.2, 45, 45, 4]


def ctx(lo=LO, hi=HI, n=200):
    c = O.OracleContext([dict(kind="MRTM", n_draws=n, lo=lo, hi=hi), dict(kind="LPNTPET", n_draws=n, lo=lo, hi=hi)])
    st = np.arange(10, dtype=np.float64) * 6.0
    c.set_input_function("PWL", np.array([0.0, 1.0, 60.0]), t=np.array([0.0, 1.0, 60.0]))
    c.set_frames(st, np.full(10, 6.0))
    return c


def lp_draws(c):
    out = []
    for i in range(c.N):
        m, th = c.draw(i)
        if m == 1:
            out.append((i, th))
    return out


def test_before_onset_and_gamma_zero_are_flat():
    c = ctx()
    lp = lp_draws(c)
    idx = np.array([[i for i, _ in lp[:40]]], dtype=np.uint64)
    q = c.response_envelope(idx, np.array([0.0, 5.0, 14.999]))  # tD >= 15 under the prior
    assert np.all(q == 1.0)
    lo0, hi0 = list(LO), list(HI)
    hi0[3] = 0.0  # gamma fixed at 0
    c0 = ctx(lo0, hi0)
    idx0 = np.array([[i for i, _ in lp_draws(c0)[:30]]], dtype=np.uint64)
    assert np.all(c0.response_envelope(idx0, np.linspace(0, 120, 13)) == 1.0)


def test_single_draw_peak_closed_form():
    c = ctx()
    for i, th in lp_draws(c)[:5]:
        tP = float(th[5])
        q = c.response_envelope(np.array([[i]], dtype=np.uint64), np.array([tP, float(th[4])]))
        want = np.float32(1.0 + float(th[3]) / float(th[2]))  # g(tP) = 1
        assert np.all(q[0, 0] == want), (q[0, 0], want)
        assert np.all(q[0, 1] == 1.0)  # g(tD) = 0


def test_no_lpntpet_draw_gives_nan_and_errors():
    c = ctx()
    mrtm = [i for i in range(c.N) if c.draw(i)[0] == 0][:10]
    q = c.response_envelope(np.array([mrtm], dtype=np.uint64), np.array([20.0, 40.0]))
    assert np.all(np.isnan(q))
    with pytest.raises(O.OracleError):
        c.response_envelope(np.array([[c.N]], dtype=np.uint64), np.array([1.0]))
    c1 = O.OracleContext([dict(kind="MRTM", n_draws=10, lo=LO, hi=HI)])
    c1.set_input_function("PWL", np.array([0.0, 1.0]), t=np.array([0.0, 60.0]))
    c1.set_frames(np.array([0.0]), np.array([60.0]))
    with pytest.raises(O.OracleError) as e:
        c1.response_envelope(np.array([[0]], dtype=np.uint64), np.array([1.0]))
    assert e.value.status == 5


def test_brute_force_numpy_quantiles():
    """Two voxels with mixed MRTM / lp-ntPET accepted lists against a direct evaluation of
    x^alpha e^{alpha(1-x)} and numpy's type-7 quantiles."""
    c = ctx()
    rng = np.random.default_rng(3)
    idx = np.stack([rng.choice(c.N, 57, replace=False) for _ in range(2)]).astype(np.uint64)
    t = np.array([0.0, 16.0, 22.5, 30.0, 44.0, 61.0, 90.0, 240.0])
    q = c.response_envelope(idx, t)
    for j in range(2):
        ths = [c.draw(int(i))[1] for i in idx[j] if c.draw(int(i))[0] == 1]
        for k, tk in enumerate(t):
            r = []
            for th in ths:
                tD, tP, al = float(th[4]), float(th[5]), float(th[6])
                g = 0.0 if tk <= tD else math.pow((tk - tD) / (tP - tD), al) * math.exp(al * (1 - (tk - tD) / (tP - tD)))
                r.append(1.0 + float(th[3]) / float(th[2]) * g)
            want = np.quantile(np.array(r), [0.025, 0.5, 0.975], method="linear").astype(np.float32)
            np.testing.assert_allclose(q[j, k], want, rtol=2e-7, atol=0)
            assert q[j, k, 0] <= q[j, k, 1] <= q[j, k, 2]
