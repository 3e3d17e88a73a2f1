"""Pins of the CPU oracle against things other than itself (closed forms, ODE solutions,
quadrature, known-answer vectors, brute force, limits).  CPU only (-m "not gpu").

Each test names the paper passage it pins.  A plausible slip in the oracle (dropped term,
wrong sign, swapped operand, wrong index) should fail at least one of them.
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest
from scipy import integrate, stats

from oracle import oracle as O

mpmath.mp.dps = 50
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))
FENG = [1.0e5, 5.0e4, 1.5e4, 10.0, 0.5, 0.02]
LO_FDG = [0.001, 0.001, 0.001, 0.0, 0.03]
HI_FDG = [1.0, 2.0, 0.5, 0.1, 0.2]


def fdg22():
    d = np.array([15] * 8 + [60] * 4 + [120] * 4 + [360] * 6, dtype=np.float64) / 60.0
    return np.concatenate([[0.0], np.cumsum(d)[:-1]]), d


def ctx_fdg(kind="2TCM_REV", N=16, lo=LO_FDG, hi=HI_FDG, input_kind="FENG", knots=None, frames=None, **kw):
    c = O.OracleContext([dict(kind=kind, n_draws=N, lo=lo, hi=hi)], **kw)
    if input_kind == "FENG":
        c.set_input_function("FENG", FENG)
    else:
        c.set_input_function("PWL", knots[1], t=knots[0])
    st, du = frames if frames is not None else fdg22()
    c.set_frames(st, du)
    return c


def feng_np(t):
    b1, b2, b3, k1, k2, k3 = FENG
    return (b1 * t - b2 - b3) * np.exp(-k1 * t) + b2 * np.exp(-k2 * t) + b3 * np.exp(-k3 * t)


def ode_2tcm_frames(theta, cp, start, dur, breaks=()):
    """Reference: DOP853 integration of eq:2TCM with Q' = eq:2TCM_op, rtol 1e-12.
    Integrates piecewise between `breaks` (input kinks) and frame bounds."""
    K1, k2, k3, k4, Vb = [float(v) for v in theta]

    def f(t, y):
        c = cp(t)
        return [K1 * c - (k2 + k3) * y[0] + k4 * y[1], k3 * y[0] - k4 * y[1],
                (1 - Vb) * (y[0] + y[1]) + Vb * c]

    pts = sorted(set([0.0] + list(breaks) + list(start) + list(start + dur)))
    y = np.zeros(3)
    Q = {0.0: 0.0}
    for a, b in zip(pts[:-1], pts[1:]):
        sol = integrate.solve_ivp(f, (a, b), y, method="DOP853", rtol=1e-13, atol=1e-10)
        y = sol.y[:, -1]
        Q[b] = y[2]
    return np.array([(Q[s + d] - Q[s]) / d for s, d in zip(start, dur)])


# ------------------------------------------------------------------ Philox / draws
def test_philox_known_answers():
    """Philox4x32-10 KATs (Random123) -- the counter-based sampler of Alg.1 l.1-2."""
    for case in GOLD["philox4x32_10_kat"]["cases"]:
        ctr = [int(x, 16) for x in case["ctr"]]
        key = [int(x, 16) for x in case["key"]]
        assert [int(x) for x in O.philox(ctr, key)] == [int(x, 16) for x in case["out"]]


def test_uniform_mapping_exact_open_interval():
    assert O.uniform(0) == 2.0 ** -24
    assert O.uniform(0xFFFFFFFF) == 1.0 - 2.0 ** -24
    assert O.uniform(0x1FF) == O.uniform(0)  # only the top 23 bits matter
    assert O.uniform(1 << 9) == 3 * 2.0 ** -24
    for x in np.random.default_rng(0).integers(0, 2 ** 32, 1000):
        u = O.uniform(int(x))
        assert 0.0 < u < 1.0 and u == ((int(x) >> 9) * 2 + 1) * 2.0 ** -24


def test_prior_draws_uniform_and_bounded():
    """eq:prior2 uniform priors: support, KS uniformity, fixed params (lo==hi)."""
    N = 20000
    lo = [0.001, 0.001, 0.001, 0.0, 0.05]
    hi = [1.0, 2.0, 0.5, 0.1, 0.05]  # Vb fixed
    c = ctx_fdg(N=N, lo=lo, hi=hi)
    th = np.array([c.draw(i)[1] for i in range(N)])
    for k in range(4):
        assert th[:, k].min() >= lo[k] and th[:, k].max() <= hi[k]
        u = (th[:, k] - lo[k]) / (hi[k] - lo[k])
        assert stats.kstest(u, "uniform").pvalue > 1e-3
    assert np.all(th[:, 4] == np.float32(0.05))
    # parameter columns are drawn from distinct Philox words: near-zero correlation
    assert abs(np.corrcoef(th[:, 0], th[:, 1])[0, 1]) < 0.05


def test_draw_matches_hand_philox_fmaf():
    """theta_k = fmaf(hi-lo, u_k, lo) with u_k from Philox(ctr={i,0,k/4,'VPET'}, key=seed)."""
    seed = 0x0123456789ABCDEF
    c = ctx_fdg(N=100, seed=seed)
    for i in (0, 1, 57, 99):
        m, th = c.draw(i)
        key = [seed & 0xFFFFFFFF, seed >> 32]
        words = list(O.philox([i, 0, 0, 0x56504554], key)) + list(O.philox([i, 0, 1, 0x56504554], key))
        for k in range(5):
            u = np.float32(((int(words[k]) >> 9) * 2 + 1) * 2.0 ** -24)
            span = np.float32(HI_FDG[k]) - np.float32(LO_FDG[k])
            exact = float(span) * float(u) + float(np.float32(LO_FDG[k]))  # fmaf: one rounding
            assert th[k] == np.float32(exact)


def test_model_blocks_irr_and_lpntpet_constraints():
    """Alg.1 l.1 (stratified blocks); IRR k4 = 0; lp-ntPET tP = tD + offset > tD."""
    c = O.OracleContext([dict(kind="2TCM_IRR", n_draws=3, lo=LO_FDG, hi=HI_FDG),
                         dict(kind="2TCM_REV", n_draws=5, lo=LO_FDG, hi=HI_FDG)])
    ms = [c.draw(i)[0] for i in range(8)]
    assert ms == [0, 0, 0, 1, 1, 1, 1, 1]
    assert all(c.draw(i)[1][3] == 0.0 for i in range(3))
    assert any(c.draw(i)[1][3] > 0.0 for i in range(3, 8))
    lo, hi = [0.5, 0.05, 0.01, 0.0, 15, 1, 0.25], [1.5, 0.6, 0.2, 0.2, 45, 45, 4]
    r = O.OracleContext([dict(kind="MRTM", n_draws=50, lo=lo, hi=hi), dict(kind="LPNTPET", n_draws=50, lo=lo, hi=hi)])
    for i in range(100):
        m, th = r.draw(i)
        assert th[5] > th[4]
        if m == 0:
            assert th[3] == 0.0


# ------------------------------------------------------------------ forward models
@pytest.mark.parametrize("theta", [
    (0.1, 0.2, 0.05, 0.01, 0.05),
    (0.8, 1.5, 0.3, 0.0, 0.15),       # irreversible
    (0.5, 0.45, 0.05, 0.0, 0.1),      # a2 = k2+k3 = 0.5 = kappa2 exactly (a == kappa branch)
    (0.05, 0.1, 0.01, 0.1, 0.03),     # slow, reversible
    (1.0, 2.0, 0.5, 0.1, 0.2),        # fast corner of the prior
    (0.3, 0.02, 0.001, 0.001, 0.05),  # tiny rates
])
def test_2tcm_feng_closed_form_vs_ode(theta):
    """eq:2TCM + eq:2TCM_op with the Feng input vs DOP853 ODE integration."""
    c = ctx_fdg()
    st, du = fdg22()
    ref = ode_2tcm_frames(theta, lambda t: feng_np(t), st, du)
    got = c.simulate("2TCM_REV", theta)
    th32 = np.float32(theta)
    ref32 = ode_2tcm_frames(th32, lambda t: feng_np(t), st, du)
    np.testing.assert_allclose(got, ref32, rtol=2e-9, atol=0)
    assert np.all(np.isfinite(ref))


def _pwl_knots():
    st, du = fdg22()
    mid = st + du / 2
    rng = np.random.default_rng(3)
    v = feng_np(mid) * (1 + 0.02 * rng.standard_normal(len(mid)))
    return np.concatenate([[0.0], mid]), np.concatenate([[0.0], v])


@pytest.mark.parametrize("theta", [(0.1, 0.2, 0.05, 0.01, 0.05), (0.8, 1.5, 0.3, 0.0, 0.15),
                                   (0.05, 0.1, 0.01, 0.1, 0.03), (0.3, 0.02, 0.001, 0.0, 0.05)])
def test_2tcm_pwl_closed_form_vs_ode(theta):
    """PWL IDIF input (reading R1: linear through (0,0),(mid_f,v_f), held after the last
    knot) -- exact recurrences vs DOP853 integrated piecewise between kinks."""
    kt, kv = _pwl_knots()
    c = ctx_fdg(input_kind="PWL", knots=(kt, kv))
    st, du = fdg22()
    th32 = np.float32(theta)
    cp = lambda t: float(np.interp(t, kt, kv))  # np.interp holds the last value
    ref = ode_2tcm_frames(th32, cp, st, du, breaks=kt)
    np.testing.assert_allclose(c.simulate("2TCM_REV", theta), ref, rtol=2e-9, atol=0)


def test_2tcm_step_input_textbook_closed_form():
    """C_p = c constant, k4 = Vb = 0: frame mean = c K1/a [k3 mid + k2/a - k2/a^2 (e^{-a ts}-e^{-a te})/dt],
    a = k2+k3 (textbook solution of eq:2TCM with a step input)."""
    cc = 123.0
    kt, kv = np.array([0.0, 60.0]), np.array([cc, cc])
    c = ctx_fdg(input_kind="PWL", knots=(kt, kv))
    st, du = fdg22()
    for th in [(0.1, 0.2, 0.05, 0.0, 0.0), (0.9, 1.7, 0.4, 0.0, 0.0), (0.01, 0.003, 0.001, 0.0, 0.0)]:
        K1, k2, k3 = [mpmath.mpf(float(np.float32(x))) for x in th[:3]]
        a = k2 + k3
        exp_ = [float(cc * K1 / a * (k3 * (mpmath.mpf(s) + mpmath.mpf(d) / 2) + k2 / a
                                     - k2 / a ** 2 * (mpmath.exp(-a * s) - mpmath.exp(-a * (s + d))) / d))
                for s, d in zip(st, du)]  # evaluated in 50-digit arithmetic
        np.testing.assert_allclose(c.simulate("2TCM_IRR", th), exp_, rtol=1e-12)


def test_2tcm_k1_zero_gives_blood_term():
    """K1 = 0: C_T = Vb C_wb (eq:2TCM_op); frame means of Feng by adaptive quadrature."""
    c = ctx_fdg()
    st, du = fdg22()
    th = (0.0, 0.3, 0.1, 0.02, 0.1)
    ref = np.array([integrate.quad(feng_np, s, s + d, epsabs=0, epsrel=1e-13, limit=200)[0] / d
                    for s, d in zip(st, du)]) * float(np.float32(0.1))
    np.testing.assert_allclose(c.simulate("2TCM_REV", th), ref, rtol=1e-10)


def test_patlak_limit_step_input():
    """Irreversible 2TCM conforms to Patlak: late-frame OLS slope of C_T/C_p vs int C_p/C_p
    equals K_i = K1 k3/(k2+k3).  Step input: exact once e^{-a t} has decayed."""
    cc = 50.0
    c = ctx_fdg(input_kind="PWL", knots=(np.array([0.0, 60.0]), np.array([cc, cc])))
    st, du = fdg22()
    mid = st + du / 2
    late = mid >= 20
    for th in [(0.2, 0.4, 0.2, 0.0, 0.0), (0.5, 1.0, 0.3, 0.0, 0.0)]:
        v = c.simulate("2TCM_IRR", th)
        slope = np.polyfit(mid[late], v[late] / cc, 1)[0]
        K1, k2, k3 = [float(np.float32(x)) for x in th[:3]]
        assert abs(slope / (K1 * k3 / (k2 + k3)) - 1) < 1e-6


def test_patlak_limit_feng_input():
    """Same with the Feng input: holds within 0.5 % once k2+k3 >= 0.25 (SURVEY A§9)."""
    c = ctx_fdg()
    st, du = fdg22()
    mid = st + du / 2
    late = mid >= 20
    cp = feng_np(mid)
    icp = np.array([integrate.quad(feng_np, 0, m, epsrel=1e-12, limit=200)[0] for m in mid])
    for th in [(0.5, 1.0, 0.3, 0.0, 0.0), (0.8, 1.5, 0.05, 0.0, 0.0)]:
        v = c.simulate("2TCM_IRR", th)
        slope = np.polyfit(icp[late] / cp[late], v[late] / cp[late], 1)[0]
        K1, k2, k3 = [float(np.float32(x)) for x in th[:3]]
        assert abs(slope / (K1 * k3 / (k2 + k3)) - 1) < 5e-3


def test_feng_zero_and_direct_value():
    g = GOLD["feng_zero"]
    assert O.feng(g["params"], g["t"]) == g["expected"]
    t = 1.3
    b1, b2, b3, k1, k2, k3 = FENG
    assert O.feng(FENG, t) == pytest.approx((b1 * t - b2 - b3) * math.exp(-k1 * t) + b2 * math.exp(-k2 * t)
                                            + b3 * math.exp(-k3 * t), rel=1e-14)


def test_gamma_variate_examples():
    for cse in GOLD["gamma_variate"]["cases"]:
        assert O.gamma_variate(cse["tD"], cse["tP"], cse["alpha"], cse["t"]) == pytest.approx(cse["g"], abs=1e-15)


def rt_ctx(kinds=("MRTM", "LPNTPET"), step=0.05, cr=None, n=4):
    st = np.arange(61, dtype=np.float64)
    du = np.ones(61)
    mid = st + 0.5
    if cr is None:
        t = np.linspace(0, 61, 400)
        cr = 1e4 * (t * np.exp(-t / 4.0) / 4.0 + 0.3 * (1 - np.exp(-t / 2.0)) * np.exp(-t / 60.0))
        cr = np.interp(mid, t, cr)
    lo, hi = [0.5, 0.05, 0.01, 0.0, 15, 1, 0.25], [1.5, 0.6, 0.2, 0.2, 45, 45, 4]
    c = O.OracleContext([dict(kind=k, n_draws=n, lo=lo, hi=hi) for k in kinds], lpnt_step_min=step)
    kt = np.concatenate([[0.0], mid])
    kv = np.concatenate([[0.0], cr])
    c.set_input_function("PWL", kv, t=kt)
    c.set_frames(st, du)
    return c, (kt, kv), st, du


def ode_rt_frames(theta, knots, st, du):
    """Reference: DOP853 on the differentiated eq:lp-ntPET, z = C_t - R1 C_r:
    z' = (k2 - R1 a(t)) C_r - a(t) z, a = k2a + gamma g(t), with Q' = z + R1 C_r."""
    R1, k2, k2a, gam, tD, tP, al = [float(v) for v in theta]
    kt, kv = knots

    def g(t):
        if t <= tD:
            return 0.0
        x = (t - tD) / (tP - tD)
        return x ** al * math.exp(al * (1 - x))

    def f(t, y):
        cr = float(np.interp(t, kt, kv))
        a = k2a + gam * g(t)
        return [(k2 - R1 * a) * cr - a * y[0], y[0] + R1 * cr]

    pts = sorted(set(list(kt) + list(st) + list(st + du) + [tD]))
    pts = [p for p in pts if p <= st[-1] + du[-1]]
    y = np.zeros(2)
    Q = {0.0: 0.0}
    for a, b in zip(pts[:-1], pts[1:]):
        sol = integrate.solve_ivp(f, (a, b), y, method="DOP853", rtol=1e-12, atol=1e-9)
        y = sol.y[:, -1]
        Q[b] = y[1]
    return np.array([(Q[s + d] - Q[s]) / d for s, d in zip(st, du)])


def test_mrtm_vs_ode_and_equals_lpntpet_gamma0():
    """MRTM = lp-ntPET with gamma = 0: closed form vs ODE, and vs the lp-ntPET integrator
    (which is exact for constant a, so the two agree to rounding although grids differ)."""
    c, knots, st, du = rt_ctx()
    th = np.float32([1.1, 0.35, 0.09, 0.0, 30.0, 42.0, 1.2])
    v_m = c.simulate("MRTM", th)
    v_l = c.simulate("LPNTPET", th)
    np.testing.assert_allclose(v_m, v_l, rtol=1e-12)
    np.testing.assert_allclose(v_m, ode_rt_frames(th, knots, st, du), rtol=1e-9)


def test_reference_zero_gives_zero():
    c, knots, st, du = rt_ctx(cr=np.zeros(61))
    th = np.float32([1.1, 0.35, 0.09, 0.05, 30.0, 42.0, 1.2])
    assert np.all(c.simulate("LPNTPET", th) == 0.0)
    assert np.all(c.simulate("MRTM", th) == 0.0)


@pytest.mark.parametrize("theta", [(1.0, 0.3, 0.1, 0.05, 35.0, 40.0, 1.0), (1.2, 0.5, 0.08, 0.15, 31.0, 36.0, 0.3),
                                   (0.8, 0.2, 0.15, 0.1, 20.0, 50.0, 3.5)])
def test_lpntpet_converges_to_ode_second_order(theta):
    """lp-ntPET (eq:lp-ntPET, eq:Bt) vs the exact ODE solution (DOP853): the midpoint-frozen
    integrator (reading R4) must converge at order min(2, 1+alpha) in delta and be within 2e-4 at
    delta=0.05."""
    th = np.float32(theta)
    errs = []
    for step in (0.1, 0.05, 0.025):
        c, knots, st, du = rt_ctx(step=step)
        ref = ode_rt_frames(th, knots, st, du)
        errs.append(np.max(np.abs(c.simulate("LPNTPET", th) - ref) / np.abs(ref).max()))
    assert errs[1] < 2e-4
    # midpoint-frozen rate: order 2 for smooth g; g ~ x^alpha near tD limits it to 1 + alpha
    order = min(2.0, 1.0 + float(theta[6]))
    assert errs[0] / errs[1] > 0.75 * 2 ** order and errs[1] / errs[2] > 0.75 * 2 ** order


# ------------------------------------------------------------------ distance
def test_distance_examples():
    y = np.float32([1.5, -2.0, 3.25])
    assert O.distance("WL2", y, y) == 0.0 and O.distance("L1", y, y) == 0.0
    s = np.float32([1.0, 1.0, 1.0])
    w = np.float32([2.0, 0.5, 1.0])
    assert O.distance("WL2", y, s, w) == 2 * 0.25 + 0.5 * 9.0 + 2.25 ** 2
    assert O.distance("L1", y, s, w) == 2 * 0.5 + 0.5 * 3.0 + 2.25
    assert O.distance("L1", [2.0], [1.0]) == 1.0 and O.distance("L1", [2.0], [3.0]) == 1.0


# ------------------------------------------------------------------ selection + reduction
def _tiny_problem(N=12, J=3, L=4, seed=5):
    rng = np.random.default_rng(seed)
    st = np.arange(L, dtype=np.float64) * 2.0
    du = np.full(L, 2.0)
    c = O.OracleContext([dict(kind="2TCM_REV", n_draws=N, lo=LO_FDG, hi=HI_FDG)], n_accept=4, seed=9)
    c.set_input_function("FENG", FENG)
    c.set_frames(st, du)
    bank = c.bank()
    y = (bank[rng.integers(0, N, J)] * rng.uniform(0.8, 1.2, (J, L))).astype(np.float32)
    return c, bank, y, st, du


def test_bank_is_rn32_of_simulation():
    c, bank, y, st, du = _tiny_problem()
    for i in range(bank.shape[0]):
        m, th = c.draw(i)
        np.testing.assert_array_equal(bank[i], c.simulate("2TCM_REV", th).astype(np.float32))


@pytest.mark.parametrize("dist", ["WL2", "L1"])
def test_topn_equals_bruteforce_sort_and_rejection_loop(dist):
    """Alg.1 l.4-5: top-n by (D, index) == enumerate-and-sort on tiny N; eps mode ==
    the sequential rejection loop of P:131 ("accepts the draw if the discrepancy ... below h")."""
    N, n = 12, 4
    c0, bank, y, st, du = _tiny_problem(N=N)
    w = np.float32([0.5, 1.0, 2.0, 1.5])
    for mode in ("TOPN", "EPS"):
        D = np.array([[sum(float(w[f]) * (abs(float(y[j, f]) - float(bank[i, f])) if dist == "L1"
                                         else (float(y[j, f]) - float(bank[i, f])) ** 2) for f in range(4))
                       for i in range(N)] for j in range(len(y))])
        eps = float(np.median(D))
        c = O.OracleContext([dict(kind="2TCM_REV", n_draws=N, lo=LO_FDG, hi=HI_FDG)], n_accept=n, seed=9,
                            distance=dist, accept=mode, epsilon=eps)
        c.set_input_function("FENG", FENG)
        c.set_frames(st, du, w)
        r = c.run_voxels(y)
        for j in range(len(y)):
            if mode == "TOPN":
                order = sorted(range(N), key=lambda i: (D[j, i], i))[:n]
                assert list(r["acc_idx"][j]) == order
                np.testing.assert_allclose(r["acc_dist"][j], D[j, order], rtol=1e-15)
            else:
                acc = [i for i in range(N) if D[j, i] <= eps]  # sequential rejection loop
                assert r["count"][j, 0] == len(acc)


def test_ties_go_to_lower_index_and_n_equals_N():
    """All draws identical (fixed prior) -> all D equal -> accepted = indices 0..n-1."""
    fixed = [0.2, 0.4, 0.1, 0.01, 0.05]
    c = ctx_fdg(N=50, lo=fixed, hi=fixed, n_accept=7)
    st, du = fdg22()
    y = np.float32(c.simulate("2TCM_REV", fixed) * 1.01)[None, :]
    r = c.run_voxels(y)
    assert list(r["acc_idx"][0]) == list(range(7))
    c2 = ctx_fdg(N=20, n_accept=20)
    r2 = c2.run_voxels(y)
    assert sorted(r2["acc_idx"][0]) == list(range(20))
    assert np.all(np.diff(r2["acc_dist"][0]) >= 0)


def test_monotone_refinement_and_probabilities():
    """Smaller n -> subset; probabilities are multiples of 1/n and sum to 1."""
    lo = LO_FDG
    c = O.OracleContext([dict(kind="2TCM_IRR", n_draws=300, lo=lo, hi=HI_FDG),
                         dict(kind="2TCM_REV", n_draws=300, lo=lo, hi=HI_FDG)], n_accept=40)
    c.set_input_function("FENG", FENG)
    st, du = fdg22()
    c.set_frames(st, du)
    y = np.float32(c.simulate("2TCM_REV", (0.3, 0.5, 0.1, 0.02, 0.05)))[None, :] * np.float32(1.03)
    r40 = c.run_voxels(y)
    c10 = O.OracleContext(c.models, n_accept=10)
    c10.set_input_function("FENG", FENG)
    c10.set_frames(st, du)
    r10 = c10.run_voxels(y)
    assert set(r10["acc_idx"][0]) <= set(r40["acc_idx"][0])
    assert list(r10["acc_idx"][0]) == list(r40["acc_idx"][0][:10])
    p = r40["prob"][0]
    assert abs(float(p.sum()) - 1) < 1e-6 and all(abs(x * 40 - round(x * 40)) < 1e-4 for x in p)
    assert r40["count"][0].sum() == 40


def test_model_probability_worked_example():
    """n=18 with 10 draws of model 1 -> P(m=1) = 10/18, preferred = 1."""
    g = GOLD["model_probability"]
    ta = [0.2, 0.4, 0.1, 0.0, 0.05]
    tb = [0.6, 0.9, 0.2, 0.05, 0.1]
    c = O.OracleContext([dict(kind="2TCM_IRR", n_draws=8, lo=ta, hi=ta),
                         dict(kind="2TCM_REV", n_draws=100, lo=tb, hi=tb)], n_accept=g["n"])
    c.set_input_function("FENG", FENG)
    st, du = fdg22()
    c.set_frames(st, du)
    y = np.float32(c.simulate("2TCM_IRR", ta))[None, :]   # model-0 draws have D = 0
    r = c.run_voxels(y)
    assert list(r["count"][0]) == [8, 10]
    assert r["prob"][0, 1] == pytest.approx(g["expected_prob1"], abs=1e-7)
    assert r["preferred"][0] == g["preferred"]
    assert list(r["acc_idx"][0]) == list(range(8)) + list(range(8, 18))


def test_preferred_tie_goes_to_model0():
    ta = [0.2, 0.4, 0.1, 0.0, 0.05]
    tb = [0.6, 0.9, 0.2, 0.05, 0.1]
    c = O.OracleContext([dict(kind="2TCM_IRR", n_draws=9, lo=ta, hi=ta),
                         dict(kind="2TCM_REV", n_draws=100, lo=tb, hi=tb)], n_accept=18)
    c.set_input_function("FENG", FENG)
    st, du = fdg22()
    c.set_frames(st, du)
    r = c.run_voxels(np.float32(c.simulate("2TCM_IRR", ta))[None, :])
    assert list(r["count"][0]) == [9, 9] and r["preferred"][0] == 0


def test_quantile_and_ki_worked_examples():
    g = GOLD["quantile_type7"]
    for q, e in zip(g["q"], g["expected"]):
        assert O.quantile7(np.array(g["x"], float), q) == pytest.approx(e, abs=1e-12)
    k = GOLD["ki"]
    fixed = [k["K1"], k["k2"], k["k3"], 0.0, 0.05]
    c = ctx_fdg(kind="2TCM_IRR", N=30, lo=fixed, hi=fixed, n_accept=10)
    r = c.run_voxels(np.float32(c.simulate("2TCM_IRR", fixed))[None, :])
    assert r["ki_mean"][0] == pytest.approx(k["expected"], rel=1e-6)
    assert r["ki_sd"][0] < 1e-12  # identical draws (two-pass variance of a constant)
    np.testing.assert_allclose(r["ki_q"][0], r["ki_mean"][0], rtol=1e-6)


def test_summaries_equal_numpy_over_accepted_draws():
    """Conditional mean / SD (ddof=1) / type-7 quantiles of the accepted draws
    recomputed with numpy (method='linear' == type 7) from the oracle's own acc_idx."""
    lo = LO_FDG
    c = O.OracleContext([dict(kind="2TCM_IRR", n_draws=400, lo=lo, hi=HI_FDG),
                         dict(kind="2TCM_REV", n_draws=400, lo=lo, hi=HI_FDG)], n_accept=60)
    c.set_input_function("FENG", FENG)
    st, du = fdg22()
    c.set_frames(st, du)
    y = np.float32(c.simulate("2TCM_REV", (0.3, 0.5, 0.1, 0.02, 0.05)))[None, :] * np.float32(0.97)
    r = c.run_voxels(y)
    pref = r["preferred"][0]
    ths = [c.draw(int(i)) for i in r["acc_idx"][0]]
    sel = np.array([th for m, th in ths if m == pref], dtype=np.float64)
    np.testing.assert_allclose(r["mean"][0], sel.mean(0).astype(np.float32), rtol=1e-6)
    np.testing.assert_allclose(r["sd"][0], sel.std(0, ddof=1).astype(np.float32), rtol=1e-5, atol=1e-12)
    qs = np.quantile(sel, [0.025, 0.5, 0.975], axis=0, method="linear").T
    np.testing.assert_allclose(r["q"][0], qs.astype(np.float32), rtol=1e-6)
    ki = sel[:, 0] * sel[:, 2] / (sel[:, 1] + sel[:, 2])
    assert r["ki_mean"][0] == pytest.approx(ki.mean(), rel=1e-6)


def test_eps_infinity_recovers_prior_moments():
    """eps -> inf accepts every draw: posterior = prior sample; mean ~ (lo+hi)/2 within
    4 sigma/sqrt(N), SD ~ (hi-lo)/sqrt(12); exactly the sample moments of the same draws."""
    N = 20000
    c = ctx_fdg(kind="2TCM_REV", N=N, accept="EPS", epsilon=1e300)
    y = np.float32(c.simulate("2TCM_REV", (0.3, 0.5, 0.1, 0.02, 0.05)))[None, :]
    r = c.run_voxels(y)
    assert r["count"][0, 0] == N
    th = np.array([c.draw(i)[1] for i in range(N)], dtype=np.float64)
    np.testing.assert_allclose(r["mean"][0], th.mean(0).astype(np.float32), rtol=1e-6)
    lo, hi = np.array(LO_FDG), np.array(HI_FDG)
    sig = (hi - lo) / math.sqrt(12)
    assert np.all(np.abs(r["mean"][0] - (lo + hi) / 2) < 4 * sig / math.sqrt(N))
    np.testing.assert_allclose(r["sd"][0], sig, rtol=0.02)
    assert np.all(np.isnan(r["q"][0]))


def test_eps_zero_concentrates_on_truth():
    """eps -> 0 / top-1 with a noise-free TAC that is a bank member: accepts exactly that draw with
    D = 0.  For theta_true outside the bank, |mean - truth| shrinks as N grows (fixed n)."""
    c = ctx_fdg(N=500, n_accept=1)
    bank = c.bank()
    y = bank[[17, 333]]
    r = c.run_voxels(y)
    assert list(r["acc_idx"][:, 0]) == [17, 333] and np.all(r["acc_dist"][:, 0] == 0.0)
    ce = ctx_fdg(N=500, accept="EPS", epsilon=0.0)
    re_ = ce.run_voxels(y)
    assert list(re_["count"][:, 0]) == [1, 1]
    truth = np.float32([0.4, 0.6, 0.12, 0.03, 0.08])
    yt = np.float32(c.simulate("2TCM_REV", truth))[None, :]
    errs = []
    for N in (500, 5000, 50000):
        cn = ctx_fdg(N=N, n_accept=5, seed=11)
        rn = cn.run_voxels(yt)
        errs.append(float(np.abs(rn["ki_mean"][0] - truth[0] * truth[2] / (truth[1] + truth[2]))))
    assert errs[2] < errs[0]


def test_validation_errors():
    with pytest.raises(O.OracleError):
        O.OracleContext([dict(kind="2TCM_REV", n_draws=10, lo=LO_FDG, hi=HI_FDG)], n_accept=11)
    with pytest.raises(O.OracleError):
        O.OracleContext([dict(kind="2TCM_REV", n_draws=10, lo=LO_FDG, hi=HI_FDG)], n_accept=0)
    c = O.OracleContext([dict(kind="2TCM_REV", n_draws=10, lo=LO_FDG, hi=HI_FDG)], n_accept=2)
    with pytest.raises(O.OracleError):
        c.run_voxels(np.zeros((1, 22), np.float32))  # state: nothing set
    with pytest.raises(O.OracleError):
        c.set_frames([0.0, 0.5], [1.0, 1.0])  # overlap
    with pytest.raises(O.OracleError):
        c.set_input_function("PWL", [0.0, 1.0], t=[0.5, 1.0])  # t0 != 0
