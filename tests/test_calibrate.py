"""Host-side statistics of the pilot calibration: pinned against brute force and
closed forms (no GPU)."""
import numpy as np

from paper_2603_14859_b200 import calibrate as CAL


def test_roc_auc_equals_brute_force_pairs():
    rng = np.random.default_rng(3)
    for _ in range(5):
        s = np.round(rng.random(60), 1)  # many ties
        y = rng.random(60) < 0.4
        pos, neg = s[y], s[~y]
        brute = np.mean([(a > b) + 0.5 * (a == b) for a in pos for b in neg])
        assert abs(CAL.roc_auc(s, y) - brute) < 1e-12
    assert CAL.roc_auc([1, 2, 3, 4], [False, False, True, True]) == 1.0
    assert CAL.roc_auc([4, 3, 2, 1], [False, False, True, True]) == 0.0


def test_fit_u_curve_recovers_the_minimum_of_a_quadratic_in_log_n():
    ns = np.array([1, 2, 3, 5, 8, 12, 18, 27, 40, 60, 90])
    x = np.log(ns)
    mse = 2.0 + 0.5 * (x - np.log(7.0)) ** 2
    fit = CAL.fit_u_curve(ns, mse)
    assert fit["u_shaped"] and abs(fit["n_opt"] - 7.0) < 1e-9
    # concave decreasing curve: no interior minimum -> the best grid point
    fit2 = CAL.fit_u_curve(ns, 10.0 - x - 0.05 * x * x)
    assert not fit2["u_shaped"] and fit2["n_opt"] == 90


def test_mse_curve_and_sens_spec():
    truth = np.array([1.0, 2.0, 3.0, 4.0])
    ns, mse = CAL.mse_curve({5: truth + 1.0, 2: truth, 9: truth - 2.0}, truth)
    assert list(ns) == [2, 5, 9] and list(mse) == [0.0, 1.0, 4.0]
    sens, spec = CAL.sens_spec([0.9, 0.4, 0.6, 0.1], [True, True, False, False])
    assert sens == 0.5 and spec == 0.5


def test_epsilon_from_pilot_is_the_quantile_of_the_nth_distance():
    d = np.sort(np.random.default_rng(1).random((101, 20)), axis=1)
    eps = CAL.epsilon_from_pilot(d, 7, q=0.5)
    assert eps == np.median(d[:, 6])
    # a voxel accepts >= 7 draws under D <= eps iff its 7th smallest D <= eps: half of them (+ the median one)
    assert np.sum(d[:, 6] <= eps) == 51
