"""Parity at BASELINE.json's full size, in bench.py's launch configuration: the config-4 batch
(145,200 TB-phantom voxels, N = 1e7 draws, n = 18, M = 2, L = 35).  The oracle cannot score
1e7 x 145k pairs, so sampled outputs are checked one by one with the oracle's own draws and
simulation (no value comes from the CUDA path):
  * every accepted draw's FP64 discrepancy equals the oracle's for that draw (sampled voxels);
  * no draw of a random 20,000-draw sample beats the n-th accepted discrepancy (top-n property);
  * model counts / probabilities / means / SDs / quantiles / K_i equal the summaries the oracle
    computes from the accepted draws.
"""
import numpy as np
import pytest

import synthetic as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def full():
    from paper_2603_14859_b200 import AbcContext
    p = S.config4_chunk(chunk=0, n_chunks=32, N=10_000_000, n=18, device="cuda")
    ctx = AbcContext(**dict(p.ctx_kwargs, flags=1))
    p.setup(ctx)
    g = ctx.run_voxels(p.tacs)
    return p, g, ctx.stats()


def _oracle(p):
    from oracle import oracle as O
    o = O.OracleContext(**p.ctx_kwargs)
    p.setup(o)
    return O, o


def test_fullsize_accepted_distances_and_topn_property(full):
    p, g, st = full
    O, o = _oracle(p)
    rng = np.random.default_rng(20261018)
    J, n = p.J, p.ctx_kwargs["n_accept"]
    sample = rng.choice(J, 6, replace=False)
    kinds = [m["kind"] for m in p.ctx_kwargs["models"]]
    cache = {}

    def curve(i):
        if i not in cache:
            m, th = o.draw(int(i))
            cache[i] = o.simulate(kinds[m], th).astype(np.float32)
        return cache[i]

    w = p.weight
    for j in sample:
        for a in range(n):
            i = int(g["acc_idx"][j, a])
            d = O.distance("WL2", p.tacs[j], curve(i), w)
            assert d == pytest.approx(float(g["acc_dist"][j, a]), rel=1e-9), (j, a, i)
        assert np.all(np.diff(g["acc_dist"][j]) >= 0)
    N = o.N
    probe = rng.choice(N, 20_000, replace=False)
    for i in probe:
        s = curve(int(i))
        for j in sample:
            tau = float(g["acc_dist"][j, n - 1])
            d = O.distance("WL2", p.tacs[j], s, w)
            assert d > tau or int(i) in set(g["acc_idx"][j].tolist()) or d == tau, (j, int(i), d, tau)
    assert st["n_voxels"] == J and st["n_draws"] == N


def test_fullsize_summaries_from_accepted_draws(full):
    p, g, _ = full
    O, o = _oracle(p)
    rng = np.random.default_rng(5)
    for j in rng.choice(p.J, 20, replace=False):
        ths = [o.draw(int(i)) for i in g["acc_idx"][j]]
        ms = np.array([m for m, _ in ths])
        cnt = np.bincount(ms, minlength=2)
        assert list(g["count"][j]) == list(cnt)
        np.testing.assert_allclose(g["prob"][j], cnt / cnt.sum(), atol=1e-7)
        pref = int(np.argmax(cnt))  # ties -> model 0 (R10)
        assert g["preferred"][j] == pref
        sel = np.array([th for m, th in ths if m == pref], dtype=np.float64)
        np.testing.assert_allclose(g["mean"][j], sel.mean(0), rtol=1e-5, atol=1e-12)
        if len(sel) >= 2:
            np.testing.assert_allclose(g["sd"][j], sel.std(0, ddof=1), rtol=1e-4, atol=1e-9)
        q = np.quantile(sel, [0.025, 0.5, 0.975], axis=0, method="linear").T
        np.testing.assert_allclose(g["q"][j], q, rtol=1e-5, atol=1e-12)
        ki = sel[:, 0] * sel[:, 2] / (sel[:, 1] + sel[:, 2])
        assert g["ki_mean"][j] == pytest.approx(ki.mean(), rel=1e-5)
