"""GPU parity with simulated-draw noise enabled (abc_set_sim_noise; SURVEY §8f-3, P:218-220 model on
the draws, R17): the noisy bank equals the oracle's up to rare 1-ulp RN32 flips (FP64
log/sin/cos/exp last-ulp differences), and the whole path matches the oracle element by element."""
import numpy as np
import pytest

import synthetic as S
from paper_2603_14859_b200 import AbcContext
from oracle import oracle as O
from tests.parity import compare

pytestmark = pytest.mark.gpu


def pair(problem, ell, thalf):
    g = AbcContext(**problem.ctx_kwargs)
    problem.setup(g)
    g.set_sim_noise(ell, thalf)
    kw = dict(problem.ctx_kwargs)
    kw.pop("flags", None)
    o = O.OracleContext(**kw)
    problem.setup(o)
    o.set_sim_noise(ell, thalf)
    return g, o


@pytest.mark.parametrize("which", ["cfg1", "tb", "rt"])
def test_noisy_bank_matches_oracle(which):
    if which == "cfg1":
        p, ell, th = S.config1(J=4, N=3000), 7.0, 109.8
    elif which == "tb":
        p, ell, th = S.config4_chunk(chunk=3, n_chunks=64, N=3000, n=5, max_voxels=4), 7.0, 109.8
    else:
        p, ell, th = S.config2(J=4, N_per_model=1500, n=5, noise="mid"), 2.0, 20.4
    g, o = pair(p, ell, th)
    g.run_voxels(p.tacs[:4])
    gb, ob = g.bank(), o.bank()
    diff = gb != ob
    assert diff.mean() < 1e-4, int(diff.sum())
    np.testing.assert_allclose(gb, ob, rtol=2.5e-7, atol=0)
    # and the noise is really there
    g0 = AbcContext(**p.ctx_kwargs)
    p.setup(g0)
    g0.run_voxels(p.tacs[:4])
    assert np.mean(g0.bank() != gb) > 0.5


def test_noisy_run_parity_config1_and_tb():
    for p, ell in [(S.config1(J=48, N=10_000), 7.0),
                   (S.config4_chunk(chunk=9, n_chunks=64, N=30_011, n=18, max_voxels=300), 7.0)]:
        g, o = pair(p, ell, 109.8)
        rg = g.run_voxels(p.tacs)
        ro = o.run_voxels(p.tacs)
        rep = compare(rg, ro)
        assert rep["matched"] >= p.J - 2


def test_zero_noise_is_identity():
    p = S.config1(J=16, N=4000)
    g = AbcContext(**p.ctx_kwargs)
    p.setup(g)
    a = g.run_voxels(p.tacs)
    g.set_sim_noise(0.0, 109.8)
    b = g.run_voxels(p.tacs)
    for k in a:
        np.testing.assert_array_equal(np.nan_to_num(a[k]), np.nan_to_num(b[k]), err_msg=k)
