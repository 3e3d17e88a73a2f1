"""GPU parity of the response-function credible envelope (abc_response_envelope; Fig. 1;
SURVEY §8f-4) against the oracle, on config-2-shaped lp-ntPET vs MRTM problems."""
import numpy as np
import pytest

import synthetic as S
from paper_2603_14859_b200 import AbcError
from tests.parity import run_gpu, run_oracle

pytestmark = pytest.mark.gpu

T_GRID = np.concatenate([np.linspace(0.0, 60.0, 121), [14.999, 30.0, 45.0, 90.0]])


@pytest.fixture(scope="module")
def rt():
    p = S.config2(J=120, N_per_model=4000, n=40, noise="mid")
    g, gc = run_gpu(p)
    o, oc = run_oracle(p)
    return p, g, gc, o, oc


def test_envelope_matches_oracle_on_common_accepted_sets(rt):
    p, g, gc, o, oc = rt
    qo = oc.response_envelope(o["acc_idx"], T_GRID)
    qg = gc.response_envelope(o["acc_idx"], T_GRID)  # same input lists: isolates the envelope kernel
    assert np.array_equal(np.isnan(qg), np.isnan(qo))
    m = ~np.isnan(qo)
    np.testing.assert_allclose(qg[m], qo[m], rtol=1e-6, atol=0)
    assert np.all(qg[m].reshape(-1, 3)[:, 0] <= qg[m].reshape(-1, 3)[:, 2])


def test_envelope_end_to_end_and_device_pointers(rt):
    import torch
    p, g, gc, o, oc = rt
    same = np.all(g["acc_idx"] == o["acc_idx"], axis=1)
    assert same.mean() > 0.9
    qg = gc.response_envelope(g["acc_idx"], T_GRID)
    qo = oc.response_envelope(o["acc_idx"], T_GRID)
    np.testing.assert_allclose(qg[same], qo[same], rtol=1e-6, atol=0)
    qd = gc.response_envelope(torch.from_numpy(g["acc_idx"].astype(np.int64)).cuda(), T_GRID)
    np.testing.assert_array_equal(qd.cpu().numpy(), qg)


def test_envelope_errors(rt):
    p, g, gc, o, oc = rt
    bad = o["acc_idx"][:2].copy()
    bad[1, 3] = gc.N + 5
    with pytest.raises(AbcError) as e:
        gc.response_envelope(bad, T_GRID)
    assert e.value.status == 1
