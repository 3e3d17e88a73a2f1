"""GPU parity of the Patlak K_i map (abc_patlak; P:282's clinical reference, DESIGN.md
R18) against the oracle on config-4 (PWL IDIF) and config-1 (Feng input) voxels."""
import numpy as np
import pytest

import synthetic as S
from tests.parity import run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("which", ["tb", "cfg1"])
def test_patlak_matches_oracle(which):
    if which == "tb":
        p = S.config4_chunk(chunk=11, n_chunks=64, N=2000, n=5, max_voxels=5000)
    else:
        p = S.config1(J=64, N=2000)
    from paper_2603_14859_b200 import AbcContext
    from oracle import oracle as O
    g = AbcContext(**p.ctx_kwargs)
    p.setup(g)
    kw = dict(p.ctx_kwargs)
    kw.pop("flags", None)
    o = O.OracleContext(**kw)
    p.setup(o)
    for t_star in (10.0, 20.0):
        kg, vg = g.patlak(p.tacs, t_star)
        ko, vo = o.patlak(p.tacs, t_star)
        assert np.all(np.isfinite(kg))
        scale_k = np.max(np.abs(ko))
        np.testing.assert_allclose(kg, ko, rtol=1e-6, atol=1e-9 * scale_k)
        np.testing.assert_allclose(vg, vo, rtol=1e-6, atol=1e-9 * np.max(np.abs(vo)))
    # device pointers
    import torch
    kd, vd = g.patlak(torch.from_numpy(np.ascontiguousarray(p.tacs)).cuda(), 20.0)
    np.testing.assert_array_equal(kd.cpu().numpy(), g.patlak(p.tacs, 20.0)[0])
    # degenerate: no late frame -> NaN
    kn, _ = g.patlak(p.tacs[:3], 1e6)
    assert np.all(np.isnan(kn))


def test_patlak_tracks_true_ki_on_irreversible_voxels():
    """On the TB phantom, the Patlak slope follows the true K_i of irreversible voxels (sanity)."""
    p = S.config4_chunk(chunk=13, n_chunks=64, N=2000, n=5, max_voxels=4000)
    from paper_2603_14859_b200 import AbcContext
    g = AbcContext(**p.ctx_kwargs)
    p.setup(g)
    th = p.truth["theta"]
    irr = th[:, 3] == 0
    ki_true = th[:, 0] * th[:, 2] / (th[:, 1] + th[:, 2])
    kg, _ = g.patlak(p.tacs, 20.0)
    r = np.corrcoef(kg[irr], ki_true[irr])[0, 1]
    assert r > 0.9, r
