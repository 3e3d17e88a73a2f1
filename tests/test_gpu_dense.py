"""GPU parity of the optional dense shared-bank tensor-core distance (ABC_FLAG_DENSE_TC, K6 in
dense_tc.cu; north star "shared-simulation-bank mode"): the y.s cross term on
tcgen05 (BF16 x 3 split), certified in FP64 with the dot-form error bound, must give the oracle's
results -- and the default pruned FP32 path's results bit for bit -- with few or no voxels sent
to the exact FP64 fallback."""
import numpy as np
import pytest

import synthetic as S
from paper_2603_14859_b200 import FLAG_DENSE_TC, AbcError
from tests.parity import compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tb_small():
    # config-4-shaped: 700 voxels (5 blocks of 128 + a ragged 60), N = 40,077 (156 tiles of 256 + 141)
    return S.config4_chunk(chunk=7, n_chunks=64, N=40_077, n=18, max_voxels=700)


def test_dense_tc_matches_oracle_tb(tb_small):
    g, gc = run_gpu(tb_small, flags=FLAG_DENSE_TC | 1)
    o, _ = run_oracle(tb_small)
    rep = compare(g, o)
    st = gc.stats()
    assert rep["matched"] >= tb_small.J - 2
    # the tensor-core pass must do the work: certification rarely needs the exact FP64 rescan
    assert st["n_fallback"] <= 0.02 * tb_small.J, st["n_fallback"]


def test_dense_tc_identical_to_fp32_path(tb_small):
    sub = tb_small.subset(np.arange(300))
    base, _ = run_gpu(sub)
    alt, _ = run_gpu(sub, flags=FLAG_DENSE_TC)
    for k in base:
        np.testing.assert_array_equal(np.nan_to_num(base[k]), np.nan_to_num(alt[k]), err_msg=k)


def test_dense_tc_config1_feng():
    """Config 1 (22 frames, Feng input, one model, n = 100 of N = 1e4 + ragged tail)."""
    p = S.config1(J=64, N=10_000)
    g, gc = run_gpu(p, flags=FLAG_DENSE_TC)
    o, _ = run_oracle(p)
    compare(g, o)
    assert gc.stats()["n_fallback"] <= 2


def test_dense_tc_tiny_and_degenerate():
    """N smaller than one draw tile, J smaller than one voxel block, n = N (everything accepted)."""
    p = S.config1(J=5, N=100, p=1.0)
    g, _ = run_gpu(p, flags=FLAG_DENSE_TC)
    o, _ = run_oracle(p)
    compare(g, o)
    p2 = S.config1(J=3, N=300, p=0.01)
    g2, _ = run_gpu(p2, flags=FLAG_DENSE_TC)
    o2, _ = run_oracle(p2)
    compare(g2, o2)


def test_dense_tc_unsupported():
    """L1 distance and eps acceptance have no dot form: ABC_E_UNSUPPORTED (5)."""
    for kw in (dict(distance="L1"), dict(accept="EPS", epsilon=1.0)):
        p = S.config1(J=4, N=500).replace(**kw)
        with pytest.raises(AbcError) as e:
            run_gpu(p, flags=FLAG_DENSE_TC)
        assert e.value.status == 5
