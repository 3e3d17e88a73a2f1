"""Element-by-element oracle parity at BASELINE.json's full sizes, in bench.py's launch
configuration (VERDICT r01 "next" item 1).

* Config 4: the CUDA path runs the WHOLE total-body volume (4,441,800 voxels, N = 1e7, n = 18,
  M = 2, L = 35) in one abc_run_voxels call -- exactly the per-rank call bench.py times at one GPU
  -- and the FP64 CPU oracle re-runs 256 voxels stratified over the 9 tissue classes at the same
  N = 1e7.  Accepted index sets must be bit-exact outside the 1e-6 boundary band, moments within
  1e-4, probabilities within 1e-3 (tests/parity.compare, which also checks the (#swaps)/n bound on
  boundary-exempt voxels).  At this size the hyper-tile level of the FP32 pass has hs = 26
  super-tiles and ~1,500 hyper-tiles, so every tree level is exercised.
* Config 3: three whole brain slices (49,152 voxels, every class incl. the activated striatum),
  MRTM vs lp-ntPET, L = 90, N = 1e6, n = 100; the oracle re-runs 96 voxels stratified over the
  6 classes.
The oracle needs roughly 1-3 minutes of the box's host cores for each.
"""
import numpy as np
import pytest

import synthetic as S
from tests.parity import compare

pytestmark = pytest.mark.gpu


def _stratified(labels, total, seed):
    rng = np.random.default_rng(seed)
    classes = np.unique(labels)
    per = int(np.ceil(total / len(classes)))
    idx = [rng.choice(np.flatnonzero(labels == c), min(per, int(np.sum(labels == c))), replace=False)
           for c in classes]
    return np.sort(np.concatenate(idx))


def _oracle(problem, tacs):
    from oracle import oracle as O
    o = O.OracleContext(**problem.ctx_kwargs)
    problem.setup(o)
    return o.run_voxels(tacs)


@pytest.fixture(scope="module")
def tb_volume():
    import torch
    from paper_2603_14859_b200 import FLAG_TIMING, AbcContext
    p = S.config4_chunk(chunk=0, n_chunks=1, N=10_000_000, n=18, device="cuda")
    assert p.J == 4_441_800
    ctx = AbcContext(**dict(p.ctx_kwargs, flags=FLAG_TIMING))
    p.setup(ctx)
    y = torch.from_numpy(p.tacs).cuda()
    g = {k: v.cpu().numpy() for k, v in ctx.run_voxels(y).items()}
    g["count"] = g["count"].view(np.uint32)
    g["acc_idx"] = g["acc_idx"].view(np.uint64)
    st = ctx.stats()
    del y, ctx
    torch.cuda.empty_cache()
    return p, g, st


def test_tb_whole_volume_stratified_oracle_parity(tb_volume):
    p, g, st = tb_volume
    assert st["n_voxels"] == p.J and st["n_draws"] == 10_000_000
    idx = _stratified(p.truth["label"], 256, 20261019)
    assert len(idx) >= 256 and len(np.unique(p.truth["label"][idx])) == 9
    o = _oracle(p, p.tacs[idx])
    rep = compare({k: v[idx] for k, v in g.items()}, o)
    assert rep["matched"] >= len(idx) - 3, rep


def test_tb_whole_volume_sanity(tb_volume):
    """Every voxel: probabilities are multiples of 1/n summing to 1, accepted lists sorted
    by (D, i), K_i finite for 2TCM voxels, and no voxel needed the exact fallback."""
    p, g, st = tb_volume
    n = p.ctx_kwargs["n_accept"]
    np.testing.assert_allclose(g["prob"].sum(1), 1.0, atol=1e-6)
    assert np.array_equal(g["count"].sum(1), np.full(p.J, n, dtype=np.uint32))
    d = g["acc_dist"]
    assert np.all(np.diff(d, axis=1) >= 0)
    assert np.all(np.isfinite(g["ki_mean"]))
    assert st["n_fallback"] <= p.J // 10000


@pytest.fixture(scope="module")
def brain_slices():
    from paper_2603_14859_b200 import AbcContext
    p = S.config3(slices=(10, 33, 35), N=1_000_000, n=100, device="cuda")
    ctx = AbcContext(**p.ctx_kwargs)
    p.setup(ctx)
    g = ctx.run_voxels(p.tacs)
    return p, g


def test_brain_slices_stratified_oracle_parity(brain_slices):
    p, g = brain_slices
    idx = _stratified(p.truth["label"], 96, 7)
    assert len(np.unique(p.truth["label"][idx])) == 6 and len(idx) >= 96
    o = _oracle(p, p.tacs[idx])
    rep = compare({k: v[idx] for k, v in g.items()}, o)
    assert rep["matched"] >= len(idx) - 2, rep
    # the activated striatum is the lp-ntPET class (qualitative)
    act = p.truth["label"] == 5
    assert np.mean(g["prob"][act, 1] > 0.5) > 0.8


def test_continuous_phantom_fullN_oracle_parity():
    """Harder data at the full draw budget: the continuous-parameter TB phantom at double noise
    (ell = 14), the 283,800 voxels of the slab set z = 0 mod 16 run through the GPU path at
    N = 1e7 (every tree level active, the slowest case of profiles/r02_hard_phantoms.json), and the
    oracle re-runs 64 of them."""
    import torch
    from paper_2603_14859_b200 import AbcContext
    p = S.config4_continuous(chunk=0, n_chunks=16, N=10_000_000, n=18, ell=14.0, device="cuda")
    ctx = AbcContext(**p.ctx_kwargs)
    p.setup(ctx)
    g = {k: v.cpu().numpy() for k, v in ctx.run_voxels(torch.from_numpy(p.tacs).cuda()).items()}
    g["count"] = g["count"].view(np.uint32)
    g["acc_idx"] = g["acc_idx"].view(np.uint64)
    del ctx
    idx = np.sort(np.random.default_rng(11).choice(p.J, 64, replace=False))
    o = _oracle(p, p.tacs[idx])
    rep = compare({k: v[idx] for k, v in g.items()}, o)
    assert rep["matched"] >= len(idx) - 2, rep


def test_host_outputs_chunked_copy_equal_device_outputs():
    """Host output buffers of >= 2^18 voxels are reduced in chunks whose device-to-host copies
    overlap the next chunk (api.cu): byte-identical to device outputs of the same call."""
    import torch
    from paper_2603_14859_b200 import AbcContext
    p = S.config4_chunk(chunk=3, n_chunks=16, N=1_000_000, n=18)
    assert p.J >= (1 << 18)
    ctx = AbcContext(**p.ctx_kwargs)
    p.setup(ctx)
    host = ctx.run_voxels(p.tacs)  # numpy in -> numpy out (host outputs, chunked copies)
    dev = ctx.run_voxels(torch.from_numpy(p.tacs).cuda())
    for k, v in host.items():
        np.testing.assert_array_equal(np.nan_to_num(v), np.nan_to_num(dev[k].cpu().numpy().view(v.dtype)), err_msg=k)
