"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element, on
seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs)."""
import numpy as np
import pytest

import synthetic as S
from tests.parity import compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg1():
    return S.config1()


@pytest.fixture(scope="module")
def tb_small():
    # config-4-shaped: TB phantom voxels, PWL IDIF, 35 frames, IRR vs REV, n = 18
    return S.config4_chunk(chunk=7, n_chunks=64, N=40_000, n=18, max_voxels=700)


@pytest.fixture(params=[False, True], ids=["auto", "rotated"])
def rot(request, monkeypatch):
    """Run a test with the library's automatic choice of scan basis (small problems keep the frame
    basis) and with the rotated eigenbasis forced (the bench volume's path)."""
    if request.param:
        monkeypatch.setenv("VPET_ROT_ALWAYS", "1")
    return request.param


@pytest.fixture(scope="module")
def rt_small():
    # config-2-shaped: lp-ntPET vs MRTM, 61 frames, PWL reference TAC
    return S.config2(J=96, N_per_model=4000, n=40, noise="mid")


@pytest.fixture(scope="module")
def brain_small():
    # config-3-shaped: brain phantom voxels of every class (incl. the activated striatum), 90 frames
    lab = np.concatenate([S.brain_geometry(z) for z in (10, 33, 35)])
    rng = np.random.default_rng(7)
    idx = np.sort(np.concatenate([rng.choice(np.flatnonzero(lab == c), 16, replace=False) for c in range(6)]))
    return S.config3(slices=(10, 33, 35), voxel_index=idx, N=8000, n=40)


def test_bank_matches_oracle_rn32(cfg1, tb_small, rt_small):
    """Alg.1 l.3: the GPU bank equals the oracle's RN32 frame averages (rare 1-ulp flips of
    values within FP64 rounding of an FP32 tie are allowed)."""
    for prob in (cfg1, tb_small, rt_small):
        small = prob.replace(models=[dict(m, n_draws=min(int(m["n_draws"]), 3000)) for m in prob.ctx_kwargs["models"]],
                             n_accept=5)
        _, g = run_gpu(small, tacs=small.tacs[:4])
        _, o = run_oracle(small, tacs=small.tacs[:4])
        gb, ob = g.bank(), o.bank()
        diff = gb != ob
        assert diff.mean() < 1e-4, (prob.name, int(diff.sum()))
        np.testing.assert_allclose(gb, ob, rtol=2.5e-7, atol=0)


def test_config1_topn_wl2(cfg1, rot):
    g, gc = run_gpu(cfg1, flags=1)
    o, _ = run_oracle(cfg1)
    rep = compare(g, o)
    assert rep["matched"] >= cfg1.J - 1
    st = gc.stats()
    assert st["gpu_launches"] >= 5 and st["n_voxels"] == cfg1.J


@pytest.mark.parametrize("distance", ["L1", "WL2"])
@pytest.mark.parametrize("weighted", [True, False])
def test_config1_distances_and_weights(cfg1, distance, weighted, rot):
    p = cfg1.replace(distance=distance)
    if not weighted:
        import dataclasses
        p = dataclasses.replace(p, weight=None)
    g, _ = run_gpu(p)
    o, _ = run_oracle(p)
    compare(g, o)


def test_tb_model_selection(tb_small, rot):
    g, gc = run_gpu(tb_small)
    o, _ = run_oracle(tb_small)
    rep = compare(g, o)
    assert rep["matched"] >= tb_small.J - 2


def test_rt_model_selection(rt_small):
    g, _ = run_gpu(rt_small)
    o, _ = run_oracle(rt_small)
    compare(g, o)


def test_brain_model_selection(brain_small, rot):
    """Config-3 shape: L = 90 (the widest frame count of the configs), MRTM vs lp-ntPET."""
    g, _ = run_gpu(brain_small)
    o, _ = run_oracle(brain_small)
    rep = compare(g, o)
    assert rep["matched"] >= brain_small.J - 2


@pytest.mark.parametrize("flags", [0x2, 0x8, 0x10, 0x8 | 0x10, 0x20, 0x20 | 0x8])
def test_exact_noprune_noreorder_notree_identical(tb_small, flags, rot):
    """ABC_FLAG_EXACT (pure FP64 scan), NO_PRUNE, NO_REORDER and NO_TREE (flat index-order scan) give
    bit-identical outputs to the default tree-ordered, bound-pruned FP32 pass."""
    sub = tb_small.subset(np.arange(130))
    base, _ = run_gpu(sub)
    alt, _ = run_gpu(sub, flags=flags)
    for k in base:
        np.testing.assert_array_equal(np.nan_to_num(base[k]), np.nan_to_num(alt[k]), err_msg=k)


def test_eps_mode(cfg1, rot):
    """eps mode: accept D <= eps; moments from streaming sums."""
    o_top, _ = run_oracle(cfg1)
    eps = float(np.median(o_top["acc_dist"][:, -1]))
    p = cfg1.replace(accept="EPS", epsilon=eps)
    g, _ = run_gpu(p)
    o, _ = run_oracle(p)
    assert np.array_equal(g["count"], o["count"])
    compare(g, o, topn=False)
    # eps -> inf accepts every draw: prior moments
    p2 = cfg1.replace(accept="EPS", epsilon=1e300)
    g2, _ = run_gpu(p2, tacs=cfg1.tacs[:3])
    o2, _ = run_oracle(p2, tacs=cfg1.tacs[:3])
    assert np.all(g2["count"] == 10_000)
    compare(g2, o2, topn=False)


def test_wide_schedule_lp128():
    """L = 100 frames: the widest scan layout (LP = 128, one voxel per thread), lp-ntPET vs MRTM."""
    p = S.config2(J=40, N_per_model=3000, n=25, noise="mid", n_frames=100)
    g, _ = run_gpu(p)
    o, _ = run_oracle(p)
    compare(g, o)


@pytest.mark.parametrize("N", [12345, 40_000 + 77])
def test_ragged_draw_counts(tb_small, N, rot):
    """N not a multiple of the tile / super-tile / hyper-tile sizes; fewer hyper-tiles than parts."""
    half = N // 2
    models = [dict(m, n_draws=(half if k == 0 else N - half)) for k, m in enumerate(tb_small.ctx_kwargs["models"])]
    p = tb_small.replace(models=models).subset(np.arange(150))
    g, _ = run_gpu(p)
    o, _ = run_oracle(p)
    compare(g, o)


def test_l1_tb_and_eps_rt(tb_small, rt_small):
    """L1 discrepancy on the TB shape; eps mode on the lp-ntPET / MRTM shape."""
    p = tb_small.replace(distance="L1").subset(np.arange(200))
    g, _ = run_gpu(p)
    o, _ = run_oracle(p)
    compare(g, o)
    o_top, _ = run_oracle(rt_small)
    eps = float(np.median(o_top["acc_dist"][:, -1]))
    q = rt_small.replace(accept="EPS", epsilon=eps)
    g, _ = run_gpu(q)
    o, _ = run_oracle(q)
    assert np.array_equal(g["count"], o["count"])
    compare(g, o, topn=False)


@pytest.mark.parametrize("J", [1, 31, 513, 1025])
def test_ragged_voxel_counts(tb_small, J):
    idx = np.arange(J) % tb_small.J
    sub = tb_small.subset(idx)
    g, _ = run_gpu(sub)
    o, _ = run_oracle(sub)
    compare(g, o)


@pytest.mark.parametrize("N,n", [(7, 3), (64, 64), (65, 1), (1000, 1000 // 8)])
def test_small_and_degenerate_budgets(cfg1, N, n):
    """N < tile, N = one tile, n = N (everything accepted), n = 1."""
    p = cfg1.replace(models=[dict(cfg1.ctx_kwargs["models"][0], n_draws=N)], n_accept=n)
    sub = p.subset(np.arange(40))
    g, _ = run_gpu(sub)
    o, _ = run_oracle(sub)
    compare(g, o)


def test_zero_voxels_and_errors(cfg1):
    from paper_2603_14859_b200 import AbcContext, AbcError
    ctx = AbcContext(**cfg1.ctx_kwargs)
    with pytest.raises(AbcError) as e:
        ctx.run_voxels(cfg1.tacs)
    assert e.value.status == 2  # state: nothing set
    cfg1.setup(ctx)
    r = ctx.run_voxels(np.zeros((0, cfg1.L), np.float32))
    assert r["prob"].shape == (0, 1)
    bad = cfg1.tacs[:4].copy()
    bad[2, 5] = np.nan
    with pytest.raises(AbcError) as e:
        ctx.run_voxels(bad)
    assert e.value.status == 1


def test_device_pointers_and_stream(tb_small):
    import torch
    from paper_2603_14859_b200 import AbcContext
    ctx = AbcContext(**tb_small.ctx_kwargs)
    tb_small.setup(ctx)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    y = torch.from_numpy(tb_small.tacs).cuda()
    with torch.cuda.stream(s):
        rd = ctx.run_voxels(y)
    torch.cuda.synchronize()
    ctx.set_stream(None)
    rh = ctx.run_voxels(tb_small.tacs)
    for k in rh:
        a = rd[k].cpu().numpy()
        b = rh[k]
        if b.dtype == np.uint64:
            a = a.astype(np.uint64)
        if b.dtype == np.uint32:
            a = a.astype(np.uint32)
        np.testing.assert_array_equal(np.nan_to_num(a), np.nan_to_num(b), err_msg=k)


def test_forced_fallback_equals_oracle_and_default(tb_small, rot):
    """ABC_FLAG_FORCE_FALLBACK sends every voxel through the uncertified-voxel path (the on-device
    list, the warp-parallel exact FP64 scan and the exact reduction): same results as the oracle
    and bit-identical to the certified FP32 path."""
    from paper_2603_14859_b200 import FLAG_FORCE_FALLBACK, FLAG_TIMING
    sub = tb_small.subset(np.arange(160))
    base, _ = run_gpu(sub)
    fb, ctx = run_gpu(sub, flags=FLAG_FORCE_FALLBACK | FLAG_TIMING)
    assert ctx.stats()["n_fallback"] == sub.J
    for k in base:
        np.testing.assert_array_equal(np.nan_to_num(base[k]), np.nan_to_num(fb[k]), err_msg=k)
    o, _ = run_oracle(sub)
    compare(fb, o)


def test_exact_ties_fixed_parameter_prior(tb_small, rot):
    """Exact D ties: model 0 has a fixed-parameter prior (lo == hi), so its whole
    block of draws simulates the same TAC; ties are resolved towards the lower draw index.  The
    fixed value is the truth of voxel 0, so the tied block fills voxel 0's accepted set."""
    th = tb_small.truth["theta"][0].astype(np.float32)
    lo, hi = S.priors_fdg()
    fixed = [float(v) for v in th]
    fixed[3] = 0.0
    models = [dict(kind="2TCM_IRR", n_draws=3000, lo=fixed, hi=fixed),
              dict(kind="2TCM_REV", n_draws=5000, lo=lo, hi=hi)]
    p = tb_small.replace(models=models).subset(np.arange(64))
    g, _ = run_gpu(p)
    o, _ = run_oracle(p)
    compare(g, o)
    # voxel 0: the oracle accepts the 18 lowest indices of the tied block; the GPU must pick the same
    # ones (compare() alone would allow swaps among draws tied exactly at the boundary)
    assert np.array_equal(o["acc_idx"][0], np.arange(18, dtype=np.uint64))
    assert np.array_equal(g["acc_idx"][0], o["acc_idx"][0])
    # every draw identical: the first n indices, D equal
    allfix = p.replace(models=[dict(kind="2TCM_IRR", n_draws=1000, lo=fixed, hi=fixed)], n_accept=7)
    g2, _ = run_gpu(allfix)
    o2, _ = run_oracle(allfix)
    assert np.array_equal(g2["acc_idx"], np.tile(np.arange(7, dtype=np.uint64), (p.J, 1)))
    compare(g2, o2)


def test_model_select_entry_point(tb_small):
    """abc_model_select (the north star's model-selection call) through the C ABI, host and device."""
    import torch
    from paper_2603_14859_b200 import AbcContext
    ctx = AbcContext(**tb_small.ctx_kwargs)
    tb_small.setup(ctx)
    full = ctx.run_voxels(tb_small.tacs)
    ms = ctx.model_select(tb_small.tacs)
    np.testing.assert_array_equal(ms["prob"], full["prob"])
    np.testing.assert_array_equal(ms["preferred"], full["preferred"])
    md = ctx.model_select(torch.from_numpy(tb_small.tacs).cuda())
    np.testing.assert_array_equal(md["prob"].cpu().numpy(), full["prob"])
    np.testing.assert_array_equal(md["preferred"].cpu().numpy(), full["preferred"])
    o, _ = run_oracle(tb_small)
    np.testing.assert_allclose(ms["prob"], o["prob"], atol=1e-3 + 1.0 / 18)


def test_nonfinite_voxel_returns_quickly(tb_small):
    """A NaN TAC value gives ABC_E_ARG without the work of an unprunable voxel (the kernels after
    the on-device finite check skip their work)."""
    import time
    from paper_2603_14859_b200 import AbcContext, AbcError
    models = [dict(m, n_draws=1_000_000) for m in tb_small.ctx_kwargs["models"]]
    p = tb_small.replace(models=models)
    ctx = AbcContext(**p.ctx_kwargs)
    p.setup(ctx)
    ctx.run_voxels(p.tacs)  # warm: buffers allocated
    t = time.perf_counter()
    ctx.run_voxels(p.tacs)
    t_ok = time.perf_counter() - t
    bad = p.tacs.copy()
    bad[5, 3] = np.nan
    t = time.perf_counter()
    with pytest.raises(AbcError) as e:
        ctx.run_voxels(bad)
    t_bad = time.perf_counter() - t
    assert e.value.status == 1
    assert t_bad < max(2.0 * t_ok, 0.2), (t_bad, t_ok)
    r = ctx.run_voxels(p.tacs)  # the context stays usable
    assert np.all(np.isfinite(r["ki_mean"]))


def test_truncation_equals_direct_runs(rt_small):
    """the summaries of the first n' entries of a top-n run's sorted accepted lists
    (abc_reduce_accepted) are those of a direct top-n' run, byte for byte (P:170-175 pilot sweep)."""
    import torch
    from paper_2603_14859_b200 import AbcContext
    big = rt_small.replace(n_accept=100)
    ctx = AbcContext(**big.ctx_kwargs)
    big.setup(ctx)
    full = ctx.run_voxels(big.tacs)
    dfull = ctx.run_voxels(torch.from_numpy(big.tacs).cuda())
    for n in (15, 50, 100):
        d, _ = run_gpu(rt_small.replace(n_accept=n))
        t = ctx.reduce_accepted(full["acc_idx"], n, want=tuple(k for k in d if k != "acc_dist"))
        td = ctx.reduce_accepted(dfull["acc_idx"], n)
        for k in t:
            np.testing.assert_array_equal(np.nan_to_num(t[k]), np.nan_to_num(d[k]), err_msg=(n, k))
        for k in td:
            a = td[k].cpu().numpy()
            if d[k].dtype == np.uint32:
                a = a.view(np.uint32)
            np.testing.assert_array_equal(np.nan_to_num(a), np.nan_to_num(d[k]), err_msg=(n, k))


def test_epsilon_calibrated_from_pilot(tb_small):
    """calibrate.epsilon_from_pilot: eps = median over voxels of the pilot's n-th smallest D makes
    about half of the voxels accept >= n draws in eps mode, and each voxel's
    eps-mode count is exactly the number of its pilot distances <= eps (below the pilot's n_max)."""
    from paper_2603_14859_b200 import calibrate as CAL
    p = tb_small.replace(n_accept=60)
    g, _ = run_gpu(p)
    eps = CAL.epsilon_from_pilot(g["acc_dist"], 18)
    e, _ = run_gpu(p.replace(accept="EPS", epsilon=eps))
    cnt = e["count"].sum(1).astype(np.int64)
    frac = np.mean(cnt >= 18)
    assert 0.5 <= frac <= 0.5 + 2.0 / p.J, frac
    below = cnt < 60
    np.testing.assert_array_equal(cnt[below], np.sum(g["acc_dist"][below] <= eps, axis=1))


@pytest.mark.parametrize("N,n,flags", [(40_000, 3000, 0), (20_000, 9000, 0), (40_000, 3000, 0x80), (16_000, 5000, 0x20)])
def test_large_n_cta_certification(tb_small, N, n, flags):
    """n beyond the warp layout (candidate sets > 2048): one CTA per voxel certifies and reduces
    (CTA bitonic sort of up to 16384 (D64, i) pairs, radix-select quantiles); n = 9000 also takes the
    single-part scan.  Forced fallback (0x80) and the flat scan (0x20) at large n too."""
    half = N // 2
    models = [dict(m, n_draws=(half if k == 0 else N - half)) for k, m in enumerate(tb_small.ctx_kwargs["models"])]
    p = tb_small.replace(models=models, n_accept=n).subset(np.arange(48))
    g, _ = run_gpu(p, flags=flags)
    o, _ = run_oracle(p)
    rep = compare(g, o)
    assert rep["matched"] >= p.J - 2


@pytest.mark.parametrize("ell", [3.5, 14.0])
def test_continuous_phantom_parity(ell, rot):
    """Harder data: kinetic parameters as continuous fields over the whole prior range, low and high
    noise (synthetic.config4_continuous); exactness does not depend on clusterability."""
    p = S.config4_continuous(chunk=5, n_chunks=64, N=200_000, n=18, ell=ell, max_voxels=2000)
    sub = p.subset(np.random.default_rng(3).choice(p.J, 96, replace=False))
    g, _ = run_gpu(sub)
    o, _ = run_oracle(sub)
    rep = compare(g, o)
    assert rep["matched"] >= sub.J - 2


def test_two_contexts_one_process(tb_small, rt_small):
    """Two live contexts in one process (different models, frame counts and shared-memory sizes of the
    certification: n = 18 vs n = 400): per-device kernel attributes and per-context buffers do not
    interfere; each equals its own single-context run."""
    from paper_2603_14859_b200 import AbcContext
    a_ref, _ = run_gpu(tb_small)
    b_prob = rt_small.replace(n_accept=400)
    b_ref, _ = run_gpu(b_prob)
    ca = AbcContext(**tb_small.ctx_kwargs)
    tb_small.setup(ca)
    cb = AbcContext(**b_prob.ctx_kwargs)
    b_prob.setup(cb)
    for _ in range(2):
        ra = ca.run_voxels(tb_small.tacs)
        rb = cb.run_voxels(b_prob.tacs)
        for k in a_ref:
            np.testing.assert_array_equal(np.nan_to_num(ra[k]), np.nan_to_num(a_ref[k]), err_msg=k)
        for k in b_ref:
            np.testing.assert_array_equal(np.nan_to_num(rb[k]), np.nan_to_num(b_ref[k]), err_msg=k)


def test_rotated_basis_adversarial_voxels(tb_small, monkeypatch):
    """The FP32 pass runs in the eigenbasis of the bank covariance with a tail bound after the first
    coordinates.  Voxels built from the ORACLE's bank probe its edge cases: exact bank
    curves (D = 0 for one draw), curves one FP32 ulp away, midpoints of two draws, far outliers,
    constant and all-zero TACs.  The rotated default must equal the oracle and, byte for byte, the
    frame-basis pass (ABC_FLAG_NO_REORDER keeps the frame basis)."""
    from oracle import oracle as O
    monkeypatch.setenv("VPET_ROT_ALWAYS", "1")
    o = O.OracleContext(**tb_small.ctx_kwargs)
    tb_small.setup(o)
    bank = o.bank()
    rng = np.random.default_rng(5)
    rows = rng.choice(bank.shape[0], 12, replace=False)
    b = bank[rows].astype(np.float32)
    y = np.concatenate([
        b[:4],                                                     # exact bank curves
        np.nextafter(b[4:6], np.float32(np.inf)),                  # one ulp up, every frame
        ((b[6:8].astype(np.float64) + b[8:10]) / 2).astype(np.float32),  # midpoints of two draws
        b[10:12] * np.float32(25.0),                               # far outliers
        np.full((1, b.shape[1]), np.float32(b.mean())),            # constant TAC
        np.zeros((1, b.shape[1]), np.float32),                     # all zeros
        tb_small.tacs[:50],                                        # ordinary voxels around them
    ]).astype(np.float32)
    g, _ = run_gpu(tb_small, tacs=y)
    ref, _ = run_oracle(tb_small, tacs=y)
    rep = compare(g, ref)
    assert rep["matched"] >= y.shape[0] - 1, rep
    # an exact bank curve accepts its own draw first, at distance 0
    np.testing.assert_array_equal(g["acc_dist"][:4, 0], 0.0)
    np.testing.assert_array_equal(np.asarray(g["acc_idx"][:4, 0]).astype(np.int64), rows[:4].astype(np.int64))
    from paper_2603_14859_b200 import FLAG_NO_REORDER
    fr, _ = run_gpu(tb_small, tacs=y, flags=FLAG_NO_REORDER)
    for k in g:
        np.testing.assert_array_equal(np.nan_to_num(g[k]), np.nan_to_num(fr[k]), err_msg=k)
