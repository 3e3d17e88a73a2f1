"""The CUDA library through the sharded pipeline (VERDICT r01 "next" item 2):
broadcast of the setup, interleaved voxel shards, per-rank abc_run_voxels through the C ABI, gather
of the maps on rank 0 -- byte-for-byte equal to one process running every voxel.

* world size 2 over gloo, both ranks on GPU 0: each rank's kernels are independent (no rank waits
  on another's kernels; the only exchange is the host-side gloo broadcast/gather), so this checks
  the host logic of the sharded path with the real CUDA runner on one GPU;
* world size 1 over NCCL: `run_volume` with device-resident TACs, device outputs and the NCCL
  gather path of bench.py.
Top-n results are exact (certified against the FP64 definition), so sharding cannot change a byte.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synthetic as S

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cuda_runner(setup, shard):
    from paper_2603_14859_b200 import AbcContext
    ctx = AbcContext(**setup["ctx_kwargs"])
    kind, value, t = setup["input"]
    ctx.set_input_function(kind, value, t=t)
    ctx.set_frames(*setup["frames"])
    return ctx.run_voxels(shard)


def _worker(rank, world, port, setup, tacs, q):
    import torch.distributed as dist

    from paper_2603_14859_b200.distributed import run_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = run_sharded(setup if rank == 0 else None, tacs if rank == 0 else None, _cuda_runner)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def _setup(p):
    return dict(ctx_kwargs=p.ctx_kwargs, input=(p.input_kind, p.input_value, p.input_t),
                frames=(p.frame_start, p.frame_dur, p.weight))


def test_two_rank_gloo_cuda_runner_equals_single_process():
    p = S.config4_chunk(chunk=11, n_chunks=64, N=200_000, n=18, max_voxels=3001)
    setup = _setup(p)
    single = _cuda_runner(setup, p.tacs)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, setup, p.tacs, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert set(got) == set(single)
    for k in single:
        assert got[k].dtype == single[k].dtype, k
        np.testing.assert_array_equal(got[k], single[k], err_msg=k)


def test_world1_nccl_run_volume_device_path():
    import torch
    import torch.distributed as dist

    from paper_2603_14859_b200 import AbcContext
    from paper_2603_14859_b200.distributed import MAP_OUTPUTS, run_volume
    p = S.config4_chunk(chunk=3, n_chunks=64, N=300_000, n=18, max_voxels=2500)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ctx = AbcContext(**p.ctx_kwargs)
        p.setup(ctx)
        ref = ctx.run_voxels(p.tacs)
        maps = run_volume(ctx, torch.from_numpy(p.tacs).cuda(), p.J)
        for k in MAP_OUTPUTS:
            a = maps[k].cpu().numpy()
            if ref[k].dtype == np.uint32:
                a = a.view(np.uint32)
            np.testing.assert_array_equal(a, ref[k], err_msg=k)
        # host TACs in, device outputs, the same gather
        outs = {k: torch.empty_like(maps[k]) for k in MAP_OUTPUTS}
        maps_h = run_volume(ctx, p.tacs, p.J, out=outs)
        for k in MAP_OUTPUTS:
            assert torch.equal(maps_h[k], maps[k]), k
    finally:
        dist.destroy_process_group()


def test_eps_mode_sharding_invariant():
    """eps mode sums the accepted draws' moments in 128-bit fixed point per (voxel,
    part): the maps of an interleaved shard are byte-identical to those of the full run although
    the FP32 pass visits the draws in a different order (other CTA-mates)."""
    from paper_2603_14859_b200 import AbcContext
    from paper_2603_14859_b200.distributed import shard_indices
    from tests.parity import run_oracle
    p = S.config4_chunk(chunk=9, n_chunks=64, N=100_000, n=18, max_voxels=1500)
    o_top, _ = run_oracle(p.subset(np.arange(40)))
    eps = float(np.median(o_top["acc_dist"][:, -1]))
    q = p.replace(accept="EPS", epsilon=eps)
    ctx = AbcContext(**q.ctx_kwargs)
    q.setup(ctx)
    full = ctx.run_voxels(q.tacs)
    for world in (2, 3):
        for r in range(world):
            idx = shard_indices(q.J, world, r)
            part = ctx.run_voxels(np.ascontiguousarray(q.tacs[idx]))
            for k in part:
                np.testing.assert_array_equal(part[k].view(np.uint8), full[k][idx].view(np.uint8), err_msg=k)
