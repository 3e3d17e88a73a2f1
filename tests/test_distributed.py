"""World-size-2 gloo tests of the voxel-sharded path (a6) on CPU: sharding + broadcast + gather must
reproduce the single-process result byte for byte.  The per-rank compute here is the CPU oracle
(tests may use it); on GPUs the runner is the CUDA library (bench.py / distributed.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2603_14859_b200.distributed import shard_indices, shard_range, shard_size


def test_shard_indices_interleaved_partition():
    for J in (0, 1, 7, 64, 1001):
        for world in (1, 2, 3, 8):
            parts = [shard_indices(J, world, r) for r in range(world)]
            assert sorted(np.concatenate(parts).tolist()) == list(range(J))
            assert [len(p) for p in parts] == [shard_size(J, world, r) for r in range(world)]
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
            assert shard_size(J, world, 0) == max(map(len, parts))


def test_shard_range_balanced_and_covering():
    for J in (0, 1, 7, 64, 1001):
        for world in (1, 2, 3, 8):
            rs = [shard_range(J, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == J
            assert all(rs[r][1] == rs[r + 1][0] for r in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_runner(setup, shard):
    from oracle import oracle as O
    ctx = O.OracleContext(**setup["ctx_kwargs"])
    kind, value, t = setup["input"]
    ctx.set_input_function(kind, value, t=t)
    ctx.set_frames(*setup["frames"])
    return ctx.run_voxels(shard)


def _worker(rank, world, port, setup, tacs, scatter, q):
    import torch.distributed as dist

    from paper_2603_14859_b200.distributed import run_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = run_sharded(setup if rank == 0 else None, tacs if (rank == 0 or not scatter) else None,
                          _oracle_runner)
        if rank == 0:
            q.put({k: v for k, v in out.items()})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scatter", [False, True])
def test_two_rank_gloo_equals_single_process(scatter):
    import synthetic as S
    p = S.config1(J=13, N=600, p=0.02)
    setup = dict(ctx_kwargs=p.ctx_kwargs, input=(p.input_kind, p.input_value, p.input_t),
                 frames=(p.frame_start, p.frame_dur, p.weight))
    single = _oracle_runner(setup, p.tacs)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, setup, p.tacs, scatter, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert set(got) == set(single)
    for k in single:
        np.testing.assert_array_equal(got[k], single[k], err_msg=k)
