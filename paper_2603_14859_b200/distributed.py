"""Multi-GPU voxel sharding (the paper runs one V100).

Voxels are independent units of Alg. 1: every rank regenerates the same N draws from the shared
seed (the bank is a pure function of the configuration), runs `abc_run_voxels` on a contiguous,
equal-count range of voxels, and the per-voxel maps are gathered.  The only collectives are one
broadcast of the (small) configuration / input function / frame table from rank 0 and one gather
of the maps -- none inside the hot loop.  One process per GPU; NCCL over NVLink for CUDA tensors,
gloo for the CPU tests.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist

_NP2T = {np.float32: torch.float32, np.float64: torch.float64, np.int32: torch.int32,
         np.uint32: torch.int64, np.uint64: torch.int64}


def shard_range(J: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split: the first J % world ranks get one extra voxel."""
    base, extra = divmod(J, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def broadcast_setup(setup: Optional[dict], src: int = 0) -> dict:
    """Broadcast the run description (context kwargs, input function, frames) from `src`."""
    obj = [setup]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def _to_tensor(a: np.ndarray, device) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    elif a.dtype == np.uint32:
        a = a.astype(np.int64)
    return torch.from_numpy(a).to(device)


def gather_maps(local: dict, J: int, device, dst: int = 0) -> Optional[dict]:
    """Gather per-voxel outputs of all ranks (shards in rank order) onto `dst`.

    Shards are padded to the largest shard so `all_gather_into_tensor` (NCCL) / `all_gather`
    (gloo) move one fixed-size buffer per field.
    """
    world, rank = dist.get_world_size(), dist.get_rank()
    sizes = [shard_range(J, world, r)[1] - shard_range(J, world, r)[0] for r in range(world)]
    mx = max(sizes)
    out = {}
    for name in sorted(local):
        a = local[name]
        dtype = a.dtype
        t = _to_tensor(a, device)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=device)
        pad[: t.shape[0]] = t
        if device.type == "cuda":
            buf = torch.empty((world * mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=device)
            dist.all_gather_into_tensor(buf, pad)
            parts = [buf[r * mx: r * mx + sizes[r]] for r in range(world)]
        else:
            lst = [torch.empty_like(pad) for _ in range(world)]
            dist.all_gather(lst, pad)
            parts = [lst[r][: sizes[r]] for r in range(world)]
        if rank == dst:
            full = torch.cat(parts).cpu().numpy()
            if dtype == np.uint64:
                full = full.view(np.uint64)
            elif dtype == np.uint32:
                full = full.astype(np.uint32)
            out[name] = full
    return out if rank == dst else None


def run_sharded(setup: Optional[dict], tacs: Optional[np.ndarray], runner: Callable, device=None,
                src: int = 0) -> Optional[dict]:
    """Run a whole volume over the process group.

    setup:  on `src`, dict(ctx_kwargs=..., input=(kind, value, t), frames=(start, dur, weight)).
    tacs:   the full J x L array on `src` (other ranks may pass None; their shard is sent by a
            broadcast of the shard bounds and a scatter of rows) -- or every rank passes the full
            array (e.g. read from a shared file) and no TAC traffic is needed.
    runner: runner(setup, tacs_shard) -> dict of per-voxel numpy arrays (the AbcContext on the GPU;
            the CPU tests pass the oracle).
    Returns the gathered maps on `src`, None elsewhere.
    """
    world, rank = dist.get_world_size(), dist.get_rank()
    device = device or torch.device("cpu")
    setup = broadcast_setup(setup, src)
    meta = [None if tacs is None else tacs.shape]
    dist.broadcast_object_list(meta, src=src)
    J, L = meta[0]
    have_all = [tacs is not None]
    flags = [None] * world
    dist.all_gather_object(flags, have_all[0])
    a, b = shard_range(J, world, rank)
    if all(flags):
        shard = np.ascontiguousarray(tacs[a:b], dtype=np.float32)
    else:  # scatter rows from src (padded)
        sizes = [shard_range(J, world, r)[1] - shard_range(J, world, r)[0] for r in range(world)]
        mx = max(sizes)
        recv = torch.zeros((mx, L), dtype=torch.float32, device=device)
        if rank == src:
            parts = []
            for r in range(world):
                ra, rb = shard_range(J, world, r)
                p = torch.zeros((mx, L), dtype=torch.float32, device=device)
                p[: rb - ra] = torch.from_numpy(np.ascontiguousarray(tacs[ra:rb], dtype=np.float32)).to(device)
                parts.append(p)
            dist.scatter(recv, parts, src=src)
        else:
            dist.scatter(recv, None, src=src)
        shard = recv[: b - a].cpu().numpy()
    local = runner(setup, shard)
    return gather_maps(local, J, device, dst=src)
