"""Multi-GPU voxel sharding (the paper runs one V100).

Voxels are independent units of Alg. 1: every rank regenerates the same N draws from the shared
seed (the bank is a pure function of the configuration), runs `abc_run_voxels` on its shard of
voxels, and the per-voxel maps are gathered on one rank.  The only collectives are one broadcast
of the (small) configuration / input function / frame table and one gather of the maps -- none
inside the hot loop.  One process per GPU; NCCL over NVLink for CUDA tensors, gloo for the CPU
tests.

Sharding is interleaved: rank r of G owns voxels j = r, r + G, r + 2G, ...  The pruned FP32 pass
costs very different amounts per voxel (tissue class, noise level, activity), and a volume stored
in raster order has long runs of one class; interleaving gives every rank the same class mix, so
the ranks finish together (contiguous ranges would hand one rank the brain and another the legs).
"""
from __future__ import annotations

from typing import Callable, Iterable, Optional

import numpy as np
import torch
import torch.distributed as dist

# the parametric maps gathered on the destination rank (K_i mean + SD, model
# probabilities; plus the other per-voxel summaries of P:177-180)
MAP_OUTPUTS = ("prob", "preferred", "count", "mean", "sd", "q", "ki_mean", "ki_sd", "ki_q")


def shard_indices(J: int, world: int, rank: int) -> np.ndarray:
    """Voxels owned by `rank`: j = rank, rank + world, ... (interleaved)."""
    return np.arange(rank, J, world, dtype=np.int64)


def shard_size(J: int, world: int, rank: int) -> int:
    return max(0, (J - rank + world - 1) // world)


def shard_range(J: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split (first J % world ranks get one extra voxel).  Kept for callers
    that stream a volume from disk in slabs; the default sharding is `shard_indices`."""
    base, extra = divmod(J, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def broadcast_setup(setup: Optional[dict], src: int = 0) -> dict:
    """Broadcast the run description (context kwargs, input function, frames) from `src`."""
    obj = [setup]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def _as_tensor(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device)
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    elif a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).to(device)


def gather_maps(local: dict, J: int, device, dst: int = 0, names: Optional[Iterable[str]] = None) -> Optional[dict]:
    """Gather the per-voxel outputs of every rank's interleaved shard onto `dst` (a point-to-point
    `gather`, not an all-gather: only `dst` receives the maps).

    local: name -> array/tensor with the rank's shard_size(J, world, rank) rows (numpy or torch,
    host or device).  Returns {name: full J-row tensor on `device`} on `dst`, None elsewhere.
    Shards are padded to the largest shard so every rank sends one fixed-size buffer per field.
    """
    world, rank = (dist.get_world_size(), dist.get_rank()) if dist.is_initialized() else (1, 0)
    mx = shard_size(J, world, 0)
    out = {}
    for name in sorted(names if names is not None else local):
        t = _as_tensor(local[name], device)
        n = t.shape[0]
        if n == mx:
            send = t.contiguous()
        else:
            send = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=device)
            send[:n] = t
        if world == 1:
            out[name] = send[:J]
            continue
        bufs = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
        dist.gather(send, gather_list=bufs, dst=dst)
        if rank == dst:
            full = torch.empty((J,) + tuple(t.shape[1:]), dtype=t.dtype, device=device)
            for r in range(world):
                full[r::world] = bufs[r][: shard_size(J, world, r)]
            out[name] = full
    return out if rank == dst else None


def to_numpy_maps(maps: dict, like: dict) -> dict:
    """Convert gathered tensors back to numpy with the dtypes of `like` (uint32/uint64 views)."""
    res = {}
    for k, t in maps.items():
        a = t.cpu().numpy()
        dt = np.asarray(like[k]).dtype if not isinstance(like[k], torch.Tensor) else None
        if dt is not None and dt in (np.uint32, np.uint64):
            a = a.view(dt)
        res[k] = a
    return res


def run_volume(ctx, tacs_shard, J: int, dst: int = 0, names=MAP_OUTPUTS, out=None) -> Optional[dict]:
    """One rank's part of a whole-volume map: run Alg. 1 on this rank's interleaved shard through
    the C ABI (`ctx` is the rank's AbcContext) and gather the maps on `dst`.

    tacs_shard: the rank's rows (shard_indices order) as a host numpy array (pinned for async
    copies) or a CUDA tensor.  With a CUDA shard the outputs stay on the device and the gather is
    an NCCL gather into HBM of `dst`; with a host shard the library copies in/out and the gather
    runs on the process group's device (`dist` backend).  Returns {name: J-row tensor} on `dst`.
    """
    res = ctx.run_voxels(tacs_shard, want=tuple(names), out=out)
    if isinstance(tacs_shard, torch.Tensor) and tacs_shard.is_cuda:
        dev = tacs_shard.device
    elif out is not None and any(isinstance(v, torch.Tensor) and v.is_cuda for v in out.values()):
        dev = next(v.device for v in out.values() if isinstance(v, torch.Tensor))
    elif dist.is_initialized() and dist.get_backend() == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    else:
        dev = torch.device("cpu")
    return gather_maps({k: res[k] for k in names}, J, dev, dst=dst, names=names)


def run_sharded(setup: Optional[dict], tacs: Optional[np.ndarray], runner: Callable, device=None,
                src: int = 0) -> Optional[dict]:
    """Run a whole volume over the process group (rank `src` holds the description).

    setup:  on `src`, dict(ctx_kwargs=..., input=(kind, value, t), frames=(start, dur, weight)).
    tacs:   the full J x L array on `src` (other ranks may pass None; their rows are then sent by
            a scatter from `src`) -- or every rank passes the full array (e.g. read from a shared
            file) and no TAC traffic is needed.
    runner: runner(setup, tacs_shard) -> dict of per-voxel numpy arrays (the AbcContext on the GPU;
            the CPU tests may pass the oracle).
    Returns the gathered maps (numpy, full J rows) on `src`, None elsewhere.
    """
    world, rank = dist.get_world_size(), dist.get_rank()
    device = device or torch.device("cpu")
    setup = broadcast_setup(setup, src)
    meta = [None if tacs is None else tuple(tacs.shape)]
    dist.broadcast_object_list(meta, src=src)
    J, L = meta[0]
    flags = [None] * world
    dist.all_gather_object(flags, tacs is not None)
    idx = shard_indices(J, world, rank)
    if all(flags):
        shard = np.ascontiguousarray(tacs[idx], dtype=np.float32)
    else:  # scatter rows from src (padded to the largest shard)
        mx = shard_size(J, world, 0)
        recv = torch.zeros((mx, L), dtype=torch.float32, device=device)
        if rank == src:
            parts = []
            for r in range(world):
                p = torch.zeros((mx, L), dtype=torch.float32, device=device)
                rows = shard_indices(J, world, r)
                p[: len(rows)] = torch.from_numpy(np.ascontiguousarray(tacs[rows], dtype=np.float32)).to(device)
                parts.append(p)
            dist.scatter(recv, parts, src=src)
        else:
            dist.scatter(recv, None, src=src)
        shard = recv[: len(idx)].cpu().numpy()
    local = runner(setup, shard)
    maps = gather_maps(local, J, device, dst=src)
    return to_numpy_maps(maps, local) if rank == src else None
