#!/usr/bin/env python
"""Benchmark of the vPET-ABC hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[3]): the total-body 50-min FDG phantom (192 x 192 x 673,
4,441,800 in-mask voxels, 35 frames, PWL IDIF), 2TCM k4 = 0 vs k4 > 0 model selection
(eq:prior2, M = 2), N = 1e7 prior draws, n = 18 accepted, weighted L2.
One step = the WHOLE-VOLUME map: every rank runs the whole hot path (prior draws -> bank
simulation -> FP32 pass -> FP64 certification -> posterior reduction) on its interleaved shard of
the volume (voxels j = rank mod G), then the parametric maps are gathered on rank 0 (NCCL gather).
Strong scaling: the total work is fixed, G GPUs share it.  Each rank regenerates the same draws
from the seed; the gather is the only data-path collective.

value  = voxel-draw discrepancy evaluations per second of the whole job (J_total * N / t), with
         the TACs resident in HBM; t = max over ranks of the step (run + gather) time.
tb_ki_map_time_s = t: measured wall time of the whole-volume K_i map.
e2e    = the same through the public API with host buffers: pinned host TAC shard -> C ABI
         (H2D inside) -> NCCL gather -> D2H of the gathered maps on rank 0, all in the timed region.
--impl reference runs the CPU oracle (the reference arm of this tier) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated draws/sec, voxels/sec and TB K_i-map time at 1/2/4/8 B200"
TB_VOXELS = 4_441_800
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "r02_scan_volume_ncu.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--draws", type=int, default=10_000_000)
    ap.add_argument("--n-accept", type=int, default=18)
    ap.add_argument("--chunks", type=int, default=1,
                    help="1 = the whole volume (default); k > 1 = axial slabs z = 0 mod k only (quick runs)")
    ap.add_argument("--max-voxels", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--cpu-draws", type=int, default=1_000_000, help="reference arm: draws per sampled voxel")
    ap.add_argument("--cpu-voxels", type=int, default=32, help="reference arm: sampled voxels per step")
    ap.add_argument("--baseline-voxels", type=int, default=32, help="cpu_baseline: sampled voxels")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (200 ms period)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
            t0 = time.time()  # let nvidia-smi initialise before the timed region starts
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.05)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        load = [r for r in self.rows if (num(r[6]) or 0) > 50] or self.rows
        sm = [num(r[0]) for r in load if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in load for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(self.rows[0][1]),
                "reasons": reasons, "samples": len(self.rows), "samples_under_load": len(load)}


def dist_init(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_ranks(x: float, world: int) -> list:
    if world == 1:
        return [x]
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [float(v.item()) for v in out]


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _strided_sample(J_total, k):
    return np.unique(np.linspace(0, J_total - 1, k).round().astype(np.int64))


def cpu_baseline_run(args, J_total, n_vox, n_draws, time_bank=True):
    """The oracle as it stands on a bounded sample of the bench workload: n_vox voxels strided over
    the whole volume, N = n_draws draws.  value = sampled voxel-draw pairs / wall time of the
    oracle's abc_run_voxels (its FP64 bank build included, as in one step of the GPU path); the
    bank build alone is also timed (ctx.bank()) and reported as bank_s."""
    import synthetic as S
    from oracle import oracle as O
    idx = _strided_sample(J_total, n_vox)
    prob = S.config4_chunk(chunk=0, n_chunks=args.chunks, N=n_draws, n=args.n_accept, voxel_index=idx,
                           max_voxels=args.max_voxels)
    ctx = O.OracleContext(**prob.ctx_kwargs)
    prob.setup(ctx)
    N = ctx.N
    t = time.perf_counter()
    ctx.run_voxels(prob.tacs)
    t_run = time.perf_counter() - t
    t_bank = float("nan")
    if time_bank:
        t = time.perf_counter()
        ctx.bank()
        t_bank = time.perf_counter() - t
    return {"value": len(idx) * N / t_run, "unit": "draws/s", "cores": O.get_threads(), "kind": "oracle",
            "sample": f"{len(idx)} voxels strided over the volume x N={N} draws, {t_run:.1f} s wall "
                      f"(FP64 bank build included; bank alone {t_bank:.1f} s)",
            "bank_s": t_bank}


def run_reference(args):
    """--impl reference: the CPU oracle (this tier's reference arm) on a bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synthetic as S
    J_total = S.tb_voxel_count() if args.chunks == 1 and args.max_voxels is None else None
    if J_total is None:
        J_total = S.config4_chunk(chunk=0, n_chunks=args.chunks, N=1000, max_voxels=args.max_voxels).J
    times = []
    for s_ in range(args.warmup + args.steps):
        r = cpu_baseline_run(args, J_total, args.cpu_voxels, args.cpu_draws, time_bank=False)
        if s_ >= args.warmup:
            times.append(r)
    # the oracle's rate including its bank build (what one step of the sample costs)
    v = statistics.median([r["value"] for r in times])
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "draws/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD + f" (oracle sample: {args.cpu_voxels} voxels strided over the "
                                   f"volume x N={args.cpu_draws} draws per step)"},
            "cpu_baseline": {"value": v, "unit": "draws/s", "cores": times[0]["cores"], "kind": "oracle",
                             "sample": times[0]["sample"]},
            "e2e": {"value": v, "unit": "draws/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


WORKLOAD = ("config4: total-body 50-min FDG phantom 192x192x673 (4,441,800 in-mask voxels), 2TCM k4=0 vs "
            "k4>0 (M=2), N=1e7 draws, n=18, L=35, weighted L2; one step = the whole-volume map "
            "(interleaved voxel shards over the ranks, maps gathered on rank 0)")


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch

    import synthetic as S
    from paper_2603_14859_b200 import FLAG_COUNT_WORK, FLAG_TIMING, AbcContext
    from paper_2603_14859_b200.distributed import MAP_OUTPUTS, gather_maps, shard_indices

    world, rank, local = dist_init(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    t0 = time.time()
    # every rank generates the same volume (deterministic) and keeps its interleaved shard: the
    # stand-in for each rank reading its own rows of the TAC file
    prob = S.config4_chunk(chunk=0, n_chunks=args.chunks, N=args.draws, n=args.n_accept, device=str(dev),
                           max_voxels=args.max_voxels)
    gen_s = time.time() - t0
    J_total, L, N = prob.J, prob.L, args.draws
    idx = shard_indices(J_total, world, rank)
    J = len(idx)
    tacs_shard = np.ascontiguousarray(prob.tacs[idx])
    del prob.truth["clean"]
    ctx = AbcContext(**dict(prob.ctx_kwargs, flags=FLAG_TIMING | args.flags, device=local))
    prob.setup(ctx)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    y = torch.from_numpy(tacs_shard).to(dev)
    tdt = {"prob": torch.float32, "preferred": torch.int32, "count": torch.int32, "mean": torch.float32,
           "sd": torch.float32, "q": torch.float32, "ki_mean": torch.float32, "ki_sd": torch.float32,
           "ki_q": torch.float32, "acc_idx": torch.int64, "acc_dist": torch.float64}
    outs = {k: torch.empty(v, dtype=tdt[k], device=dev) for k, v in ctx.shapes(J).items()}
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step(tacs, o):
        ctx.run_voxels(tacs, out=o)
        return gather_maps({k: o[k] for k in MAP_OUTPUTS}, J_total, dev, dst=0, names=MAP_OUTPUTS)

    for _ in range(args.warmup):
        step(y, outs)
    torch.cuda.synchronize()
    step_ms, run_ms, stage = [], [], []
    launches = 0
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))  # L2 flush between timed iterations (outside the events)
            barrier(world)
            torch.cuda.synchronize()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            ctx.run_voxels(y, out=outs)
            e1.record(stream)
            gather_maps({k_: outs[k_] for k_ in MAP_OUTPUTS}, J_total, dev, dst=0, names=MAP_OUTPUTS)
            e2.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e2))
            run_ms.append(e0.elapsed_time(e1))
            st = ctx.stats()
            stage.append(st)
            launches += st["gpu_launches"]
    clocks = clk.summary()
    total_ms = max_over_ranks(sum(step_ms), world)
    ms_step = total_ms / args.steps
    rank_run_ms = all_ranks(statistics.median(run_ms), world)
    pairs_per_step_all = float(J_total) * N
    value = pairs_per_step_all / (ms_step / 1e3)
    vox_rate = J_total / (ms_step / 1e3)

    # executed frame updates of the FP32 pass (deterministic for this input): one counted run
    cctx = AbcContext(**dict(prob.ctx_kwargs, flags=FLAG_TIMING | FLAG_COUNT_WORK | args.flags, device=local))
    prob.setup(cctx)
    cctx.set_stream(stream.cuda_stream)
    cctx.run_voxels(y, out=outs)
    cst = cctx.stats()
    frame_updates = cst["frame_updates"]
    bound_updates = cst.get("bound_updates", 0)
    del cctx
    scan_s = statistics.median([s_["ms_scan"] for s_ in stage]) / 1e3
    sm_mhz = clocks.get("sm_max_mhz") or 1965.0
    peak_ops = 148 * 128 * sm_mhz * 1e6  # FP32 lane-ops/s (148 SMs x 128 FP32 lanes x clock)
    # executed FP32 lane-ops: a distance frame update is FADD + FFMA (2), a bound frame update is
    # 2 FADD + FMNMX3 + FFMA (4) -- counted on device in a separate, untimed run of the same input
    achieved = (2.0 * frame_updates + 4.0 * bound_updates) / scan_s
    dense_equiv = 2.0 * J * N * L / scan_s
    roof = {"bound": "alu", "kernel": "scan_tree_kernel (K2, FP32 pass)", "achieved": achieved / 1e12,
            "peak": peak_ops / 1e12, "unit": "TFLOP/s", "frac": achieved / peak_ops,
            "peak_basis": f"148 SM x 128 FP32 lanes x {sm_mhz:.0f} MHz (derived, DESIGN.md)",
            "traffic": None, "executed_frame_updates_per_launch": frame_updates,
            "executed_bound_updates_per_launch": bound_updates,
            "dense_equivalent_tflops": dense_equiv / 1e12,
            "pruned_fraction_of_dense": frame_updates / float(J * N * L),
            "scan_ms": scan_s * 1e3, "scan_share_of_step": scan_s * 1e3 / statistics.median(step_ms),
            # the same executed lane-ops against the rate the FADD2+FFMA2 distance step itself reaches in
            # the microbenchmark (115.7 lane-op/clk/SM, profiles/r02_fp_rates.txt)
            "peak_measured_mix": 148 * 115.7 * sm_mhz * 1e6 / 1e12,
            "frac_vs_measured_mix": achieved / (148 * 115.7 * sm_mhz * 1e6)}
    if os.path.exists(PROFILE_SUMMARY):
        try:
            ps = json.load(open(PROFILE_SUMMARY))
            roof["traffic"] = ps.get("dram_bytes_per_launch")
            roof["traffic_source"] = os.path.relpath(PROFILE_SUMMARY, ROOT)
            roof["traffic_workload"] = ps.get("workload")
        except Exception:
            pass

    # e2e: the same map through the public API with host buffers: pinned host TAC shard -> C ABI
    # (H2D inside) -> host maps: written by the library itself at one rank (its K4 chunks overlap
    # their D2H), else device outputs -> NCCL gather -> D2H of the gathered maps on rank 0
    e2e = None
    if not args.no_e2e:
        hy = torch.from_numpy(tacs_shard).pin_memory().numpy()
        host_maps = None
        d2h = 0
        if rank == 0:
            host_maps = {k: torch.empty((J_total,) + tuple(outs[k].shape[1:]), dtype=outs[k].dtype, pin_memory=True)
                         for k in MAP_OUTPUTS}
            d2h = sum(int(v.numel() * v.element_size()) for v in host_maps.values())

        def e2e_step():
            if world == 1:  # one rank: the library writes the maps into the pinned host buffers itself
                ctx.run_voxels(hy, out=host_maps)  # (its K4 chunks overlap their device-to-host copies)
                return
            maps = step(hy, outs)
            if rank == 0:
                for k_ in MAP_OUTPUTS:
                    host_maps[k_].copy_(maps[k_], non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        e2e_ms = []
        for k in range(args.steps):
            flush.fill_(float(k))
            barrier(world)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e2e_step()
            b.record(stream)
            torch.cuda.synchronize()
            e2e_ms.append(a.elapsed_time(b))
        e2e_tot = max_over_ranks(sum(e2e_ms), world)
        e2e = {"value": pairs_per_step_all / (e2e_tot / args.steps / 1e3), "unit": "draws/s",
               "h2d_bytes_per_step": int(J_total * L * 4), "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_tot / args.steps, "tb_ki_map_time_s": e2e_tot / args.steps / 1e3}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_run(args, J_total, args.baseline_voxels, args.cpu_draws)

    med = {k: statistics.median([s_[k] for s_ in stage]) for k in
           ("ms_h2d", "ms_bank", "ms_order", "ms_scan", "ms_certify", "ms_fallback", "ms_d2h", "ms_total")}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "draws/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "step_ms": [round(v, 3) for v in step_ms],
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD if args.chunks == 1 else WORKLOAD + f" [slabs z = 0 mod {args.chunks} only]",
                       "voxels_total": J_total, "voxels_per_rank": J, "draws": N, "n_accept": args.n_accept,
                       "frames": L, "sharding": "interleaved voxels j = rank mod G; maps gathered on rank 0",
                       "l2": "flushed (512 MB write) between timed steps; bank 2x1.44 GB > L2",
                       "dtype_detail": "FP32 pass + FP64 simulation/certification/reduction"},
            "voxels_per_s": vox_rate,
            "tb_ki_map_time_s": ms_step / 1e3 if args.chunks == 1 and args.max_voxels is None else None,
            "tb_ki_map_time_basis": "measured: whole volume (4,441,800 voxels), TACs resident in HBM -> maps "
                                    "gathered on rank 0 (max over ranks); e2e.tb_ki_map_time_s from pinned host TACs "
                                    "to host maps on rank 0",
            "rank_run_ms": rank_run_ms,
            "rank_imbalance": (max(rank_run_ms) / min(rank_run_ms)) if min(rank_run_ms) > 0 else None,
            "paper_context": {"v100_tb_time_s": 36000, "v100_pairs_per_s": 1.22e9, "source": "P:460, BASELINE.md"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "gpu_launches_per_step": launches // args.steps,
            "clocks": clocks,
            "stage_ms_median": med,
            "n_fallback_voxels": stage[-1]["n_fallback"],
            "input_generation_s": gen_s,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
