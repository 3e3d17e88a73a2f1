#!/usr/bin/env python
"""Benchmark of the vPET-ABC hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[3]): the total-body 50-min FDG phantom (192 x 192 x 673,
4.44 M in-mask voxels, 35 frames, PWL IDIF), 2TCM k4 = 0 vs k4 > 0 model selection
(eq:prior2, M = 2), N = 1e7 prior draws, n = 18 accepted, weighted L2.
One step = one pass of the whole hot path (prior draws -> bank simulation -> FP32 pass ->
FP64 certification -> posterior reduction) over one batch: axial slices z = r, r + 32, ... of
the phantom (1/32 of the volume, ~139 k voxels) on rank r -- weak scaling, no data-path
collective (voxels are independent; each rank regenerates the same draws from the seed).

value  = voxel-draw discrepancy evaluations per second (J * N / t), whole job, max over ranks.
e2e    = the same through the C ABI with host buffers (pinned), H2D/D2H inside the timed region.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated draws/sec, voxels/sec and TB K_i-map time at 1/2/4/8 B200"
TB_VOXELS = 4_441_800
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "scan_ncu_summary.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--draws", type=int, default=10_000_000)
    ap.add_argument("--n-accept", type=int, default=18)
    ap.add_argument("--chunks", type=int, default=32, help="the volume is split into this many interleaved slabs")
    ap.add_argument("--max-voxels", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--cpu-draws", type=int, default=1_000_000)
    ap.add_argument("--cpu-voxels", type=int, default=32)
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


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_baseline_run(problem, n_draws, n_vox):
    """The oracle as it stands on a bounded sample: n_vox voxels of the batch, N = n_draws."""
    from oracle import oracle as O
    models = problem.ctx_kwargs["models"]
    scale = n_draws / sum(int(m["n_draws"]) for m in models)
    kw = dict(problem.ctx_kwargs)
    kw["models"] = [dict(m, n_draws=max(1, int(round(int(m["n_draws"]) * scale)))) for m in models]
    N = sum(m["n_draws"] for m in kw["models"])
    ctx = O.OracleContext(**kw)
    problem.setup(ctx)
    idx = list(range(0, problem.J, max(1, problem.J // n_vox)))[:n_vox]
    y = problem.tacs[idx]
    t = time.perf_counter()
    ctx.run_voxels(y)
    dt = time.perf_counter() - t
    return {"value": len(idx) * N / dt, "unit": "draws/s", "cores": O.get_threads(), "kind": "oracle",
            "sample": f"{len(idx)} voxels of the batch (strided) x N={N} draws (bank build included), "
                      f"{dt:.1f} s wall"}


def run_reference(args):
    """--impl reference: the CPU oracle (this tier's reference arm) on a bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synthetic as S
    prob = S.config4_chunk(chunk=0, n_chunks=args.chunks, N=args.draws, n=args.n_accept,
                           max_voxels=4 * args.cpu_voxels)
    times = []
    for s in range(args.warmup + args.steps):
        r = cpu_baseline_run(prob, args.cpu_draws, args.cpu_voxels)
        if s >= args.warmup:
            times.append(r)
    v = statistics.median([r["value"] for r in times])
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "draws/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config4: total-body FDG phantom 192x192x673, 2TCM k4 selection, "
                                   f"N={args.draws} (oracle sample N={args.cpu_draws}), n={args.n_accept}, L=35"},
            "cpu_baseline": {"value": v, "unit": "draws/s", "cores": times[0]["cores"], "kind": "oracle",
                             "sample": times[0]["sample"]},
            "e2e": {"value": v, "unit": "draws/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch

    import synthetic as S
    from paper_2603_14859_b200 import FLAG_COUNT_WORK, FLAG_TIMING, AbcContext

    world, rank, local = dist_init(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    t0 = time.time()
    prob = S.config4_chunk(chunk=rank % args.chunks, n_chunks=args.chunks, N=args.draws, n=args.n_accept,
                           device=str(dev), max_voxels=args.max_voxels)
    gen_s = time.time() - t0
    J, L, N = prob.J, prob.L, args.draws
    ctx = AbcContext(**dict(prob.ctx_kwargs, flags=FLAG_TIMING | args.flags, device=local))
    prob.setup(ctx)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    y = torch.from_numpy(prob.tacs).to(dev)
    outs = {k: torch.empty(v, dtype=dt, device=dev) for (k, v), dt in zip(
        ctx.shapes(J).items(),
        [torch.float32, torch.int32, torch.int32, torch.float32, torch.float32, torch.float32, torch.float32,
         torch.float32, torch.float32, torch.int64, torch.float64])}
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step(o):
        ctx.run_voxels(y, out=o)

    for _ in range(args.warmup):
        step(outs)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    step_ms, scan_ms, stage = [], [], []
    launches = 0
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))  # L2 flush between timed iterations (outside the events)
            barrier(world)
            torch.cuda.synchronize()
            ev[k][0].record(stream)
            step(outs)
            ev[k][1].record(stream)
            torch.cuda.synchronize()
            step_ms.append(ev[k][0].elapsed_time(ev[k][1]))
            st = ctx.stats()
            scan_ms.append(st["ms_scan"])
            stage.append(st)
            launches += st["gpu_launches"]
    clocks = clk.summary()
    total_ms = max_over_ranks(sum(step_ms), world)
    ms_step = total_ms / args.steps
    pairs_per_step_all = float(J) * N * world  # weak scaling: every rank holds an equal-size batch
    value = pairs_per_step_all / (ms_step / 1e3)
    vox_rate = J * world / (ms_step / 1e3)

    # executed frame updates of the FP32 pass (deterministic for this input): one counted run
    cctx = AbcContext(**dict(prob.ctx_kwargs, flags=FLAG_TIMING | FLAG_COUNT_WORK | args.flags, device=local))
    prob.setup(cctx)
    cctx.set_stream(stream.cuda_stream)
    cctx.run_voxels(y, out=outs)
    cst = cctx.stats()
    frame_updates = cst["frame_updates"]
    bound_updates = cst.get("bound_updates", 0)
    del cctx
    scan_s = statistics.median(scan_ms) / 1e3
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
            "scan_ms": scan_s * 1e3, "scan_share_of_step": scan_s * 1e3 / statistics.median(step_ms)}
    if os.path.exists(PROFILE_SUMMARY):
        try:
            ps = json.load(open(PROFILE_SUMMARY))
            roof["traffic"] = ps.get("dram_bytes_per_launch")
            roof["traffic_source"] = os.path.relpath(PROFILE_SUMMARY, ROOT)
        except Exception:
            pass

    # e2e: same step through the C ABI with pinned host buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        hy = torch.from_numpy(prob.tacs).pin_memory().numpy()
        houts = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True).numpy() for k, v in outs.items()}
        e2e_ms = []
        ctx.run_voxels(hy, out=houts)
        for k in range(args.steps):
            flush.fill_(float(k))
            barrier(world)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.run_voxels(hy, out=houts)
            b.record(stream)
            torch.cuda.synchronize()
            e2e_ms.append(a.elapsed_time(b))
        e2e_tot = max_over_ranks(sum(e2e_ms), world)
        e2e = {"value": pairs_per_step_all / (e2e_tot / args.steps / 1e3), "unit": "draws/s",
               "h2d_bytes_per_step": int(hy.nbytes), "d2h_bytes_per_step": int(sum(v.nbytes for v in houts.values())),
               "ms_per_step": e2e_tot / args.steps}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_run(prob, args.cpu_draws, args.cpu_voxels)

    med = {k: statistics.median([s[k] for s in stage]) for k in
           ("ms_h2d", "ms_bank", "ms_order", "ms_scan", "ms_certify", "ms_fallback", "ms_d2h", "ms_total")}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "draws/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "step_ms": [round(v, 3) for v in step_ms], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "config4: total-body 50-min FDG phantom 192x192x673 (4.44M voxels), 2TCM "
                                   "k4=0 vs k4>0 (M=2), N=1e7 draws, n=18, L=35, weighted L2; one step = axial "
                                   f"slab set {rank % args.chunks} mod {args.chunks} per rank",
                       "voxels_per_rank": J, "draws": N, "n_accept": args.n_accept, "frames": L,
                       "l2": "flushed (512 MB write) between timed steps; bank 2x1.44 GB > L2",
                       "dtype_detail": "FP32 pass + FP64 simulation/certification/reduction"},
            "voxels_per_s": vox_rate,
            "tb_ki_map_time_s": TB_VOXELS / vox_rate,
            "tb_ki_map_time_basis": "projected: 4,441,800 in-mask voxels / measured voxels/s",
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
