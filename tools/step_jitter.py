"""Per-step timing jitter diagnosis: outer CUDA events around run_voxels vs the library's internal
stage events vs host wall time of the call, with and without an nvidia-smi sampler running.
python tools/step_jitter.py [--steps 20]"""
import argparse
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2603_14859_b200 import FLAG_TIMING, AbcContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
p = S.config4_chunk(chunk=0, n_chunks=32, N=10_000_000, n=18, device="cuda")
ctx = AbcContext(**dict(p.ctx_kwargs, flags=FLAG_TIMING))
p.setup(ctx)
st = torch.cuda.current_stream()
ctx.set_stream(st.cuda_stream)
y = torch.from_numpy(p.tacs).cuda()
out = ctx.run_voxels(y)
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
for mode in ("plain", "smi", "plain"):
    proc = None
    if mode == "smi":
        proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                                stdout=subprocess.DEVNULL)
        time.sleep(1.0)
    rows = []
    for k in range(a.steps):
        flush.fill_(k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        ctx.run_voxels(y, out=out)
        e1.record(st)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        s = ctx.stats()
        rows.append((e0.elapsed_time(e1), s["ms_total"], s["ms_scan"], (t1 - t0) * 1e3))
    if proc:
        proc.terminate()
        proc.wait()
    print(mode)
    for r in rows:
        print("  outer %7.2f  inner %7.2f  scan %7.2f  host %7.2f" % r)
