"""Summarise an ncu report (.ncu-rep) or a launch-list CSV into profiles/.

python tools/ncu_summary.py report gpurun_out/scan.ncu-rep profiles/r01_scan_ncu.json
python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "sm__maximum_warps_per_active_cycle_pct", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__cycles_elapsed.avg.per_second",
    "l1tex__t_bytes.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "launch__shared_mem_per_block_dynamic",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {h: (v, u) for h, v, u in zip(hdr, r, units)}
        kernels.append(d)
    return kernels


def stalls(k):
    st = {}
    for name, (v, u) in k.items():
        if name.startswith("smsp__average_warp_latency_issue_stalled_") or name.startswith("smsp__pcsamp_warps_issue_stalled_"):
            try:
                st[name] = float(v.replace(",", ""))
            except ValueError:
                pass
    return dict(sorted(st.items(), key=lambda x: -x[1])[:12])


def report(path, dst):
    ks = raw(path)
    out = []
    for k in ks:
        d = {"kernel": k.get("Kernel Name", ("?", ""))[0][:120]}
        for m in WANT:
            if m in k:
                v, u = k[m]
                try:
                    d[m] = [float(v.replace(",", "")), u]
                except ValueError:
                    d[m] = [v, u]
        d["top_stalls"] = stalls(k)
        out.append(d)
    if out:
        k0 = out[0]
        rd = k0.get("dram__bytes_read.sum", [0, ""])
        wr = k0.get("dram__bytes_write.sum", [0, ""])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        tot = rd[0] * scale.get(rd[1], 1) + wr[0] * scale.get(wr[1], 1)
        summary = {"source": path, "dram_bytes_per_launch": tot, "kernels": out}
    else:
        summary = {"source": path, "kernels": []}
    json.dump(summary, open(dst, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:4000])


def launches(path, dst):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:100]
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3,
                 "s": 1e3}.get(r[ui], 1.0)
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    T = sum(tot.values())
    res = [{"kernel": k, "ms": v, "share": v / T, "launches": cnt[k]} for k, v in sorted(tot.items(), key=lambda x: -x[1])]
    json.dump({"source": path, "total_ms": T, "kernels": res}, open(dst, "w"), indent=1)
    for r in res:
        print(f"{r['ms']:10.3f} ms {100 * r['share']:6.2f}% x{r['launches']:4d} {r['kernel']}")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
