"""Attribute ncu warp-stall samples and executed instructions to CUDA source lines.

ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
fname, hdr = "?", None
cur = None
samp, inst, text = defaultdict(float), defaultdict(float), {}
stalls = defaultdict(lambda: defaultdict(float))
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()[:90]
        continue
    if cur is None:
        continue
    try:
        s = float(r[4])
        n = float(r[7])
    except (ValueError, IndexError):
        continue
    samp[cur] += s
    inst[cur] += n
    for k, h in enumerate(hdr):
        if h.startswith("stall_") and k < len(r):
            try:
                stalls[cur][h] += float(r[k])
            except ValueError:
                pass
T = sum(samp.values())
TI = sum(inst.values())
print(f"total samples {T:.0f}, warp instructions {TI:.3e}")
for key in sorted(samp, key=lambda k: -samp[k])[:top]:
    st = sorted(stalls[key].items(), key=lambda x: -x[1])[:3]
    sts = " ".join(f"{h[6:]}:{100 * v / max(samp[key], 1):.0f}%" for h, v in st)
    print(f"{100 * samp[key] / T:5.1f}% {100 * inst[key] / TI:5.1f}%i {key[0][:14]}:{key[1]:<4} {text[key][:70]:70s} {sts}")
