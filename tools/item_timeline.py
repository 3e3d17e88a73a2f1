"""Summarise a per-item scan timeline written with VPET_ITEMLOG=<file> (diagnostics).
python tools/item_timeline.py <file>"""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 4)
a = a[a[:, 1] > 0]
t0 = a[:, 0].min()
st = (a[:, 0] - t0) / 1e6
en = (a[:, 1] - t0) / 1e6
dur = en - st
T = en.max()
print(f"items {len(a)}  kernel span {T:.2f} ms  item ms: mean {dur.mean():.3f} p50 {np.median(dur):.3f} "
      f"p90 {np.percentile(dur, 90):.3f} p99 {np.percentile(dur, 99):.3f} max {dur.max():.3f}")
sm_end = {}
for s, e in zip(a[:, 2], en):
    sm_end[int(s)] = max(sm_end.get(int(s), 0.0), e)
ends = np.array(sorted(sm_end.values()))
print(f"SM last-item end: min {ends.min():.2f}  p10 {np.percentile(ends, 10):.2f}  p50 {np.median(ends):.2f}  max {ends.max():.2f} ms")
late = a[np.argsort(-en)[:10]]
print("last-finishing items (start, dur ms, vt):")
for r in late:
    print(f"  {(r[0]-t0)/1e6:7.2f} {(r[1]-r[0])/1e6:7.3f} vt={int(r[3])}")
order = np.argsort(st)
q = len(a) // 10
for k in range(10):
    sl = order[k * q:(k + 1) * q]
    print(f"  queue decile {k}: mean item {dur[sl].mean():.3f} ms  max {dur[sl].max():.3f}")
