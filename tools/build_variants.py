"""Build tuning variants of libvpetabc.so into tune/ (compile-time VPET_TILE / VPET_SUPER / VPET_CH)."""
import concurrent.futures as cf
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14859_b200 import build as B  # noqa: E402

VARIANTS = {
    "v3s025": ("VPET_VOXKEY=3", "VPET_VOXS=0.25f"),
    "v3s0125": ("VPET_VOXKEY=3", "VPET_VOXS=0.125f"),
    "v3a": ("VPET_VOXKEY=3", "VPET_VOXS=0.35f", "VPET_VOXS3=0.12f"),
    "v3b": ("VPET_VOXKEY=3", "VPET_VOXS=0.25f", "VPET_VOXS3=0.5f"),
    "v4s025": ("VPET_VOXKEY=4", "VPET_VOXS=0.25f"),
    "v4a": ("VPET_VOXKEY=4", "VPET_VOXS=0.35f", "VPET_VOXS3=0.12f"),
}
names = sys.argv[1:] or list(VARIANTS)
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tune")
os.makedirs(root, exist_ok=True)
with cf.ThreadPoolExecutor(max_workers=2) as ex:
    futs = {n: ex.submit(B.build, True, False, os.path.join(root, f"libvpetabc_{n}.so"), VARIANTS[n] or ("VPET_BASE=1",))
            for n in names}
    for n, f in futs.items():
        print(n, f.result(), flush=True)
