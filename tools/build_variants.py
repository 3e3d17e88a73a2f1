"""Build tuning variants of libvpetabc.so (compile-time VPET_* knobs) into paper_2603_14859_b200/_variants/
(git-ignored *.so, but shipped to the GPU box by gpurun); select one with VPET_LIB=<path>.

python tools/build_variants.py base acc2 ...
"""
import concurrent.futures as cf
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14859_b200 import build as B  # noqa: E402

VARIANTS = {
    "base": (),
    "acc2": ("VPET_ACC2=1",),
    "tr3": ("VPET_TREFRESH=3",),
    "tr4": ("VPET_TREFRESH=4",),
    "hinl": ("VPET_HEAP_INLINE=1",),
    "pair": ("VPET_PAIR=1",),
    "nt128": ("VPET_NT=128",),
    "nt32": ("VPET_NT=32",),
    "hsort512": ("VPET_HSORTMAX=512",),
    "qorder0": ("VPET_QORDER=0",),
    "union": ("VPET_UNION_STATS=1",),
    "pushstats": ("VPET_PUSH_STATS=1",),
    "trav": ("VPET_TRAV_STATS=1",),
    "nocontig": ("VPET_WARP_CONTIG=0",),
    "morton": ("VPET_HILBERT=0",),
    "hbank": ("VPET_HILBERT=1", "VPET_HILBERT_VOX=0"),
    "hvox": ("VPET_HILBERT=0", "VPET_HILBERT_VOX=1"),
    "union_contig": ("VPET_UNION_STATS=1",),
    "minb9": ("VPET_MINB=9",),
    "minb10": ("VPET_MINB=10",),
    "nst3": ("VPET_NST=3",),
    "ch12": ("VPET_CH=12",),
    "ch20": ("VPET_CH=20",),
    "ch24": ("VPET_CH=24",),
    "ch36": ("VPET_CH=36",),
    "ch36b12": ("VPET_CH=36", "VPET_CHB=12"),
    "ch36b16": ("VPET_CH=36", "VPET_CHB=16"),
    "ch36b20": ("VPET_CH=36", "VPET_CHB=20"),
    "old16": ("VPET_CH=16", "VPET_CHB=16"),
    "super4": ("VPET_SUPER=4",),
    "super16": ("VPET_SUPER=16",),
    "nst3b": ("VPET_NST=3",),
    "tile16": ("VPET_TILE=16",),
    "chb8": ("VPET_CHB=8",),
    "c3ch32": ("VPET_CH=32", "VPET_CHB=12"),
    "tr3acc2": ("VPET_TREFRESH=3", "VPET_ACC2=1"),
    "npc3": ("VPET_NPC=3",),
    "npc5": ("VPET_NPC=5",),
    "quota0": ("VPET_QUOTA=0",),
    "rpair0": ("VPET_RPAIR=0",),
    "tr0": ("VPET_TREFRESH=0",),
    "boxhead4": ("VPET_BOXHEAD=4",),
    "href1": ("VPET_HREFRESH=1",),
    "s1h3": ("VPET_REFRESH=1", "VPET_HREFRESH=3"),
    "s3h3": ("VPET_REFRESH=3", "VPET_HREFRESH=3"),
    "s1h7": ("VPET_REFRESH=1", "VPET_HREFRESH=7"),
    "sref1": ("VPET_REFRESH=1",),
    "href3": ("VPET_HREFRESH=3",),
    "h16box4": ("VPET_HEAD=16", "VPET_BOXHEAD=4"),
    "h16box8": ("VPET_HEAD=16", "VPET_BOXHEAD=8"),
    "h12box8": ("VPET_HEAD=12", "VPET_BOXHEAD=8"),
    "h12box4": ("VPET_HEAD=12", "VPET_BOXHEAD=4"),
    "rhinl": ("VPET_HEAP_INLINE=1",),
    "rssort0": ("VPET_SSORT=0",),
    "rqorder0": ("VPET_QORDER=0",),
    "rhsort512": ("VPET_HSORTMAX=512",),
    "rhsort128": ("VPET_HSORTMAX=128",),
    "certminb6": ("CERT_MINB=6",),
    "certminb8": ("CERT_MINB=8",),
    "certminb3": ("CERT_MINB=3",),
    "rnt128": ("VPET_NT=128",),
    "rnt128m4": ("VPET_NT=128", "VPET_MINB_ROT=4"),
    "voxkey4": ("VPET_VOXKEY=4",),
    "vk4s05": ("VPET_VOXKEY=4", "VPET_VOXS=0.5f"),
    "vk4s1": ("VPET_VOXKEY=4", "VPET_VOXS=1.0f"),
    "voxs05": ("VPET_VOXS=0.5f",),
    "voxs1": ("VPET_VOXS=1.0f",),
    "voxs0125": ("VPET_VOXS=0.125f",),
    "rnst3": ("VPET_NST=3",),
    "tr1": ("VPET_TREFRESH=1",),
    "sheap1": ("VPET_SHEAP=1",),
    "h12m6": ("VPET_HEAD=12", "VPET_MINB_ROT=6"),
    "h12m8": ("VPET_HEAD=12", "VPET_MINB_ROT=8"),
    "h12": ("VPET_HEAD=12",),
    "tr0ref0": ("VPET_TREFRESH=0", "VPET_REFRESH=0"),
    "head4": ("VPET_HEAD=4",),
    "head12": ("VPET_HEAD=12",),
    "minb7": ("VPET_MINB=7",),
    "rtr3": ("VPET_TREFRESH=3",),
    "rtile16": ("VPET_TILE=16",),
    "rsuper4": ("VPET_SUPER=4",),
    "rsuper16": ("VPET_SUPER=16",),
    "rchb8": ("VPET_CHB=8",),
    "rchb16": ("VPET_CHB=16",),
    "r1ch12": ("VPET_R=1", "VPET_CH=12"),
    "r1ch16": ("VPET_R=1", "VPET_CH=16"),
    "r1ch36": ("VPET_R=1", "VPET_CH=36"),
    "r1ch12m12": ("VPET_R=1", "VPET_CH=12", "VPET_MINB=12"),
    "r1nt128ch12": ("VPET_R=1", "VPET_CH=12", "VPET_NT=128"),
    "r1nt128ch16": ("VPET_R=1", "VPET_CH=16", "VPET_NT=128"),
}
names = sys.argv[1:] or list(VARIANTS)
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2603_14859_b200", "_variants")
os.makedirs(root, exist_ok=True)
with cf.ThreadPoolExecutor(max_workers=2) as ex:
    futs = {n: ex.submit(B.build, True, False, os.path.join(root, f"libvpetabc_{n}.so"), VARIANTS[n] or ("VPET_BASE=1",))
            for n in names}
    for n, f in futs.items():
        print(n, f.result(), flush=True)
