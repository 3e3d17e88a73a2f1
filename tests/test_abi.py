"""CPU checks of the boundary: the CUDA library loads and exports every symbol include/vpetabc.h
declares; the ctypes structs match the header layout; argument validation (no GPU needed for the
calls that fail before touching a device)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "vpetabc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:abc_status|const char\*|void|uint32_t)\s+(abc_\w+)\s*\(", src, re.M)))


def test_header_declares_the_north_star_entry_points():
    syms = header_symbols()
    for s in ("abc_init", "abc_set_input_function", "abc_set_frames", "abc_run_voxels", "abc_model_select"):
        assert s in syms


def test_library_loads_and_exports_every_header_symbol():
    from paper_2603_14859_b200 import _abi
    lib = _abi.load_library()
    for s in header_symbols():
        assert hasattr(lib, s), s
    assert set(header_symbols()) == set(_abi.SYMBOLS)
    assert lib.abc_abi_version() == 2


def test_struct_layouts():
    from paper_2603_14859_b200 import _abi
    assert C.sizeof(_abi.ModelSpec) == 80
    assert C.sizeof(_abi.Config) == 376
    assert _abi.Config.model.offset == 56
    assert C.sizeof(_abi.Result) == 11 * 8
    assert C.sizeof(_abi.Stats) == 4 + 4 + 8 * 6 + 4 + 4 + 8 * 8


def test_init_rejects_bad_configs_before_touching_a_device():
    from paper_2603_14859_b200 import AbcContext, AbcError
    lo, hi = [0.001, 0.001, 0.001, 0.0, 0.03], [1.0, 2.0, 0.5, 0.1, 0.2]
    bad = [
        dict(models=[dict(kind="2TCM_REV", n_draws=10, lo=lo, hi=hi)], n_accept=11),        # n > N
        dict(models=[dict(kind="2TCM_REV", n_draws=10, lo=lo, hi=hi)], n_accept=0),         # n = 0
        dict(models=[dict(kind="2TCM_REV", n_draws=10, lo=hi, hi=lo)], n_accept=1),         # lo > hi
        dict(models=[dict(kind="2TCM_REV", n_draws=10, lo=[0.1, 0.1, 0.0, 0, 0.1], hi=hi)], n_accept=1),  # k3 lo 0
        dict(models=[dict(kind="2TCM_REV", n_draws=10, lo=lo, hi=hi),
                     dict(kind="MRTM", n_draws=10, lo=[0.5] * 7, hi=[1.0] * 7)], n_accept=1),            # mixed families
        dict(models=[dict(kind="2TCM_REV", n_draws=10, lo=lo, hi=hi)], accept="EPS", epsilon=-1.0),
        dict(models=[dict(kind="2TCM_REV", n_draws=2 ** 32, lo=lo, hi=hi)], n_accept=1),
        dict(models=[dict(kind="2TCM_REV", n_draws=100000, lo=lo, hi=hi)], n_accept=15361),  # n > 15360
    ]
    for kw in bad:
        with pytest.raises(AbcError) as e:
            AbcContext(**kw)
        assert e.value.status == 1, kw


def test_bench_reference_arm_json_contract():
    """bench.py --impl reference (the CPU oracle arm) prints one JSON line with the contract's keys."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--cpu-voxels", "2", "--cpu-draws", "2000"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
