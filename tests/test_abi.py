"""The C-ABI library builds for sm_100a, loads, and exports every entry point
include/gputx.h declares (no compute calls: runs without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gputx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gputx_[a-z_]+)\s*\(", src)))


def test_library_exports_header():
    from paper_1103_3105_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    names = _declared()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    from paper_1103_3105_b200 import gputx
    assert set(gputx.EXPORTED) == set(names)


def test_sass_is_sm100a():
    from paper_1103_3105_b200 import build
    out = subprocess.run(["cuobjdump", "--list-elf", build.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_out_stride_without_gpu():
    from paper_1103_3105_b200 import gputx
    lib = gputx.load_library()
    assert [lib.gputx_out_stride(s) for s in (1, 2, 3)] == [8, 40, 200]


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    from paper_1103_3105_b200 import gputx
    monkeypatch.setattr(gputx, "_lib", None)
    monkeypatch.setattr(gputx, "_LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        gputx.Database(1, (1, 1, 1, 0), 4)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1103_3105_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f


def test_bench_reference_arm_line():
    """bench.py --impl reference (the oracle as the reference arm) prints one JSON line
    with the contract's keys, on the host, without a GPU."""
    import json
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          "tpcb_tiny", "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["config"]["workload"].startswith("TPC-B tiny")
