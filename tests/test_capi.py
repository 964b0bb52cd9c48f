"""CPU checks of the boundary: the C-ABI library loads, exports every symbol
include/amber.h declares, and the product package never touches oracle/."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT


def header_functions():
    src = open(os.path.join(ROOT, "include", "amber.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(amber_\w+)\s*\(", src, flags=re.M)))


def test_header_parse_is_nonempty():
    fns = header_functions()
    assert "amber_model_create" in fns and "amber_sweep" in fns and len(fns) >= 18


def test_library_exports_every_header_symbol():
    from paper_2601_16292_b200 import capi
    L = capi.lib()
    for fn in header_functions():
        assert hasattr(L, fn), fn
    assert sorted(capi.SYMBOLS) == header_functions()
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (amber_\w+)", out))
    assert set(header_functions()) <= exported


def test_version_and_error_without_gpu():
    from paper_2601_16292_b200 import capi
    L = capi.lib()
    assert L.amber_version() == 1
    # a call that must fail cleanly (no CUDA device here, or bad args): never crashes
    h = C.c_void_p()
    p = capi.amber_wealth_params(1, 1, 0, 0)
    rc = L.amber_model_create(0, 0, C.byref(p), C.sizeof(p), 1, None, C.byref(h))
    assert rc == -1 and b"n_agents" in L.amber_last_error()
    rc = L.amber_model_create(7, 10, C.byref(p), C.sizeof(p), 1, None, C.byref(h))
    assert rc in (-2, -5)
    rc = L.amber_step(None, 1)
    assert rc == -1


def test_sass_is_sm100a():
    from paper_2601_16292_b200 import capi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2601_16292_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "amber_oracle" not in txt and "liboracle" not in txt, f


def test_only_allowed_places_import_oracle():
    # oracle/ is test infrastructure: besides tests/, only bench.py's reference /
    # cpu_baseline legs, __graft_entry__ (build + smoke) and the golden-file
    # writer (a script that calls nothing but oracle/) may import it
    allowed = {"bench.py", "__graft_entry__.py", os.path.join("tools", "make_oracle_goldens.py")}
    for dirpath, dirs, files in os.walk(ROOT):
        rel = os.path.relpath(dirpath, ROOT)
        if rel.split(os.sep)[0] in ("tests", "oracle", ".git", "baseline", "gpurun_out"):
            continue
        for f in files:
            if not f.endswith(".py"):
                continue
            path = os.path.normpath(os.path.join(rel, f))
            txt = open(os.path.join(dirpath, f), errors="ignore").read()
            if re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M):
                assert path in allowed, path


@pytest.mark.parametrize("workload", ["c1", "c2"])
def test_bench_reference_arm_small_workloads(workload):
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", workload,
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["workload"] == workload
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_bounds_build_carries_device_checks():
    # the AMBER_BOUNDS library (built by __graft_entry__.build) contains the
    # device-side check messages; the product library does not
    import os
    pkg = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2601_16292_b200")
    prod, bnd = os.path.join(pkg, "libamber.so"), os.path.join(pkg, "libamber_bounds.so")
    if not os.path.exists(bnd):
        import pytest
        pytest.skip("bounds build not present (run __graft_entry__.build())")
    assert b"AMBER_BOUNDS" in open(bnd, "rb").read()
    assert b"AMBER_BOUNDS" not in open(prod, "rb").read()
