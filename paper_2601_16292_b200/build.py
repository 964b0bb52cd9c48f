"""Build libamber.so (the product's C-ABI library) in-tree for sm_100a.

Each csrc/*.cu is compiled with nvcc -gencode arch=compute_100a,code=sm_100a
-lineinfo and linked into paper_2601_16292_b200/libamber.so (the .so travels
to the GPU box with the repo snapshot).  `--bounds` (or build(bounds=True))
builds the same sources with -DAMBER_BOUNDS into libamber_bounds.so: device-side
index checks (AMBER_DCHECK) on every computed counter word, CSR arc, neighbour
id, cell run and sorted slot, for the bounds test (tests/test_gpu_bounds.py;
load it with AMBER_LIB_PATH, add AMBER_SYNC_DEBUG=1 to fault at the launch).  boids.cu is compiled with
-fmad=false as part of the float contract B7 (its arithmetic also uses
explicit _rn intrinsics, so the flag is belt and braces).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.environ.get("AMBER_BUILD_OUT") or os.path.join(PKG, "libamber.so")
BUILD = os.environ.get("AMBER_BUILD_DIR") or os.path.join(PKG, "build")
OUT_BOUNDS = os.path.join(PKG, "libamber_bounds.so")
BUILD_BOUNDS = os.path.join(PKG, "build_bounds")
EXTRA = os.environ.get("AMBER_NVCC_EXTRA", "").split()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_include() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc = os.path.join(base, "nccl", "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    return "/usr/include"


def _flags(src: str, bounds: bool = False) -> list[str]:
    f = (["-DAMBER_BOUNDS"] if bounds else []) + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", nccl_include(),
         "--expt-relaxed-constexpr"] + ARCH + EXTRA
    if os.path.basename(src) in ("boids.cu", "population.cu"):
        f += ["-fmad=false", "-prec-div=true", "-prec-sqrt=true"]
    return f


def _compile(src: str, bounds: bool = False) -> tuple[str, str]:
    bdir = BUILD_BOUNDS if bounds else BUILD
    obj = os.path.join(bdir, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "amber.h")]
    if os.path.exists(obj) and all(os.path.getmtime(obj) >= os.path.getmtime(d) for d in deps):
        return obj, ""
    r = subprocess.run([NVCC, "-c", src, "-o", obj] + _flags(src, bounds), capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    log = os.path.join(bdir, os.path.basename(src) + ".ptxas.txt")
    with open(log, "w") as fh:
        fh.write(r.stderr)
    return obj, r.stderr


def build(verbose: bool = False, bounds: bool = False) -> str:
    bdir, out = (BUILD_BOUNDS, OUT_BOUNDS) if bounds else (BUILD, OUT)
    os.makedirs(bdir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s_: _compile(s_, bounds), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if not os.path.exists(out) or any(os.path.getmtime(o) > os.path.getmtime(out) for o in objs):
        cmd = [NVCC, "-shared", "-o", out] + objs + ARCH + ["-lcudart_static", "-ldl", "-lpthread", "-lrt"]
        subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, bounds="--bounds" in sys.argv))
