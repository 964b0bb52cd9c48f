"""Build libamber.so (the product's C-ABI library) in-tree for sm_100a.

Each csrc/*.cu is compiled with nvcc -gencode arch=compute_100a,code=sm_100a
-lineinfo and linked into paper_2601_16292_b200/libamber.so (the .so travels
to the GPU box with the repo snapshot).  boids.cu is compiled with
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


def _flags(src: str) -> list[str]:
    f = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", nccl_include(),
         "--expt-relaxed-constexpr"] + ARCH + EXTRA
    if os.path.basename(src) in ("boids.cu", "population.cu"):
        f += ["-fmad=false", "-prec-div=true", "-prec-sqrt=true"]
    return f


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "amber.h")]
    if os.path.exists(obj) and all(os.path.getmtime(obj) >= os.path.getmtime(d) for d in deps):
        return obj, ""
    r = subprocess.run([NVCC, "-c", src, "-o", obj] + _flags(src), capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    log = os.path.join(BUILD, os.path.basename(src) + ".ptxas.txt")
    with open(log, "w") as fh:
        fh.write(r.stderr)
    return obj, r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(_compile, srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        cmd = [NVCC, "-shared", "-o", OUT] + objs + ARCH + ["-lcudart_static", "-ldl", "-lpthread", "-lrt"]
        subprocess.check_call(cmd)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
