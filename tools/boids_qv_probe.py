#!/usr/bin/env python
"""Boids stencil A/B: the pre-quantised-velocity stencil (option qv=1, default
where valid) vs the float-velocity stencil (qv=0) at C3 and V3, per-kernel
device times from the library's event profiler.  python tools/boids_qv_probe.py"""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_16292_b200 import Model, boids_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

K = ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")
QVS = (1, 0) if "--quick" not in sys.argv else (1,)
LANES = (4, 8) if "--quick" not in sys.argv else (4,)
for name, c, steps in (("c3", W.C3_BOIDS, 100), ("v3", W.V3_BOIDS_SCALE, 10)):
    for qv in QVS:
        for lanes in LANES:
            m = Model("boids", c["n"], boids_params(*[c[k] for k in K]), c["seed"])
            m.set_option("qv", qv)
            m.set_option("lanes", lanes)
            m.step(1)
            m.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(m.stream)
            m.step(steps - 1)
            e1.record(m.stream)
            m.synchronize()
            ms = e0.elapsed_time(e1) / (steps - 1)
            m.profile(True)
            m.step(2)
            m.synchronize()
            prof = {k: round(t / n, 4) for k, n, t in m.profile_results()}
            print(json.dumps({"lib": os.environ.get("AMBER_LIB_PATH", "default"), "sx": m.get_option("x_subdivision"), "config": name, "qv": qv, "lanes": lanes, "ms_per_step": round(ms, 4),
                              "kernel_ms": prof}), flush=True)
            m.close()
