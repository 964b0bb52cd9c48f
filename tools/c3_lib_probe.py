#!/usr/bin/env python
"""C3 Boids us/step (100 steps from creation, best of 3) with the library at
AMBER_LIB_PATH (build variants), digest printed for the identity check.
python tools/c3_lib_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2601_16292_b200 import Model, boids_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

c = W.C3_BOIDS
bp = boids_params(*[c[k] for k in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")])
best, dig = None, None
for _ in range(3):
    m = Model("boids", c["n"], bp, c["seed"])
    m.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    m.step(c["steps"])
    e1.record(m.stream)
    m.synchronize()
    ms = e0.elapsed_time(e1) / c["steps"]
    best = ms if best is None else min(best, ms)
    dig = m.digest("pos_x")
    m.close()
print(os.environ.get("AMBER_LIB_PATH", "default"), f"{best * 1e3:.2f} us/step", dig)
