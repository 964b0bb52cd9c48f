#!/usr/bin/env python
"""C3 Boids step time vs stencil-kernel grid size (0 = default cap of 8 blocks
per SM; larger grids let the block scheduler balance the flock-dependent work).
python tools/boids_grid_probe.py"""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_16292_b200 import Model, boids_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

c = W.C3_BOIDS
bp = boids_params(*[c[k] for k in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")])
res = {}
digs = set()
for grid in (0, 592, 2368, 3125, 6250):
    m = Model("boids", c["n"], bp, c["seed"])
    m.set_option("grid", grid)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    m.step(c["steps"])
    e1.record(m.stream)
    m.synchronize()
    res[f"grid{grid}_us"] = round(e0.elapsed_time(e1) / c["steps"] * 1e3, 2)
    digs.add(m.digest("pos_x"))
    m.close()
assert len(digs) == 1
print(json.dumps(res))
