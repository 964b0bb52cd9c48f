#!/usr/bin/env python
"""Boids step time vs lanes per agent in the stencil (option "lanes"), C3 (100
steps from creation) and V3 (steps 1..9): identical results (digest checked).
python tools/boids_lanes_probe.py"""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_16292_b200 import Model, boids_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

res = {}
for name, c, first, k in (("c3", W.C3_BOIDS, 0, 100), ("v3", W.V3_BOIDS_SCALE, 1, 9)):
    bp = boids_params(*[c[x] for x in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")])
    digs = set()
    for lanes in (4, 8, 16):
        m = Model("boids", c["n"], bp, c["seed"])
        m.set_option("lanes", lanes)
        if first:
            m.step(first)
        m.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(m.stream)
        m.step(k)
        e1.record(m.stream)
        m.synchronize()
        res[f"{name}_lanes{lanes}_ms"] = round(e0.elapsed_time(e1) / k, 4)
        digs.add(m.digest("pos_x"))
        m.close()
    assert len(digs) == 1
print(json.dumps(res))
