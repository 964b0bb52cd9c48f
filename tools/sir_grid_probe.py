#!/usr/bin/env python
"""C2 SIR step time vs persistent grid size and agents per lane (latency-bound
regime: the grid barrier vs. work per warp).  python tools/sir_grid_probe.py"""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_16292_b200 import Model, sir_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

c = W.C2_SIR
p = sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"])
res = {}
for apl in (1, 2):
    for grid in (0, 74, 148, 222, 296, 444):
        best = 1e9
        for _ in range(3):
            m = Model("sir", c["n"], p, c["seed"])
            m.set_option("apl", apl)
            m.set_option("grid", grid)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(m.stream)
            m.step(c["steps"])
            e1.record(m.stream)
            m.synchronize()
            best = min(best, e0.elapsed_time(e1) / c["steps"] * 1e3)
            m.close()
        res[f"apl{apl}_grid{grid}_us"] = round(best, 3)
print(json.dumps(res))
