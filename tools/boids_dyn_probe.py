#!/usr/bin/env python
"""C3 Boids: static block order vs dynamic warp scheduling of the stencil
(option "dyn"), for 4 and 8 lanes per agent; 100 steps from creation, CUDA
events on the model stream, best of 3; final digests must agree.
python tools/boids_dyn_probe.py"""
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
res, digs = {}, set()
for lanes in (4, 8):
    for dyn in (0, 1):
        best = None
        for _ in range(3):
            m = Model("boids", c["n"], bp, c["seed"])
            m.set_option("lanes", lanes)
            m.set_option("dyn", dyn)
            m.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(m.stream)
            m.step(c["steps"])
            e1.record(m.stream)
            m.synchronize()
            ms = e0.elapsed_time(e1) / c["steps"]
            best = ms if best is None else min(best, ms)
            digs.add((m.digest("pos_x"), m.digest("vel_y")))
            m.close()
        res[f"lanes{lanes}_dyn{dyn}"] = round(best * 1e3, 2)
        print(lanes, dyn, f"{best * 1e3:.2f} us/step", flush=True)
print(json.dumps({"c3_us_per_step": res, "digests_agree": len(digs) == 1}))
