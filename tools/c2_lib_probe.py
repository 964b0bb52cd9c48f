#!/usr/bin/env python
"""C2 SIR us/step (200 steps from creation, best of 5) with the library at
AMBER_LIB_PATH (build variants), final digest for the identity check.
python tools/c2_lib_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2601_16292_b200 import Model, sir_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

c = W.C2_SIR
sp = sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"])
best, dig = None, None
for _ in range(5):
    m = Model("sir", c["n"], sp, c["seed"])
    m.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    m.step(c["steps"])
    e1.record(m.stream)
    m.synchronize()
    ms = e0.elapsed_time(e1) / c["steps"]
    best = ms if best is None else min(best, ms)
    dig = m.digest("state")
    m.close()
print(os.environ.get("AMBER_LIB_PATH", "default"), f"{best * 1e3:.3f} us/step", dig)
