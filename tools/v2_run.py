#!/usr/bin/env python
"""V2 (SURVEY 8(d) variant: SIR on G(1e8, 5e8)) built once and stepped 20
steps in the bench configuration (one persistent direction-optimizing launch),
for ncu captures:  python tools/v2_run.py [steps]"""
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_16292_b200 import Model, sir_params  # noqa: E402
from paper_2601_16292_b200.workloads import V2_SIR_SCALE as c  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else c["steps"]
m = Model("sir", c["n"], sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"]), c["seed"])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
m.synchronize()
e0.record(m.stream)
m.step(steps)
e1.record(m.stream)
m.synchronize()
print(f"V2 {steps} steps: {e0.elapsed_time(e1) / steps:.4f} ms/step, I = {m.metrics('I')[-1]}")
m.close()
