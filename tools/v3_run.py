#!/usr/bin/env python
"""V3 (SURVEY 8(d) variant: Boids N = 1e8, L = 31,623) stepped in the bench
configuration, for ncu captures:  python tools/v3_run.py [steps]"""
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_16292_b200 import Model, boids_params  # noqa: E402
from paper_2601_16292_b200.workloads import V3_BOIDS_SCALE as c  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else c["steps"]
K = ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")
m = Model("boids", c["n"], boids_params(*[c[k] for k in K]), c["seed"])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
m.synchronize()
e0.record(m.stream)
m.step(steps)
e1.record(m.stream)
m.synchronize()
print(f"V3 {steps} steps: {e0.elapsed_time(e1) / steps:.4f} ms/step, mean speed = {m.metrics('mean_speed')[-1]:.6f}")
m.close()
