#!/usr/bin/env python
"""Fixed cost of a V2-size push step: N = 1e8, mean degree 10, one forced-push
step (one cooperative launch) from init fractions 1e-6 .. 1e-2, CUDA events.
  python tools/v2_push_probe.py [init_frac ...]"""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_16292_b200 import Model, sir_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

c = W.V2_SIR_SCALE
fracs = [float(f) for f in sys.argv[1:]] or [1e-6, 1e-4, 1e-2]
for f in fracs:
    m = Model("sir", c["n"], sir_params(c["mean_degree"], c["beta"], c["gamma"], f), c["seed"])
    m.set_option("direction", 2)
    res = []
    for k in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(m.stream)
        m.step(1)
        e1.record(m.stream)
        m.synchronize()
        res.append(round(e0.elapsed_time(e1), 4))
    print(json.dumps({"init_frac": f, "I": int(m.metrics("I")[-1]), "push_ms": res}), flush=True)
    m.close()
