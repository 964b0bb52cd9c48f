#!/usr/bin/env python
"""Per-step device time of the V2 SIR variant (N = 1e8) by direction: two
models with the same seed step through the same states (S3: identical
results), one forced to pull, one forced to push; each step is one cooperative
launch timed with CUDA events.  Step 0 pulls on both (push needs the previous
counts).  Prints one JSON object.
  python tools/v2_steps.py [steps]
"""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_16292_b200 import Model, sir_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402


def timed_step(m):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    m.step(1)
    e1.record(m.stream)
    m.synchronize()
    return e0.elapsed_time(e1)


c = W.V2_SIR_SCALE
steps = int(sys.argv[1]) if len(sys.argv) > 1 else c["steps"]
p = sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"])
ms = {}
for d in (1, 2):
    m = Model("sir", c["n"], p, c["seed"])
    m.set_option("direction", d)
    rows = []
    for k in range(steps):
        t = timed_step(m)
        rows.append(dict(step=k, ms=t, S=int(m.metrics("S")[-1]), I=int(m.metrics("I")[-1])))
    ms[d] = rows
    dig = m.digest("state")
    m.close()
    ms[f"digest{d}"] = dig
assert ms["digest1"] == ms["digest2"]
out = [dict(step=a["step"], S_after=a["S"], I_after=a["I"], pull_ms=a["ms"], push_ms=b["ms"])
       for a, b in zip(ms[1], ms[2])]
print(json.dumps(dict(variant="V2 per-step by direction", rows=out,
                      auto_ms=sum(min(r["pull_ms"], r["push_ms"]) for r in out))))
