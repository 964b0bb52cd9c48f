#!/usr/bin/env python
"""SIR step time vs agents per lane ("apl") of the step kernels: C2 (N = 1e5,
200 steps) and V2 (N = 1e8, 20 steps), default direction-optimizing
persistent launch, CUDA events.  python tools/sir_apl_probe.py"""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_16292_b200 import Model, sir_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402


def run(c, apl, reps):
    p = sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"])
    out = []
    for _ in range(reps):
        m = Model("sir", c["n"], p, c["seed"])
        m.set_option("apl", apl)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(m.stream)
        m.step(c["steps"])
        e1.record(m.stream)
        m.synchronize()
        out.append(e0.elapsed_time(e1) / c["steps"])
        d = m.digest("state")
        m.close()
    return min(out), d


res = {}
for name, c, reps in (("c2", W.C2_SIR, 5), ("v2", W.V2_SIR_SCALE, 1)):
    digs = set()
    for apl in (1, 2, 4, 8):
        ms, d = run(c, apl, reps)
        digs.add(d)
        res[f"{name}_apl{apl}_ms"] = ms
    assert len(digs) == 1
print(json.dumps(res))
