"""Run C3 Boids for K steps (ncu captures of a late, clustered step):
python tools/c3_run.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_16292_b200 import Model, boids_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 100
c = W.C3_BOIDS
m = Model("boids", c["n"], boids_params(*[c[x] for x in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")]), c["seed"])
m.step(k)
m.synchronize()
print("candidates at the last step", m.get_option("stencil_candidates"))
m.close()
