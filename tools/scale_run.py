"""Run a few steps of the V2 (SIR N=1e8) or V3 (Boids N=1e8) variant, for ncu:
python tools/scale_run.py v2|v3 [steps] [persistent]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_16292_b200 import Model, boids_params, sir_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

which = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pers = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if which == "v2":
    c = W.V2_SIR_SCALE
    m = Model("sir", c["n"], sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"]), c["seed"])
else:
    c = W.V3_BOIDS_SCALE
    m = Model("boids", c["n"], boids_params(*[c[k] for k in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")]),
              c["seed"])
m.set_option("persistent", pers)
m.step(steps)
m.synchronize()
print(which, "ok", m.step_count)
m.close()
