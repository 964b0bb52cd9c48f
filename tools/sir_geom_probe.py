"""C2 and V2 step time of the current libamber (AMBER_LIB_PATH) -- launch-geometry probe."""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_16292_b200 import Model, sir_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

out = {}
for key, c, k in (("c2", W.C2_SIR, 200), ("v2", W.V2_SIR_SCALE, 20)):
    m = Model("sir", c["n"], sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"]), c["seed"])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    m.step(k)
    e1.record(m.stream)
    m.synchronize()
    out[key] = e0.elapsed_time(e1) / k
    m.close()
print(json.dumps(out))
