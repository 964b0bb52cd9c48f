"""Time raw fused wealth launches (no overflow check / replay): experiment builds only.
python tools/wealth_time_raw.py [steps]"""
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_16292_b200 import Model, wealth_params  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 100
m = Model("wealth", 100_000_000, wealth_params(), 11)
m.set_option("metrics_capacity", 4 * k + 64)  # no window check inside the run
m.step(3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(m.stream)
m.step(k)
e1.record(m.stream)
torch.cuda.synchronize()
print({"ms_per_step": e0.elapsed_time(e1) / k})
