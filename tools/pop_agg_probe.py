"""Time a Population aggregate at 1e8 rows (interpreter path)."""
import os
import sys
import time

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_16292_b200.population import Population, col  # noqa: E402

n = 100_000_000
p = Population({"wealth": "i32", "state": "u8"}, capacity=n)
p.add_agents(n, wealth=3, state=0)
p.aggregate("sum", col("wealth"), where=col("state") == 0)
t0 = time.perf_counter()
for _ in range(10):
    v = p.aggregate("sum", col("wealth"), where=col("state") == 0)
dt = (time.perf_counter() - t0) / 10
print({"ms_per_aggregate": dt * 1e3, "value": v, "GBps": 6.0 * n / dt / 1e9})
