"""Run a few C4 wealth steps with a chosen scatter (for ncu captures):
python tools/wealth_run.py [counter_bits] [steps] [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_16292_b200 import Model, wealth_params  # noqa: E402

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n = int(float(sys.argv[3])) if len(sys.argv) > 3 else 100_000_000
m = Model("wealth", n, wealth_params(counter_bits=bits), 11)
m.step(steps)
m.synchronize()
print("scatter", m.get_option("scatter"), "replays", m.get_option("replays"))
m.close()
