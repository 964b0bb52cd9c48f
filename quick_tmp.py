import time, torch, numpy as np, sys
sys.path.insert(0,'.')
from paper_2601_16292_b200 import Model, wealth_params
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for bits in ((4, 8, 32) if steps > 10 else (4,)):
    m = Model('wealth', 100_000_000, wealth_params(counter_bits=bits), 11)
    m.step(5); m.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    m.profile(True)
    s.record(m.stream); m.step(steps); e.record(m.stream); m.synchronize()
    ms = s.elapsed_time(e)/steps
    print(f"bits={bits} ms/step={ms:.4f} agent-updates/s={1e8/ms*1e3:.3e}", m.profile_results(), flush=True)
    m.close()
