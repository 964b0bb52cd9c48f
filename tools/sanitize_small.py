"""Small end-to-end run of every kernel family (for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import threading
import numpy as np
from paper_2601_16292_b200 import Model, wealth_params, sir_params, boids_params, sweep, loopback_id

m = Model("wealth", 5003, wealth_params(), 1, torch_alloc=False); m.step(5); m.read_column("wealth"); m.close()
m = Model("wealth", 70_001, wealth_params(counter_bits=2), 2, torch_alloc=False); m.set_option("digest", 1); m.step(6); m.read_column("wealth"); m.close()
m = Model("wealth", 300_000, wealth_params(counter_bits=-1), 3, torch_alloc=False); m.step(3); m.read_column("wealth"); m.close()
m = Model("sir", 20_000, sir_params(), 7, torch_alloc=False); m.step(10); m.set_option("persistent", 0); m.step(3); m.read_column("state"); m.close()
m = Model("boids", 4000, boids_params(L=200.0), 3, torch_alloc=False); m.step(3); m.set_option("tiled", 1); m.step(2); m.set_option("tiled", 0); m.set_option("fused", 1); m.step(2); m.read_column("pos_x"); m.close()
print(sweep(2000, sir_params(8.0, 0.0, 0.1, 0.01), [0.05, 0.2], [1, 2], 50, torch_alloc=False))
uid = loopback_id()
ms = [Model("wealth", 9001, wealth_params(), 4, rank=r, world=2, unique_id=uid, torch_alloc=False) for r in range(2)]
th = [threading.Thread(target=lambda mm: (mm.step(4), mm.read_column("wealth")), args=(mm,)) for mm in ms]
[t.start() for t in th]; [t.join() for t in th]
print("sanitize run ok")
