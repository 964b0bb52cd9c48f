"""Small end-to-end run of every kernel family (for compute-sanitizer):
python tools/sanitize_small.py"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_16292_b200 import (Model, boids_params, loopback_id, sir_params, sir_space_params,  # noqa: E402
                                   sweep, walk_params, wealth_params)


def run_sharded(kind, n, params, seed, world, fn):
    uid = loopback_id()
    ms = [Model(kind, n, params, seed, rank=r, world=world, unique_id=uid, torch_alloc=False) for r in range(world)]
    th = [threading.Thread(target=fn, args=(mm,)) for mm in ms]
    [t.start() for t in th]
    [t.join() for t in th]
    for mm in ms:
        mm.close()


m = Model("wealth", 5003, wealth_params(), 1, torch_alloc=False); m.step(5); m.read_column("wealth"); m.close()
m = Model("wealth", 70_001, wealth_params(counter_bits=2), 2, torch_alloc=False); m.set_option("digest", 1); m.step(6); m.read_column("wealth"); m.close()
m = Model("wealth", 300_000, wealth_params(), 3, torch_alloc=False); m.set_option("persistent", 0); m.step(3); m.read_column("wealth"); m.close()
m = Model("sir", 20_000, sir_params(), 7, torch_alloc=False); m.step(10); m.set_option("persistent", 0); m.step(3); m.read_column("state"); m.close()
m = Model("sir", 300_000, sir_params(), 8, torch_alloc=False); m.set_option("digest", 1); m.step(12); m.read_column("state"); m.close()
m = Model("boids", 4000, boids_params(L=200.0), 3, torch_alloc=False); m.step(3); m.set_option("lanes", 8); m.step(2); m.set_option("lanes", 16); m.step(2); m.read_column("pos_x"); m.close()
m = Model("boids", 30_000, boids_params(L=3000.0), 5, torch_alloc=False); m.step(3); m.read_column("vel_x"); m.close()
m = Model("sir_space", 5000, sir_space_params(L=70.0), 3, torch_alloc=False); m.step(5); m.read_column("state"); m.close()
m = Model("walk", 5000, walk_params(), 3, torch_alloc=False); m.step(5); m.read_column("pos_x"); m.close()
print(sweep(2000, sir_params(8.0, 0.0, 0.1, 0.01), [0.05, 0.2], [1, 2], 50, torch_alloc=False))
run_sharded("wealth", 9001, wealth_params(), 4, 2, lambda mm: (mm.step(4), mm.read_column("wealth")))
run_sharded("sir", 9001, sir_params(), 4, 3, lambda mm: (mm.step(6), mm.read_column("state")))
run_sharded("boids", 3000, boids_params(L=150.0), 4, 3, lambda mm: (mm.step(4), mm.read_column("pos_x")))
print("sanitize run ok")
