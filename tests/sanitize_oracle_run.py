"""Run every oracle entry point on small inputs (driven by
tests/test_oracle_sanitizers.py under AddressSanitizer + UBSan)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402

w, tot, act, dig = oracle.wealth_run(np.ones(1001, np.int32), 5, 0, 20, digests=True)
oracle.wealth_run(np.full(257, 3, np.int32), 9, 0, 5, amount=2, exclude_self=1)
oracle.wealth_run(np.ones(1, np.int32), 1, 0, 3)
rp, col, mu = oracle.er_graph(3000, 12000, 7)
st = oracle.sir_init(3000, 30, 7)
oracle.sir_run(rp, col, st, 7, 0.1, 0.1, 0, 15, digests=True)
oracle.sir_sweep(500, 6.0, 0.1, 0.02, np.array([0.05, 0.3]), np.array([1, 2], np.uint64), 30)
P = oracle.boids_params(L=200.0)
b = oracle.boids_init(1500, 200.0, 3)
b1 = oracle.boids_step(b, P)
oracle.boids_step(b, P, brute=True)
oracle.boids_step_sample(b, P, np.arange(0, 1500, 37))
oracle.boids_run(b, P, 3)
oracle.boids_step_f64(b, P)
oracle.boids_step(oracle.boids_init(3, 40.0, 1), oracle.boids_params(L=40.0))
px, py = oracle.walk_init(999, 50.0, 2)
oracle.walk_run(px, py, 50.0, 1.0, 2, 0, 5)
sx, sy, ss = oracle.sirs_init(2000, 40.0, 20, 4)
r1, c1 = oracle.sirs_contacts(sx, sy, 2.0)
r2, c2 = oracle.sirs_contacts_grid(sx, sy, 40.0, 2.0)
assert np.array_equal(r1, r2) and np.array_equal(c1, c2)
oracle.sirs_run(r1, c1, ss, 4, 0.2, 0.1, 0, 10)
oracle.digest(w)
oracle.digest(st)
print("oracle sanitizer run ok")
