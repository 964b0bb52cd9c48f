"""Seeded synthetic workloads (BASELINE.json configs 1-5) -- inputs only.

This module holds the parameters and seeds of the five configurations and the
parameter-sweep layout.  It contains none of the method's arithmetic: every
population is generated *from these seeds* by each side's own counter-based
generator (DESIGN.md "Contract" R1-R8).  Both the CUDA path's tests/bench and
the oracle's callers read it; neither side imports the other.
"""
from __future__ import annotations

import numpy as np

# C1: wealth transfer, N = 1,000, w0 = 1, Philox seed 42, 100 steps (BJ config 1)
C1_WEALTH_SMALL = dict(kind="wealth", n=1_000, w0=1, amount=1, exclude_self=0, seed=42,
                       steps=100)

# C2: SIR on G(n, M), N = 1e5, mean degree 10, 1% initially infected,
# beta = 0.05, gamma = 0.1, 200 steps, seed 7 (BJ config 2)
C2_SIR = dict(kind="sir", n=100_000, mean_degree=10.0, beta=0.05, gamma=0.1, init_frac=0.01,
              seed=7, steps=200)

# C3: Boids, N = 1e5 in a 1000 x 1000 periodic box, R = 10, r_s = 2,
# weights (0.01, 0.125, 0.05), vmax 2, dt 1, 100 steps, seed 3 (BJ config 3)
C3_BOIDS = dict(kind="boids", n=100_000, L=1000.0, R=10.0, rs=2.0, wc=0.01, wa=0.125, ws=0.05,
                vmax=2.0, dt=1.0, seed=3, steps=100)

# C4: wealth at scale, N = 1e8, seed 11, 1000 steps, sharded over 1/2/4/8 GPUs (BJ config 4)
C4_WEALTH_SCALE = dict(kind="wealth", n=100_000_000, w0=1, amount=1, exclude_self=0, seed=11,
                       steps=1_000)

# C5: 4096 SIR replicates, N = 1e4, mean degree 8, 64 betas in [0.01, 0.2] x 64 seeds,
# gamma = 0.1, 300 steps (BJ config 5)
C5_SWEEP = dict(kind="sweep", n=10_000, mean_degree=8.0, gamma=0.1, init_frac=0.01, n_beta=64,
                n_seed=64, beta_lo=0.01, beta_hi=0.2, steps=300)

# NEXT-2: the paper's Random Walk benchmark at the paper's size
# (N = 10,000, 100 steps; Sec. 5.1.2 l.209) and at N = 1e8 (HBM-bound)
WALK_PAPER = dict(kind="walk", n=10_000, L=100.0, vmax=1.0, seed=3, steps=100)
WALK_SCALE = dict(kind="walk", n=100_000_000, L=10_000.0, vmax=1.0, seed=3, steps=100)

# NEXT-1: the paper's SIR benchmark in continuous space at the paper's
# size (N = 10,000, 100 steps) with SPEC's parameters (L = 100, r = 2,
# p_infect 0.1, p_recover 0.05, 1% infected), and at N = 1e7 with the same density
SIRS_PAPER = dict(kind="sir_space", n=10_000, L=100.0, r=2.0, p_infect=0.1, p_recover=0.05,
                  init_frac=0.01, seed=7, steps=100)
SIRS_SCALE = dict(kind="sir_space", n=10_000_000, L=3162.2776, r=2.0, p_infect=0.1, p_recover=0.05,
                  init_frac=0.01, seed=7, steps=100)

# SURVEY 8(d) added roofline variants (labelled as such; parity stays on C1-C5):
# V2 = C2's SIR at N = 1e8 (2M ~ 1e9 arcs, HBM-bound CSR streaming), 20 steps;
# V3 = C3's Boids at N = 1e8 with L = 31,623 (same density 0.1 per unit^2), 10 steps
V2_SIR_SCALE = dict(kind="sir", n=100_000_000, mean_degree=10.0, beta=0.05, gamma=0.1, init_frac=0.01,
                    seed=7, steps=20)
V3_BOIDS_SCALE = dict(kind="boids", n=100_000_000, L=31623.0, R=10.0, rs=2.0, wc=0.01, wa=0.125, ws=0.05,
                      vmax=2.0, dt=1.0, seed=3, steps=10)

CONFIGS = {"c1": C1_WEALTH_SMALL, "c2": C2_SIR, "c3": C3_BOIDS, "c4": C4_WEALTH_SCALE,
           "c5": C5_SWEEP, "walk": WALK_PAPER, "walk_scale": WALK_SCALE,
           "sirs": SIRS_PAPER, "sirs_scale": SIRS_SCALE, "v2": V2_SIR_SCALE, "v3": V3_BOIDS_SCALE}


def sweep_replicates(cfg=C5_SWEEP):
    """Contract S6: replicate r = n_seed*b + q (beta-major); beta_b equals
    numpy.linspace(lo, hi, n_beta)[b]; seed_r = r.  Returns (betas, seeds)."""
    betas_grid = np.linspace(cfg["beta_lo"], cfg["beta_hi"], cfg["n_beta"])
    betas = np.repeat(betas_grid, cfg["n_seed"]).astype(np.float64)
    seeds = np.arange(cfg["n_beta"] * cfg["n_seed"], dtype=np.uint64)
    return betas, seeds
