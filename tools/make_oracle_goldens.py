#!/usr/bin/env python
"""Write oracle-only golden files for full-size parity tests (test infrastructure;
calls nothing but oracle/):

  tests/golden/c4_wealth_oracle.txt   BASELINE config 4 (N = 1e8, seed 11): for
      each of the 1,000 steps, the D1 digest of the wealth column, the total
      wealth and the number of agents with wealth > 0 (~1 h single-threaded)
  tests/golden/c5_sweep_oracle.txt    BASELINE config 5: the final R fraction of
      all 4,096 replicates as exact ratios R/N (~1-2 min, one process per core)

  tests/golden/v2_sir_oracle.txt      SURVEY 8(d) variant V2 (SIR on G(1e8, 5e8),
      seed 7): the D1 digests of the oracle's CSR row_ptr / col arrays (array
      index as id), then S, I, R and the state digest after each of the 20
      steps (~10 min, ~20 GB of host memory)

python tools/make_oracle_goldens.py [c4] [c5] [v2]
"""
import multiprocessing as mp
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402  (seeds and layout only)


def git_rev():
    try:
        return subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                              text=True).stdout.strip()
    except OSError:
        return "?"


def c4():
    c = W.C4_WEALTH_SCALE
    t0 = time.time()
    w = np.full(c["n"], c["w0"], np.int32)
    _, tot, act, dig = oracle.wealth_run(w, c["seed"], 0, c["steps"], amount=c["amount"],
                                         exclude_self=c["exclude_self"], digests=True)
    path = os.path.join(ROOT, "tests", "golden", "c4_wealth_oracle.txt")
    with open(path, "w") as f:
        f.write(f"# BASELINE config 4 (wealth N={c['n']}, seed {c['seed']}, w0 {c['w0']}, "
                f"{c['steps']} steps) by oracle/ (tools/make_oracle_goldens.py, repo {git_rev()}, "
                f"{time.time() - t0:.0f} s)\n# step digest total active\n")
        for t in range(c["steps"]):
            f.write(f"{t} {int(dig[t])} {int(tot[t])} {int(act[t])}\n")
    print("wrote", path)


def _rep(args):
    n, kbar, gamma, init_frac, beta, seed, steps = args
    return oracle.sir_sweep(n, kbar, gamma, init_frac, np.array([beta]), np.array([seed], np.uint64), steps)[0]


def c5():
    c = W.C5_SWEEP
    betas, seeds = W.sweep_replicates(c)
    t0 = time.time()
    jobs = [(c["n"], c["mean_degree"], c["gamma"], c["init_frac"], float(b), int(s), c["steps"])
            for b, s in zip(betas, seeds)]
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        res = pool.map(_rep, jobs, chunksize=16)
    path = os.path.join(ROOT, "tests", "golden", "c5_sweep_oracle.txt")
    with open(path, "w") as f:
        f.write(f"# BASELINE config 5 ({len(res)} SIR replicates, N={c['n']}, mean degree {c['mean_degree']}, "
                f"gamma {c['gamma']}, {c['steps']} steps; replicate r = 64*b + q, seed r) by oracle/ "
                f"(tools/make_oracle_goldens.py, repo {git_rev()}, {time.time() - t0:.0f} s)\n"
                f"# replicate beta R_count final_R_fraction\n")
        for r, (b, x) in enumerate(zip(betas, res)):
            f.write(f"{r} {float(b)!r} {int(round(x * c['n']))} {float(x)!r}\n")
    print("wrote", path)


def v2():
    c = W.V2_SIR_SCALE
    t0 = time.time()
    n = c["n"]
    m = oracle.round_count(n * c["mean_degree"] / 2.0)
    k = oracle.round_count(c["init_frac"] * n)
    rp, col, mu = oracle.er_graph(n, m, c["seed"])
    d_rp = oracle.digest(rp.view(np.uint32))
    d_col = oracle.digest(col.view(np.uint32))
    st = oracle.sir_init(n, k, c["seed"])
    _, counts, dig = oracle.sir_run(rp, col, st, c["seed"], c["beta"], c["gamma"], 0, c["steps"], digests=True)
    path = os.path.join(ROOT, "tests", "golden", "v2_sir_oracle.txt")
    with open(path, "w") as f:
        f.write(f"# SURVEY 8(d) variant V2 (SIR on G(n={n}, M={m}), seed {c['seed']}, beta {c['beta']}, gamma "
                f"{c['gamma']}, K={k} initially infected, {c['steps']} steps) by oracle/ "
                f"(tools/make_oracle_goldens.py, repo {git_rev()}, {time.time() - t0:.0f} s)\n")
        f.write(f"graph edges {mu} arcs {col.size} row_ptr_digest {d_rp} col_digest {d_col}\n")
        f.write("# step S I R state_digest\n")
        for t in range(c["steps"]):
            f.write(f"{t} {int(counts[t, 0])} {int(counts[t, 1])} {int(counts[t, 2])} {int(dig[t])}\n")
    print("wrote", path)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c5", "c4"]
    for w in which:
        {"c4": c4, "c5": c5, "v2": v2}[w]()
