"""CPU checks of the oracle-written full-size golden files (tools/make_oracle_goldens.py):
format, exact-ratio consistency and the invariants the paper fixes (wealth is
conserved; R fractions lie in [0, 1] and rise with beta)."""
import os

import numpy as np
import pytest

from paper_2601_16292_b200.workloads import C4_WEALTH_SCALE, C5_SWEEP, sweep_replicates

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rows(name):
    return [ln.split() for ln in open(os.path.join(GOLD, name)) if not ln.startswith("#")]


def test_c5_golden_consistent():
    r = rows("c5_sweep_oracle.txt")
    betas, _ = sweep_replicates(C5_SWEEP)
    assert len(r) == 4096 and [int(x[0]) for x in r] == list(range(4096))
    assert np.array_equal(np.array([float(x[1]) for x in r]), betas)
    cnt = np.array([int(x[2]) for x in r])
    frac = np.array([float(x[3]) for x in r])
    assert np.array_equal(frac, cnt / C5_SWEEP["n"])  # exact ratios (S5)
    assert (cnt >= 100).all() and (cnt <= C5_SWEEP["n"]).all()  # the 1% initially infected recover (gamma > 0)
    per_beta = frac.reshape(64, 64).mean(axis=1)
    assert per_beta[-1] > 0.95 and per_beta[0] < 0.3 and per_beta[-1] > per_beta[0]


def test_c4_golden_consistent():
    path = os.path.join(GOLD, "c4_wealth_oracle.txt")
    if not os.path.exists(path):
        pytest.skip("c4 golden not generated yet")
    raw = [[int(v) for v in x] for x in rows("c4_wealth_oracle.txt")]
    assert all(0 <= x[1] < 2 ** 64 for x in raw)  # D1 digests are uint64
    r = np.array([[x[0], x[2], x[3]] for x in raw], dtype=np.int64)  # step, total, active
    c = C4_WEALTH_SCALE
    assert r.shape == (c["steps"], 3) and (r[:, 0] == np.arange(c["steps"])).all()
    r = np.column_stack([r[:, 0], np.zeros(len(r), np.int64), r[:, 1], r[:, 2]])
    assert len({x[1] for x in raw}) == c["steps"]  # the column changes every step
    assert (r[:, 2] == c["n"] * c["w0"]).all()  # W pin (i): total wealth conserved at every step
    assert ((r[:, 3] > 0) & (r[:, 3] <= c["n"])).all()
    # active fraction settles near 2 - sqrt(2) (sanity band only)
    assert abs(r[-100:, 3].mean() / c["n"] - (2 - np.sqrt(2))) < 0.02


def test_v2_golden_consistent():
    from paper_2601_16292_b200.workloads import V2_SIR_SCALE as c
    lines = rows("v2_sir_oracle.txt")
    g = dict(zip(lines[0][1::2], (int(v) for v in lines[0][2::2])))
    m = int(np.floor(c["n"] * c["mean_degree"] / 2 + 0.5))
    assert g["arcs"] == 2 * g["edges"]
    dup = m - g["edges"]  # G4: expected duplicates M(M-1)/(N(N-1)) ~ 25
    assert 0 < dup < 80
    raw = [[int(v) for v in x] for x in lines[1:]]
    assert all(0 <= x[4] < 2 ** 64 for x in raw) and len({x[4] for x in raw}) == c["steps"]
    r = np.array([x[:4] for x in raw], dtype=np.int64)
    assert r.shape == (c["steps"], 4) and (r[:, 0] == np.arange(c["steps"])).all()
    assert (r[:, 1:4].sum(1) == c["n"]).all()  # S pin (i)
    assert (np.diff(r[:, 1]) <= 0).all() and (np.diff(r[:, 3]) >= 0).all()
