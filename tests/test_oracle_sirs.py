"""Pins for the oracle's SIR in continuous space (the paper's SIR benchmark,
PAPER.md Sec. 5.1.1 l.203 + Listing 2 l.134-145; C1-C4).
Expected values: scipy's KD-tree pair query (library), cuRAND-drawn positions
and keys + stable argsort, SPEC's worked special cases, and the single-draw
infection law (probability p whatever the number of infected contacts)."""
import numpy as np
from scipy.spatial import cKDTree

TAG_POS, TAG_INIT = 0x40, 0x42


def u01(x):
    return (np.asarray(x, np.uint32) >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)


def test_init_positions_and_infected(orc, curand_host):
    n, L, k, seed = 3000, 50.0, 30, 9
    px, py, st = orc.sirs_init(n, L, k, seed)
    i = np.arange(n, dtype=np.uint64)
    assert np.array_equal(px, np.float32(L) * u01(curand_host.lane32(seed, TAG_POS, 2 * i, 0)))
    assert np.array_equal(py, np.float32(L) * u01(curand_host.lane32(seed, TAG_POS, 2 * i + 1, 0)))
    keys = curand_host.lane64(seed, TAG_INIT, i, 0)
    assert set(np.nonzero(st == 1)[0].tolist()) == set(np.argsort(keys, kind="stable")[:k].tolist())


def test_contacts_equal_kdtree(orc):
    px, py, _ = orc.sirs_init(4000, 60.0, 0, 3)
    rp, col = orc.sirs_contacts(px, py, 2.0)
    pts = np.stack([px, py], 1).astype(np.float64)
    pairs = cKDTree(pts).query_pairs(2.0)
    d = lambda a, b: np.hypot(*(pts[a] - pts[b]))
    ours = {(i, j) for i in range(4000) for j in col[rp[i]:rp[i + 1]] if i < j}
    for a, b in ours ^ pairs:  # differences only at the float/double rounding of the boundary
        assert abs(d(a, b) - 2.0) < 1e-4
    assert len(ours ^ pairs) <= 2
    for i in range(0, 4000, 111):
        assert (np.diff(col[rp[i]:rp[i + 1]]) > 0).all()


def test_special_cases(orc):
    n, L = 500, 20.0
    px, py, st = orc.sirs_init(n, L, 5, 1)
    rp, col = orc.sirs_contacts(px, py, 2.0)
    _, c = orc.sirs_run(rp, col, st, 1, 0.0, 0.3, 0, 30)
    assert (c[:, 0] == n - 5).all()  # p_infect = 0: S constant
    rp2, col2 = orc.sirs_contacts(px, py, L * 1.5, cap=n * n)  # r >= L*sqrt(2): all contacts
    s1 = orc.sirs_step(rp2, col2, st, 1, 0, 1.0, 0.0)
    assert (s1 == 1).all()  # SPEC: p_recover = 0, p_infect = 1, full contact -> all infected after step 1


def test_single_draw_per_exposed_susceptible(orc):
    # P(infect) = p for any k_I >= 1 (Listing 2), not 1 - (1-p)^k_I
    k, p = 6, 0.1
    n = k + 1
    rp = np.array([0, k] + list(range(k + 1, 2 * k + 1)), np.int32)
    col = np.array(list(range(1, k + 1)) + [0] * k, np.int32)
    st = np.array([0] + [1] * k, np.uint8)
    hits = trials = 0
    for seed in range(300):
        for t in range(40):
            hits += int(orc.sirs_step(rp, col, st, seed, t, p, 0.0)[0] == 1)
            trials += 1
    sd = np.sqrt(p * (1 - p) / trials)
    assert abs(hits / trials - p) < 5 * sd


def test_invariants(orc):
    n = 5000
    px, py, st = orc.sirs_init(n, 70.0, 50, 4)
    rp, col = orc.sirs_contacts(px, py, 2.0)
    _, c = orc.sirs_run(rp, col, st, 4, 0.1, 0.05, 0, 120)
    assert (c.sum(1) == n).all() and (np.diff(c[:, 0]) <= 0).all() and (np.diff(c[:, 2]) >= 0).all()
