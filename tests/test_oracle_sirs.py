"""Pins for the oracle's SIR in continuous space (the paper's SIR benchmark,
PAPER.md Sec. 5.1.1 l.203 + Listing 2 l.134-145; C1-C4).
Expected values: scipy's KD-tree pair query (library), cuRAND-drawn positions
and keys + stable argsort, SPEC's worked special cases, and the single-draw
infection law (probability p whatever the number of infected contacts)."""
import numpy as np
import pytest
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


# ---------------------------------------------------------------------------
# Bit-level pin of the contact rule and the step's draw keying (C2/C3, R4/R7):
# contacts by a numpy float32 all-pairs evaluation of dx*dx + dy*dy <= r*r
# (each op rounded to float32, as the C oracle under -ffp-contract=off), and
# a columnar step whose draws come from cuRAND's Philox routine: one draw
# lane32(0x41, s, t) per exposed susceptible, recovery lane32(0x43, i, t).
# ---------------------------------------------------------------------------
TAG_TX, TAG_REC = 0x41, 0x43


def t_exact(p):
    import math
    from fractions import Fraction
    return 1 << 32 if p >= 1 else math.ceil(Fraction(p) * (1 << 32))


def numpy_contacts(px, py, r):
    dx = px[None, :] - px[:, None]  # [i, j] = x_j - x_i, float32
    dy = py[None, :] - py[:, None]
    d2 = dx * dx + dy * dy
    A = d2 <= np.float32(r) * np.float32(r)
    np.fill_diagonal(A, False)
    return A


def numpy_sirs_step(A, x, seed, t, p_inf, p_rec, curand_host):
    ids = np.arange(x.size, dtype=np.uint64)
    exposed = (A & (x == 1)[None, :]).any(axis=1)
    u_inf = curand_host.lane32(seed, TAG_TX, ids, t).astype(np.uint64)
    u_rec = curand_host.lane32(seed, TAG_REC, ids, t).astype(np.uint64)
    y = x.copy()
    y[(x == 0) & exposed & (u_inf < np.uint64(t_exact(p_inf)))] = 1
    y[(x == 1) & (u_rec < np.uint64(t_exact(p_rec)))] = 2
    return y


@pytest.mark.parametrize("seed,t0", [(9, 0), ((3 << 32) | 1, 5)])
def test_step_equals_curand_reformulation(orc, curand_host, seed, t0):
    n, L, r, k = 2500, 50.0, 2.0, 25
    px, py, x = orc.sirs_init(n, L, k, seed)
    A = numpy_contacts(px, py, r)
    rp, col = orc.sirs_contacts(px, py, r)
    B = np.zeros((n, n), bool)
    B[np.repeat(np.arange(n), np.diff(rp)), col] = True
    assert np.array_equal(A, B)  # contact lists bit-exact vs the float32 all-pairs rule
    run_state, counts = orc.sirs_run(rp, col, x, seed, 0.1, 0.05, t0, 22)
    ref, changed = x.copy(), 0
    for j in range(22):
        nxt = numpy_sirs_step(A, ref, seed, t0 + j, 0.1, 0.05, curand_host)
        assert np.array_equal(orc.sirs_step(rp, col, ref, seed, t0 + j, 0.1, 0.05), nxt), f"step {t0 + j}"
        assert counts[j].tolist() == [int((nxt == s).sum()) for s in range(3)]
        changed += int((nxt != ref).sum())
        ref = nxt
    assert np.array_equal(run_state, ref) and changed > 100


@pytest.mark.parametrize("n,L,r,seed", [(1, 10.0, 1.0, 1), (40, 3.0, 2.5, 2), (3000, 60.0, 2.0, 3),
                                        (2500, 31.0, 0.7, 4), (2000, 20.0, 7.9, 5)])
def test_grid_contacts_equal_brute_force(orc, n, L, r, seed):
    # the oracle's grid search (used at N = 1e7) equals its all-pairs definition
    px, py, _ = orc.sirs_init(n, L, 0, seed)
    rp, col = orc.sirs_contacts(px, py, r, cap=n * n + 1)
    rp2, col2 = orc.sirs_contacts_grid(px, py, L, r, cap=n * n + 1)
    assert np.array_equal(rp, rp2) and np.array_equal(col, col2)
