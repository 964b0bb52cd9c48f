"""Pins for the oracle's G(n, M) graph (G1-G4) and SIR step (S1-S6).

Expected values come from scipy/numpy library routines (np.unique, scipy CSR
construction, breadth-first search), closed-form special cases (beta = 0,
gamma = 1, beta = 1), and binomial statistics of the per-edge rule, with draws
made by cuRAND's Philox routine rather than the oracle's generator.
"""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import breadth_first_order, shortest_path

from conftest import mulhi64_bigint
from paper_2601_16292_b200.workloads import C2_SIR, C5_SWEEP, sweep_replicates

TAG_GRAPH, TAG_INIT, TAG_TX, TAG_REC = 0x13, 0x12, 0x10, 0x11


def indep_graph(n, m, seed, curand_host):
    """G2/G3 with cuRAND draws + np.unique + scipy CSR (independent of the oracle)."""
    e = np.arange(m, dtype=np.uint64)
    u = mulhi64_bigint(curand_host.lane64(seed, TAG_GRAPH, 2 * e, 0), n)
    vp = mulhi64_bigint(curand_host.lane64(seed, TAG_GRAPH, 2 * e + 1, 0), n - 1)
    v = vp + (vp >= u)
    a, b = np.minimum(u, v), np.maximum(u, v)
    keys = np.unique(a.astype(np.int64) * n + b)
    a, b = keys // n, keys % n
    rows = np.concatenate([a, b])
    cols = np.concatenate([b, a])
    A = sp.csr_matrix((np.ones(rows.size, np.int8), (rows, cols)), shape=(n, n))
    A.sort_indices()
    return A.indptr.astype(np.int32), A.indices.astype(np.int32), keys.size


@pytest.mark.parametrize("n,m,seed", [(50, 200, 1), (1000, 5000, 7), (10_000, 40_000, 3)])
def test_graph_equals_library_construction(orc, curand_host, n, m, seed):
    rp, col, mu = orc.er_graph(n, m, seed)
    rp2, col2, mu2 = indep_graph(n, m, seed, curand_host)
    assert mu == mu2
    assert np.array_equal(rp, rp2) and np.array_equal(col, col2)


def test_graph_invariants(orc):
    n, m = 5000, 25_000
    rp, col, mu = orc.er_graph(n, m, 11)
    deg = np.diff(rp)
    assert deg.sum() == 2 * mu  # handshake
    src = np.repeat(np.arange(n), deg)
    assert (src != col).all()  # no self-loops
    for i in range(0, n, 97):
        row = col[rp[i]:rp[i + 1]]
        assert (np.diff(row) > 0).all()  # ascending, no multi-edges
    A = sp.csr_matrix((np.ones(col.size), (src, col)), shape=(n, n))
    assert (A != A.T).nnz == 0  # symmetric


def test_graph_duplicate_count_sanity(orc):
    # G4 sanity: expected duplicates M(M-1)/(N(N-1)) ~ 25 for C2
    m = orc.round_count(C2_SIR["n"] * C2_SIR["mean_degree"] / 2.0)
    _, _, mu = orc.er_graph(C2_SIR["n"], m, C2_SIR["seed"])
    dup = m - mu
    assert 5 < dup < 60


def test_init_selects_k_smallest_keys(orc, curand_host):
    # S1 pinned by a stable argsort of independently drawn keys
    n, k, seed = 3000, 30, 7
    st = orc.sir_init(n, k, seed)
    keys = curand_host.lane64(seed, TAG_INIT, np.arange(n, dtype=np.uint64), 0)
    want = np.argsort(keys, kind="stable")[:k]
    assert (st == 1).sum() == k and (st == 2).sum() == 0
    assert set(np.nonzero(st == 1)[0].tolist()) == set(want.tolist())


@pytest.fixture(scope="module")
def small_graph(orc):
    n, m = 4000, 20_000
    rp, col, _ = orc.er_graph(n, m, 5)
    return n, rp, col


def test_sir_invariants(orc, small_graph):
    # S pin (i): S+I+R = N, S non-increasing, R non-decreasing
    n, rp, col = small_graph
    st = orc.sir_init(n, 40, 5)
    _, counts, _ = orc.sir_run(rp, col, st, 5, 0.05, 0.1, 0, 150)
    assert (counts.sum(axis=1) == n).all()
    assert (np.diff(counts[:, 0]) <= 0).all()
    assert (np.diff(counts[:, 2]) >= 0).all()


def test_beta_zero_keeps_susceptibles(orc, small_graph):
    # S pin (ii)
    n, rp, col = small_graph
    st = orc.sir_init(n, 40, 9)
    _, counts, _ = orc.sir_run(rp, col, st, 9, 0.0, 0.3, 0, 40)
    assert (counts[:, 0] == n - 40).all()


def test_gamma_one_recovers_everyone_next_step(orc, small_graph):
    # S pin (iii)
    n, rp, col = small_graph
    st = orc.sir_init(n, 40, 9)
    for t in range(10):
        nxt = orc.sir_step(rp, col, st, 9, t, 0.2, 1.0)
        assert (nxt[st == 1] == 2).all()
        st = nxt


def _bfs_dist(n, rp, col, sources):
    A = sp.csr_matrix((np.ones(col.size), col, rp), shape=(n, n))
    d = shortest_path(A, unweighted=True, indices=sources, directed=False)
    return d.min(axis=0)


def test_beta_one_gamma_zero_is_bfs_ball(orc, small_graph):
    # S pin (iv): I u R after t steps = vertices within graph distance <= t
    n, rp, col = small_graph
    st = orc.sir_init(n, 3, 21)
    dist = _bfs_dist(n, rp, col, np.nonzero(st == 1)[0])
    for t in range(8):
        st = orc.sir_step(rp, col, st, 21, t, 1.0, 0.0)
        assert np.array_equal(st != 0, dist <= t + 1)


def test_beta_one_gamma_one_is_bfs_front(orc, small_graph):
    # S pin (v): I at step t = vertices at distance exactly t
    n, rp, col = small_graph
    st = orc.sir_init(n, 3, 22)
    dist = _bfs_dist(n, rp, col, np.nonzero(st == 1)[0])
    for t in range(8):
        st = orc.sir_step(rp, col, st, 22, t, 1.0, 1.0)
        assert np.array_equal(st == 1, dist == t + 1)
        assert np.array_equal(st == 2, dist <= t)


def test_per_edge_infection_probability(orc):
    # S4: P(infect) = 1 - (1 - beta)^{k_I} for a susceptible with k_I infected
    # neighbours (per-edge draws), NOT beta (Listing 2's single draw).
    k, beta = 6, 0.1
    n = k + 1  # star: centre 0, leaves 1..k
    rp = np.array([0, k] + list(range(k + 1, 2 * k + 1)), np.int32)
    col = np.array(list(range(1, k + 1)) + [0] * k, np.int32)
    st = np.array([0] + [1] * k, np.uint8)
    trials, hits = 0, 0
    for seed in range(400):
        for t in range(25):
            hits += int(orc.sir_step(rp, col, st, seed, t, beta, 0.0)[0] == 1)
            trials += 1
    p = 1 - (1 - beta) ** k
    sd = np.sqrt(p * (1 - p) / trials)
    assert abs(hits / trials - p) < 5 * sd
    assert abs(hits / trials - beta) > 10 * sd


def test_recovery_probability(orc):
    n = 20_000
    rp = np.zeros(n + 1, np.int32)
    col = np.zeros(0, np.int32)
    st = np.ones(n, np.uint8)
    nxt = orc.sir_step(rp, col, st, 3, 0, 0.5, 0.1)
    frac = (nxt == 2).mean()
    assert abs(frac - 0.1) < 5 * np.sqrt(0.09 / n)


def test_tx_draw_is_symmetric_in_the_pair(orc, curand_host):
    # S3: keyed on the unordered pair -> push and pull see one draw
    for a, b, t in [(1, 2, 0), (99, 3, 7), (12345, 67890, 199)]:
        w = orc.sir_tx_word(7, a, b, t)
        assert w == orc.sir_tx_word(7, b, a, t)
        ref = curand_host.blocks([[min(a, b), max(a, b), t, TAG_TX]], [[7, 0]])[0, 0]
        assert w == int(ref)


def test_sweep_replicate_matches_run(orc):
    # consistency of the sweep entry point with graph + init + run
    n, kbar, beta, gamma, frac, seed, steps = 2000, 8.0, 0.08, 0.1, 0.01, 17, 60
    m, k = orc.round_count(n * kbar / 2), orc.round_count(frac * n)
    rp, col, _ = orc.er_graph(n, m, seed)
    st = orc.sir_init(n, k, seed)
    st2, counts, _ = orc.sir_run(rp, col, st, seed, beta, gamma, 0, steps)
    assert orc.sir_replicate(n, kbar, beta, gamma, frac, seed, steps) == counts[-1, 2]
    out = orc.sir_sweep(n, kbar, gamma, frac, [beta, beta], [seed, seed + 1], steps)
    assert out[0] == counts[-1, 2] / n


def test_sweep_layout(orc):
    # S6: beta-major layout, 64 betas equal numpy.linspace(0.01, 0.2, 64), seed_r = r
    betas, seeds = sweep_replicates(C5_SWEEP)
    assert betas.size == 4096 and seeds.size == 4096
    assert betas[0] == 0.01 and betas[-1] == 0.2
    grid = np.linspace(0.01, 0.2, 64)
    for b in (0, 1, 31, 63):
        assert betas[64 * b] == grid[b] == betas[64 * b + 63]
        assert orc.bernoulli_threshold(betas[64 * b]) == orc.bernoulli_threshold(
            0.01 + b * ((0.2 - 0.01) / 63))
    assert seeds[4095] == 4095


def test_final_size_sanity(orc):
    # S pin (vii), sanity only: bond-percolation estimate of the final size
    n = 10_000
    lo = orc.sir_replicate(n, 8.0, 0.01, 0.1, 0.01, 1, 300) / n
    hi = orc.sir_replicate(n, 8.0, 0.2, 0.1, 0.01, 1, 300) / n
    assert lo < 0.2 and hi > 0.95


# ---------------------------------------------------------------------------
# Bit-level pin of the step's draw keying (S2/S3, R3-R5, R7): an independent
# columnar re-formulation over the arc list whose every draw comes from
# cuRAND's Philox routine (tests/pins) with explicitly composed counters, and
# whose thresholds are exact rationals.  An off-by-one step index, a swapped
# tag, a lane64/lane32 mix-up, a (max, min) pair order or a dropped key word
# changes some state within a few steps and fails here.
# ---------------------------------------------------------------------------
def t_exact(p):
    """R7 by exact rational arithmetic: ceil(p * 2^32); p >= 1 -> 2^32."""
    import math
    from fractions import Fraction
    if p >= 1:
        return 1 << 32
    return math.ceil(Fraction(p) * (1 << 32))


def numpy_sir_step(rp, col, x, seed, t, beta, gamma, curand_host):
    """S2 over the arc list: s in S becomes I iff some arc (s, i) with x[i] = I has
    word0(Philox(key = seed, ctr = (min, max, t, 0x10))) < T(beta); i in I
    becomes R iff lane32(0x11, i, t) < T(gamma); R stays R."""
    n = x.size
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    dst = col.astype(np.int64)
    si = (x[src] == 0) & (x[dst] == 1)
    s, i = src[si], dst[si]
    lo, hi = np.minimum(s, i), np.maximum(s, i)
    infected = np.zeros(n, bool)
    if lo.size:
        ctr = np.stack([lo.astype(np.uint32), hi.astype(np.uint32),
                        np.full(lo.size, t, np.uint32), np.full(lo.size, TAG_TX, np.uint32)], 1)
        w0 = curand_host.blocks(ctr, [[seed & 0xFFFFFFFF, seed >> 32]])[:, 0].astype(np.uint64)
        infected[s[w0 < np.uint64(t_exact(beta))]] = True
    rec = curand_host.lane32(seed, TAG_REC, np.arange(n, dtype=np.uint64), t).astype(np.uint64)
    y = x.copy()
    y[(x == 0) & infected] = 1
    y[(x == 1) & (rec < np.uint64(t_exact(gamma)))] = 2
    return y


def test_t_exact_matches_survey_values(orc):
    # R7 printed values, exact
    for p, want in [(0.05, 214_748_365), (0.1, 429_496_730), (0.01, 42_949_673), (0.2, 858_993_460)]:
        assert t_exact(p) == want == orc.bernoulli_threshold(p)


@pytest.mark.parametrize("seed,beta,gamma,t0", [(7, 0.05, 0.1, 0), ((5 << 32) | 7, 0.05, 0.1, 3),
                                                (11, 0.3, 0.25, 17)])
def test_sir_step_equals_curand_reformulation(orc, curand_host, seed, beta, gamma, t0):
    # >= 20 steps at the BJ rates (and a fast epidemic), from step index t0,
    # on a cuRAND/scipy-built graph and argsort-chosen initial infected
    n, m, k = 3000, 15_000, 30
    rp, col, _ = indep_graph(n, m, seed, curand_host)
    keys = curand_host.lane64(seed, TAG_INIT, np.arange(n, dtype=np.uint64), 0)
    x = np.zeros(n, np.uint8)
    x[np.argsort(keys, kind="stable")[:k]] = 1
    assert np.array_equal(orc.sir_init(n, k, seed), x)
    ref = x.copy()
    run_state, counts, _ = orc.sir_run(rp, col, x, seed, beta, gamma, t0, 24)
    changed = 0
    for j in range(24):
        nxt = numpy_sir_step(rp, col, ref, seed, t0 + j, beta, gamma, curand_host)
        got = orc.sir_step(rp, col, ref, seed, t0 + j, beta, gamma)
        assert np.array_equal(got, nxt), f"step {t0 + j}"
        assert counts[j].tolist() == [int((nxt == s).sum()) for s in range(3)]
        changed += int((nxt != ref).sum())
        ref = nxt
    assert np.array_equal(run_state, ref)
    assert changed > 200  # the epidemic actually moves (both transitions exercised)
