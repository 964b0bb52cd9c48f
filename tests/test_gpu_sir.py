"""GPU parity: SIR on G(n, M) (C2) and the replicate sweep (C5) vs the oracle, bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2601_16292_b200 import Model, sir_params, sweep
from paper_2601_16292_b200.workloads import C2_SIR, C5_SWEEP, sweep_replicates


def sir_counts(cfg):
    """G1/S1 sizes by the oracle's own rounding (orc_round_count)."""
    import oracle
    return (oracle.round_count(cfg["n"] * cfg["mean_degree"] / 2.0),
            oracle.round_count(cfg["init_frac"] * cfg["n"]))


def oracle_graph(orc, m, cfg):
    """The ORACLE's G(n, M) for cfg (orc_er_graph, never the device's CSR),
    after checking that the device built exactly that graph; the oracle is
    then stepped on its own graph."""
    rp, col, mu = orc.er_graph(cfg["n"], sir_counts(cfg)[0], cfg["seed"])
    assert np.array_equal(m.read_column("row_ptr"), rp)
    assert np.array_equal(m.read_column("col_idx"), col)
    return rp, col


def make(cfg, **kw):
    p = sir_params(cfg["mean_degree"], cfg["beta"], cfg["gamma"], cfg["init_frac"])
    return Model("sir", cfg["n"], p, cfg["seed"], **kw)


@pytest.mark.parametrize("n,kbar,seed", [(2, 1.0, 1), (50, 4.0, 3), (1000, 10.0, 7), (100_000, 10.0, 7)])
def test_graph_and_initial_state(orc, n, kbar, seed):
    cfg = dict(n=n, mean_degree=kbar, beta=0.05, gamma=0.1, init_frac=0.01, seed=seed)
    m = make(cfg)
    m_draws, k = sir_counts(cfg)
    rp, col, mu = orc.er_graph(n, m_draws, seed)
    assert np.array_equal(m.read_column("row_ptr"), rp)
    assert np.array_equal(m.read_column("col_idx"), col)
    assert m.get_option("edges") == mu
    assert np.array_equal(m.read_column("state"), orc.sir_init(n, k, seed))


@pytest.mark.parametrize("persistent,digest", [(0, 1), (1, 1), (1, 0)])
def test_c2_every_step_bit_exact(orc, persistent, digest):
    # persistent + digest off enables the push direction when I < S (S3: same result)
    cfg = C2_SIR
    m = make(cfg)
    m.set_option("persistent", persistent)
    m.set_option("digest", digest)
    rp, col = oracle_graph(orc, m, cfg)
    st = orc.sir_init(cfg["n"], sir_counts(cfg)[1], cfg["seed"])
    st_ref, counts, dig = orc.sir_run(rp, col, st, cfg["seed"], cfg["beta"], cfg["gamma"], 0,
                                      cfg["steps"], digests=True)
    if persistent:
        m.step(cfg["steps"])
    else:
        x = st.copy()
        for t in range(cfg["steps"]):
            m.step(1)
            x = orc.sir_step(rp, col, x, cfg["seed"], t, cfg["beta"], cfg["gamma"])
            if t % 20 == 0:
                assert np.array_equal(m.read_column("state"), x), f"step {t}"
    assert np.array_equal(m.read_column("state"), st_ref)
    for k, name in enumerate("SIR"):
        assert np.array_equal(m.metrics(name), counts[:, k]), name
    if digest:
        assert np.array_equal(m.metrics("digest"), dig.astype(np.uint64))
    assert m.digest("state") == orc.digest(st_ref)


@pytest.mark.parametrize("beta,gamma", [(0.0, 0.3), (1.0, 0.0), (1.0, 1.0), (0.3, 1.0)])
def test_special_cases(orc, beta, gamma):
    cfg = dict(n=3000, mean_degree=5.0, beta=beta, gamma=gamma, init_frac=0.003, seed=21)
    m = make(cfg)
    m.step(12)
    rp, col = oracle_graph(orc, m, cfg)
    st = orc.sir_init(3000, 9, 21)
    ref, _, _ = orc.sir_run(rp, col, st, 21, beta, gamma, 0, 12)
    assert np.array_equal(m.read_column("state"), ref)


def test_geometry_and_chunking_invariance(orc):
    cfg = dict(C2_SIR, n=20_000, steps=40)
    a = make(cfg)
    a.step(40)
    d = make(cfg)  # push/pull switching at different points of the run
    d.step(1)
    d.step(5)
    d.step(34)
    assert np.array_equal(d.read_column("state"), a.read_column("state"))
    b = make(cfg)
    b.set_option("persistent", 0)
    b.set_option("block", 64)
    b.step(17)
    b.step(23)
    c = make(cfg)
    c.set_option("grid", 5)
    c.step(40)
    ref = a.read_column("state")
    assert np.array_equal(b.read_column("state"), ref)
    assert np.array_equal(c.read_column("state"), ref)


def test_checkpoint_resume_state():
    cfg = dict(C2_SIR, n=20_000)
    full = make(cfg)
    full.step(60)
    a = make(cfg)
    a.step(30)
    saved = a.read_column("state")
    b = make(cfg)
    b.write_column("state", saved)
    b.set_step(30)
    b.step(30)
    assert np.array_equal(b.read_column("state"), full.read_column("state"))


def test_sweep_subset_bit_exact(orc):
    c = C5_SWEEP
    betas, seeds = sweep_replicates(c)
    pick = np.arange(0, 4096, 61)  # 68 replicates spanning all betas
    got = sweep(c["n"], sir_params(c["mean_degree"], 0.0, c["gamma"], c["init_frac"]), betas[pick],
                seeds[pick], c["steps"])
    want = orc.sir_sweep(c["n"], c["mean_degree"], c["gamma"], c["init_frac"], betas[pick],
                         seeds[pick], c["steps"])
    assert np.array_equal(got, want)


def test_sweep_full_c5_sampled(orc):
    # the full 4096-replicate batch in the bench configuration; 96 sampled replicates
    c = C5_SWEEP
    betas, seeds = sweep_replicates(c)
    got, st = sweep(c["n"], sir_params(c["mean_degree"], 0.0, c["gamma"], c["init_frac"]), betas,
                    seeds, c["steps"], with_stats=True)
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(4096, 96, replace=False))
    want = orc.sir_sweep(c["n"], c["mean_degree"], c["gamma"], c["init_frac"], betas[pick],
                         seeds[pick], c["steps"])
    assert np.array_equal(got[pick], want)
    assert st["agent_updates"] == 4096 * 10_000 * 300
    assert 0 < st["active_updates"] <= st["agent_updates"]
    # final size rises with beta (sanity)
    per_beta = got.reshape(64, 64).mean(axis=1)
    assert per_beta[-1] > 0.95 and per_beta[0] < 0.3


def test_sweep_global_graph_path(orc):
    # n large enough that the CSR cannot be staged in shared memory (global-memory path)
    n, kbar, g, f = 30_000, 8.0, 0.1, 0.001
    betas = np.array([0.02, 0.05, 0.1, 0.2])
    seeds = np.array([5, 6, 7, 8], dtype=np.uint64)
    got = sweep(n, sir_params(kbar, 0.0, g, f), betas, seeds, 120)
    want = orc.sir_sweep(n, kbar, g, f, betas, seeds, 120)
    assert np.array_equal(got, want)


def test_sweep_edge_cases(orc):
    n = 500
    got = sweep(n, sir_params(6.0, 0.0, 0.1, 0.0), [0.5, 1.0], [1, 2], 50)
    assert (got == 0).all()  # nobody infected initially
    got = sweep(n, sir_params(6.0, 0.0, 1.0, 0.02), [0.0], [3], 5)
    assert got[0] == 10 / n  # gamma = 1, beta = 0: exactly the initial infected recover
    assert sweep(n, sir_params(6.0, 0.0, 0.1, 0.02), [], [], 5).size == 0


@pytest.mark.parametrize("digest", [0, 1])
def test_large_population_dynamic_chunks(orc, digest):
    # n large enough that the persistent launch hands out warp chunks from the
    # per-region queues, with push (I < S) and pull steps and the I/S bitmaps
    cfg = dict(n=1_000_000, mean_degree=10.0, beta=0.05, gamma=0.1, init_frac=0.01, seed=17, steps=30)
    m = make(cfg)
    m.set_option("digest", digest)
    m.step(1)      # first call: push allowed from the seeded counts
    m.step(29)
    rp, col = oracle_graph(orc, m, cfg)
    st = orc.sir_init(cfg["n"], 10_000, cfg["seed"])
    ref, counts, dig = orc.sir_run(rp, col, st, cfg["seed"], cfg["beta"], cfg["gamma"], 0, 30, digests=True)
    assert np.array_equal(m.read_column("state"), ref)
    for k, name in enumerate("SIR"):
        assert np.array_equal(m.metrics(name), counts[:, k]), name
    if digest:
        assert np.array_equal(m.metrics("digest"), dig.astype(np.uint64))


def test_mixed_launch_modes_and_column_write(orc):
    cfg = dict(n=300_000, mean_degree=8.0, beta=0.08, gamma=0.15, init_frac=0.002, seed=23, steps=40)
    a = make(cfg)
    a.step(40)
    b = make(cfg)
    for k, pers in enumerate([1, 0, 1, 1, 0, 0, 1]):  # persistent / per-step pull calls interleaved
        b.set_option("persistent", pers)
        b.step([3, 2, 7, 1, 4, 3, 20][k])
    assert np.array_equal(b.read_column("state"), a.read_column("state"))
    # a column write mid-epidemic, then push steps from the written state
    c = make(cfg)
    c.step(10)
    crp, ccol = oracle_graph(orc, c, cfg)
    mid = orc.sir_run(crp, ccol, orc.sir_init(cfg["n"], sir_counts(cfg)[1], cfg["seed"]), cfg["seed"],
                      cfg["beta"], cfg["gamma"], 0, 10)[0]
    assert np.array_equal(c.read_column("state"), mid)
    d = make(dict(cfg, seed=99))  # another graph: only the state matters after the write
    rp, col = oracle_graph(orc, d, dict(cfg, seed=99))
    d.write_column("state", mid)
    d.set_step(10)
    d.step(15)
    ref = orc.sir_run(rp, col, mid, 99, cfg["beta"], cfg["gamma"], 10, 15)[0]
    assert np.array_equal(d.read_column("state"), ref)


def test_full_occupancy_path_bit_exact(orc):
    # n_pad > 2^22: full-occupancy persistent launch with dynamic chunk queues
    cfg = dict(n=5_000_000, mean_degree=10.0, beta=0.05, gamma=0.1, init_frac=0.002, seed=29, steps=14)
    m = make(cfg)
    m.step(cfg["steps"])
    rp, col = oracle_graph(orc, m, cfg)
    st = orc.sir_init(cfg["n"], 10_000, cfg["seed"])
    ref, counts, _ = orc.sir_run(rp, col, st, cfg["seed"], cfg["beta"], cfg["gamma"], 0, cfg["steps"])
    assert np.array_equal(m.read_column("state"), ref)
    assert np.array_equal(m.metrics("I"), counts[:, 1])


def test_small_metrics_ring_wraps(orc):
    # metrics_capacity 16 over 70 steps: the ring wraps several times; the counts slot
    # that steers push/pull (step t-1) must survive every chunk's slot zeroing
    cfg = dict(n=50_000, mean_degree=8.0, beta=0.07, gamma=0.1, init_frac=0.01, seed=41, steps=70)
    m = make(cfg)
    m.set_option("metrics_capacity", 16)
    m.step(33)
    m.step(37)
    rp, col = oracle_graph(orc, m, cfg)
    st = orc.sir_init(cfg["n"], 500, cfg["seed"])
    ref, counts, _ = orc.sir_run(rp, col, st, cfg["seed"], cfg["beta"], cfg["gamma"], 0, cfg["steps"])
    assert np.array_equal(m.read_column("state"), ref)
    got = m.metrics("I")
    assert len(got) == 16 and np.array_equal(got, counts[-16:, 1])


def test_sweep_full_c5_all_replicates_vs_oracle_golden():
    # all 4,096 final R fractions of BASELINE config 5 against the oracle's values
    # (tests/golden/c5_sweep_oracle.txt, written by tools/make_oracle_goldens.py,
    # which calls only oracle/); exact ratios, so compared bit for bit
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "c5_sweep_oracle.txt")
    rows = [ln.split() for ln in open(path) if not ln.startswith("#")]
    want = np.array([float(r[3]) for r in rows])
    c = C5_SWEEP
    betas, seeds = sweep_replicates(c)
    assert np.array_equal(np.array([float(r[1]) for r in rows]), betas)
    got = sweep(c["n"], sir_params(c["mean_degree"], 0.0, c["gamma"], c["init_frac"]), betas, seeds, c["steps"])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [37, 129, 4_097, 100_003])
@pytest.mark.parametrize("direction", [1, 2])
@pytest.mark.parametrize("apl", [1, 2, 4, 8])
def test_forced_direction_every_step_ragged(orc, n, direction, apl):
    # "direction" 1 = pull only, 2 = push whenever possible; both are the same
    # S3 draws, so each step must equal the oracle (128-agent chunks with a
    # ragged tail, one-step cooperative launches and multi-step launches)
    cfg = dict(n=n, mean_degree=6.0, beta=0.2, gamma=0.15, init_frac=0.05, seed=n % 97)
    m = make(cfg)
    m.set_option("direction", direction)
    m.set_option("apl", apl)  # agents per lane of the step kernels
    assert m.get_option("apl") == apl
    m.set_option("digest", 1)
    rp, col = oracle_graph(orc, m, cfg)
    x = orc.sir_init(n, sir_counts(cfg)[1], cfg["seed"])
    t = 0
    for chunk in (1, 1, 3, 1, 5, 2):
        m.step(chunk)
        for _ in range(chunk):
            x = orc.sir_step(rp, col, x, cfg["seed"], t, cfg["beta"], cfg["gamma"])
            t += 1
        assert np.array_equal(m.read_column("state"), x), f"step {t}"
    counts = np.array([(x == s).sum() for s in range(3)])
    assert [int(m.metrics(k)[-1]) for k in "SIR"] == counts.tolist()
    assert m.digest("state") == orc.digest(x)
    assert int(m.metrics("digest")[-1]) == orc.digest(x)


def test_column_write_recounts_and_keeps_history(orc):
    # after a state write the model counts the new state (so the next step may
    # push); the records of the steps before the write are unchanged
    cfg = dict(n=30_011, mean_degree=8.0, beta=0.15, gamma=0.1, init_frac=0.02, seed=5)
    m = make(cfg)
    m.set_option("digest", 1)
    rp, col = oracle_graph(orc, m, cfg)
    x = orc.sir_init(cfg["n"], sir_counts(cfg)[1], cfg["seed"])
    m.step(4)
    hist = [m.metrics(k).copy() for k in "SIR"]
    for t in range(4):
        x = orc.sir_step(rp, col, x, cfg["seed"], t, cfg["beta"], cfg["gamma"])
    # a mostly susceptible state with few infected agents: the next step should push
    w = np.where(x == 1, 0, x).astype(np.uint8)
    w[::997] = 1
    m.write_column("state", w)
    for k, h in zip("SIR", hist):
        assert np.array_equal(m.metrics(k)[:4], h)
    m.step(3)
    x = w
    for t in range(4, 7):
        x = orc.sir_step(rp, col, x, cfg["seed"], t, cfg["beta"], cfg["gamma"])
    assert np.array_equal(m.read_column("state"), x)
    counts = [int((x == s).sum()) for s in range(3)]
    assert [int(m.metrics(k)[-1]) for k in "SIR"] == counts
    assert int(m.metrics("digest")[-1]) == orc.digest(x)
    m.set_step(2)  # a step reset recounts as well
    m.step(1)
    y = orc.sir_step(rp, col, x, cfg["seed"], 2, cfg["beta"], cfg["gamma"])
    assert np.array_equal(m.read_column("state"), y)


def _v2_golden():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "v2_sir_oracle.txt")
    lines = [ln.split() for ln in open(path) if not ln.startswith("#")]
    g = dict(zip(lines[0][1::2], (int(v) for v in lines[0][2::2])))
    steps = np.array([[int(v) for v in ln] for ln in lines[1:]], dtype=np.uint64)
    return g, steps


def test_v2_full_size_vs_oracle_golden():
    # the SURVEY 8(d) roofline variant V2 at its full size (N = 1e8, 1e9 arcs), in
    # the configuration the bench times (persistent, direction-optimizing, digest
    # off): the device CSR against the oracle's row_ptr / col digests, the
    # per-step S, I, R against the oracle's, and the final state's D1 digest --
    # all from tests/golden/v2_sir_oracle.txt (written by tools/make_oracle_goldens.py
    # v2, which calls only oracle/)
    from paper_2601_16292_b200.workloads import V2_SIR_SCALE as cfg
    g, want = _v2_golden()
    m = make(cfg)
    assert m.get_option("edges") == g["edges"]
    assert m.digest("row_ptr") == g["row_ptr_digest"]
    assert m.digest("col_idx") == g["col_digest"]
    m.step(1)
    m.step(cfg["steps"] - 1)
    for k, name in enumerate("SIR"):
        assert np.array_equal(m.metrics(name).astype(np.uint64), want[:, 1 + k]), name
    assert m.digest("state") == int(want[-1, 4])


@pytest.mark.parametrize("direction", [0, 2])
def test_apl8_push_counts_deferred(orc, direction):
    # 8 agents per lane, digest off: pushers set the next bits with no-return
    # REDs and the new infections are counted after the step (sir_count_new);
    # the per-step S/I/R must still equal the oracle's, including the last step
    # of every call and across calls
    cfg = dict(n=100_003, mean_degree=8.0, beta=0.2, gamma=0.15, init_frac=0.01, seed=13)
    m = make(cfg)
    m.set_option("apl", 8)
    m.set_option("direction", direction)
    rp, col = oracle_graph(orc, m, cfg)
    x = orc.sir_init(cfg["n"], sir_counts(cfg)[1], cfg["seed"])
    t = 0
    for chunk in (1, 4, 2, 7):
        m.step(chunk)
        x, counts, _ = orc.sir_run(rp, col, x, cfg["seed"], cfg["beta"], cfg["gamma"], t, chunk)
        t += chunk
        assert np.array_equal(m.read_column("state"), x), f"step {t}"
        for k, name in enumerate("SIR"):
            assert np.array_equal(m.metrics(name)[-chunk:], counts[:, k]), (name, t)


@pytest.mark.parametrize("kbar", [1.5, 3.0, 24.0])
@pytest.mark.parametrize("direction", [1, 2])
@pytest.mark.parametrize("digest", [0, 1])
def test_apl8_walk_owner_lookup_sparse_and_dense(orc, kbar, direction, digest):
    # the 8-agents-per-lane walk looks owners up by row-end bits when the
    # non-empty rows form a lane prefix and falls back to the shuffle search
    # otherwise: sparse graphs (many empty rows, both lookups in one run) and
    # dense ones (rows spanning several 128-arc windows) must both equal the
    # oracle at every step.  digest 0 also runs the push chunk pass's
    # compacted recovery draws and byte-parallel state deltas.
    cfg = dict(n=70_001, mean_degree=kbar, beta=0.3, gamma=0.1, init_frac=0.02, seed=int(kbar * 10) + direction)
    m = make(cfg)
    m.set_option("apl", 8)
    m.set_option("direction", direction)
    m.set_option("digest", digest)
    rp, col = oracle_graph(orc, m, cfg)
    x = orc.sir_init(cfg["n"], sir_counts(cfg)[1], cfg["seed"])
    for t in range(8):
        m.step(1)
        x = orc.sir_step(rp, col, x, cfg["seed"], t, cfg["beta"], cfg["gamma"])
        assert np.array_equal(m.read_column("state"), x), f"step {t}"
        assert [int(m.metrics(k)[-1]) for k in "SIR"] == [int((x == v).sum()) for v in range(3)], f"step {t}"
    assert m.digest("state") == orc.digest(x)


@pytest.mark.parametrize("digest", [0, 1])
@pytest.mark.parametrize("apl", [1, 8])
def test_epidemic_end_identity_steps(orc, digest, apl):
    # once no agent is infected every further step is the identity; the
    # persistent launch records those steps' counts without a pass and leaves
    # early (copying the state to the other buffer set when an odd number of
    # steps remains).  Calls of odd and even lengths across the end of the
    # epidemic, then a write that re-seeds infections (the push runs on the
    # back buffers again): every step equals the oracle.
    cfg = dict(n=20_011, mean_degree=3.0, beta=0.08, gamma=0.45, init_frac=0.01, seed=3)
    m = make(cfg)
    m.set_option("apl", apl)
    m.set_option("digest", digest)
    rp, col = oracle_graph(orc, m, cfg)
    x = orc.sir_init(cfg["n"], sir_counts(cfg)[1], cfg["seed"])
    t = 0
    saw_zero = False
    for chunk in (5, 9, 1, 12, 3, 7, "write", 2, 11, 4, 1, 9):
        if chunk == "write":
            w = x.copy()
            w[::1013] = 1  # re-seed: ~20 infected agents
            m.write_column("state", w)
            x = w
            continue
        m.step(chunk)
        x, counts, _ = orc.sir_run(rp, col, x, cfg["seed"], cfg["beta"], cfg["gamma"], t, chunk)
        t += chunk
        assert np.array_equal(m.read_column("state"), x), f"step {t}"
        for k, name in enumerate("SIR"):
            assert np.array_equal(m.metrics(name)[-chunk:], counts[:, k]), (name, t)
        saw_zero |= bool((counts[:, 1] == 0).any())
        if digest:
            assert m.digest("state") == orc.digest(x)
            assert int(m.metrics("digest")[-1]) == orc.digest(x)
    assert saw_zero


def test_identity_steps_with_small_ring(orc):
    # identity steps across several persistent launches of one call (metrics
    # capacity 16: 15 steps per launch), the records of the last 16 steps checked
    cfg = dict(n=20_011, mean_degree=3.0, beta=0.08, gamma=0.45, init_frac=0.01, seed=3)
    m = make(cfg)
    m.set_option("metrics_capacity", 16)
    m.set_option("digest", 1)
    rp, col = oracle_graph(orc, m, cfg)
    x = orc.sir_init(cfg["n"], sir_counts(cfg)[1], cfg["seed"])
    m.step(47)
    x, counts, _ = orc.sir_run(rp, col, x, cfg["seed"], cfg["beta"], cfg["gamma"], 0, 47)
    assert counts[-1, 1] == 0
    assert np.array_equal(m.read_column("state"), x)
    for k, name in enumerate("SIR"):
        assert np.array_equal(m.metrics(name), counts[-16:, k]), name
    assert m.digest("state") == orc.digest(x)
    assert int(m.metrics("digest")[-1]) == orc.digest(x)
