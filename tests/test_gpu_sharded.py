"""GPU parity of the SHARDED paths on one B200 via the in-process loopback
transport (amber_loopback_id): `world` virtual shards of one wealth model,
each driven from its own host thread, exchange cross-shard receivers through
host barriers + device-to-device copies.  Everything except the transport
(remote bucketing kernel, exchange bookkeeping, receive-apply kernel,
all-reduced overflow check and exact replay, global metrics) is the code the
NCCL path runs.  Results must equal the unsharded oracle bit for bit."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2601_16292_b200 import Model, boids_params, loopback_id, shard_range, sir_params, sweep, wealth_params
from paper_2601_16292_b200.workloads import C5_SWEEP, sweep_replicates


@pytest.fixture(autouse=True)
def _release_device_memory():
    # the models allocate through torch's caching allocator: return the cached
    # blocks after each test, so the full-size tests (8 ranks x N = 1e8 wealth,
    # 8 graph builds of 1e9 arcs) do not meet a fragmented cache
    yield
    import gc

    import torch
    gc.collect()
    torch.cuda.empty_cache()


def oracle_graph(orc, cfg, m=None):
    """The ORACLE's G(n, M) (orc_er_graph); when a one-GPU model is given, its
    CSR must equal it.  The oracle is never stepped on a device-built graph."""
    rp, col, _ = orc.er_graph(cfg["n"], orc.round_count(cfg["n"] * cfg["mean_degree"] / 2.0), cfg["seed"])
    if m is not None:
        assert np.array_equal(m.read_column("row_ptr"), rp) and np.array_equal(m.read_column("col_idx"), col)
    return rp, col


def par(items, fn):
    out = [None] * len(items)
    err = []

    def run(k):
        try:
            out[k] = fn(items[k])
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)

    th = [threading.Thread(target=run, args=(k,)) for k in range(len(items))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


def sharded(world, n, seed, bits=0, exclude_self=0):
    uid = loopback_id()
    p = wealth_params(counter_bits=bits, exclude_self=exclude_self)
    return [Model("wealth", n, p, seed, rank=r, world=world, unique_id=uid) for r in range(world)]


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("n", [1001, 65_543])
def test_sharded_wealth_equals_oracle(orc, world, n):
    seed, steps = 31, 25
    ms = sharded(world, n, seed)
    for r, m in enumerate(ms):
        _, g, off, ln = m.column_info("wealth")
        assert g == n and (off, off + ln) == shard_range(n, world, r)
    par(ms, lambda m: m.step(steps))
    w = np.concatenate(par(ms, lambda m: m.read_column("wealth")))
    ref, tot, act, _ = orc.wealth_run(np.ones(n, np.int32), seed, 0, steps)
    assert np.array_equal(w, ref)
    for tt in par(ms, lambda m: m.metrics("total_wealth")):
        assert np.array_equal(tt, tot)  # global (all-shard) observables
    for aa in par(ms, lambda m: m.metrics("active")):
        assert np.array_equal(aa, act)
    dg = par(ms, lambda m: m.digest("wealth"))
    assert all(d == orc.digest(ref) for d in dg)


@pytest.mark.parametrize("world,n,mode", [(2, 3_000_017, "sparse"), (3, 2_000_003, "nccl"), (33, 50_021, "sparse")])
def test_sharded_wealth_bucket_slices(orc, monkeypatch, world, n, mode):
    # many warp chunks per bucket slice (> 64 chunks per rank: slices shared by
    # several chunks, cursors accumulating), both transports; world > 32 takes the
    # direct (unstaged) warp-aggregated append
    monkeypatch.setenv("AMBER_WEALTH_EXCHANGE", mode)
    seed, steps = 19, 6
    ms = sharded(world, n, seed)
    par(ms, lambda m: (m.step(2), m.step(4)))
    w = np.concatenate(par(ms, lambda m: m.read_column("wealth")))
    ref, tot, _, _ = orc.wealth_run(np.ones(n, np.int32), seed, 0, steps)
    assert np.array_equal(w, ref)
    for tt in par(ms, lambda m: m.metrics("total_wealth")):
        assert np.array_equal(tt, tot)


@pytest.mark.parametrize("world,mode", [(8, "sparse"), (2, "nccl"), (8, "dense"), (3, "dense")])
def test_sharded_c4_full_size_vs_oracle_golden(monkeypatch, world, mode):
    # BASELINE config 4 at full size (N = 1e8) sharded over `world` virtual ranks:
    # the first 40 steps' global digest / total / active against the oracle-written
    # golden (tests/golden/c4_wealth_oracle.txt) -- real bucket sizes, slices shared
    # by ~380 warp chunks each, staged flushes, both transports
    import os
    from paper_2601_16292_b200.workloads import C4_WEALTH_SCALE as cfg
    path = os.path.join(os.path.dirname(__file__), "golden", "c4_wealth_oracle.txt")
    if not os.path.exists(path):
        pytest.skip("golden file not generated (tools/make_oracle_goldens.py c4)")
    rows = [[int(x) for x in ln.split()] for ln in open(path) if not ln.startswith("#")]
    monkeypatch.setenv("AMBER_WEALTH_EXCHANGE", mode)
    steps = 40
    ms = sharded(world, cfg["n"], cfg["seed"])
    for m in ms:
        m.set_option("digest", 1)
    par(ms, lambda m: (m.step(7), m.step(steps - 7)))
    for dg in par(ms, lambda m: m.metrics("digest")):
        assert [int(x) for x in dg] == [r[1] for r in rows[:steps]]
    for tt in par(ms, lambda m: m.metrics("total_wealth")):
        assert [int(x) for x in tt] == [r[2] for r in rows[:steps]]
    for aa in par(ms, lambda m: m.metrics("active")):
        assert [int(x) for x in aa] == [r[3] for r in rows[:steps]]
    par(ms, lambda m: m.close())


@pytest.mark.parametrize("mode", ["default", "sparse", "nccl", "dense"])
def test_sharded_wealth_exchange_modes(orc, monkeypatch, mode):
    # dense (the default up to 8 ranks): every rank counts all its transfers in
    # global packed counters, owners sum the peers' words of their shard in place;
    # sparse: owners read the peers' id buckets in place after a stream-ordered
    # barrier; nccl: counts + payload send/recv through the transport
    if mode != "default":
        monkeypatch.setenv("AMBER_WEALTH_EXCHANGE", mode)
    world, n, seed, steps = 4, 30_011, 21, 20
    ms = sharded(world, n, seed)
    par(ms, lambda m: (m.step(7), m.step(13)))
    assert all(m.get_option("exchange") == {"default": 3, "sparse": 2, "nccl": 1, "dense": 3}[mode]
               for m in ms)  # mapped at the first step
    w = np.concatenate(par(ms, lambda m: m.read_column("wealth")))
    ref, tot, _, _ = orc.wealth_run(np.ones(n, np.int32), seed, 0, steps)
    assert np.array_equal(w, ref)
    for tt in par(ms, lambda m: m.metrics("total_wealth")):
        assert np.array_equal(tt, tot)


def test_sharded_dense_falls_back_when_blocks_straddle_words(orc, monkeypatch):
    # 2-bit counters with shards of 8 x odd agents: a shard's block of the global
    # packed counters would not start on a word, so the sparse buckets run instead
    monkeypatch.setenv("AMBER_WEALTH_EXCHANGE", "dense")
    world, n, seed, steps = 3, 70, 4, 9  # shard = 24 agents: 48 bits
    ms = sharded(world, n, seed, bits=2)
    par(ms, lambda m: m.step(steps))
    assert all(m.get_option("exchange") == 2 for m in ms)
    w = np.concatenate(par(ms, lambda m: m.read_column("wealth")))
    assert np.array_equal(w, orc.wealth_run(np.ones(n, np.int32), seed, 0, steps)[0])


@pytest.mark.parametrize("mode", ["sparse", "dense"])
def test_sharded_overflow_replay_is_collective(orc, monkeypatch, mode):
    # 2-bit counters overflow on some shard nearly every window: all shards replay
    monkeypatch.setenv("AMBER_WEALTH_EXCHANGE", mode)
    world, n, seed, steps = 4, 40_000, 5, 12
    ms = sharded(world, n, seed, bits=2)
    par(ms, lambda m: m.step(steps))
    w = np.concatenate(par(ms, lambda m: m.read_column("wealth")))
    assert np.array_equal(w, orc.wealth_run(np.ones(n, np.int32), seed, 0, steps)[0])
    reps = par(ms, lambda m: m.get_option("replays"))
    assert reps[0] > 0 and len(set(reps)) == 1


def test_sharded_exclude_self_and_chunked_steps(orc):
    world, n, seed = 3, 9_999, 8
    ms = sharded(world, n, seed, exclude_self=1)
    par(ms, lambda m: (m.step(3), m.step(7)))
    w = np.concatenate(par(ms, lambda m: m.read_column("wealth")))
    assert np.array_equal(w, orc.wealth_run(np.ones(n, np.int32), seed, 0, 10, exclude_self=1)[0])


def test_split_sweep_equals_single(orc):
    c = C5_SWEEP
    betas, seeds = sweep_replicates(c)
    pick = np.arange(0, 4096, 97)
    sp = sir_params(c["mean_degree"], 0.0, c["gamma"], c["init_frac"])
    single = sweep(c["n"], sp, betas[pick], seeds[pick], 120)
    uid = loopback_id()
    outs = par(list(range(4)), lambda r: sweep(c["n"], sp, betas[pick], seeds[pick], 120, rank=r, world=4,
                                               unique_id=uid))
    for o in outs:
        assert np.array_equal(o, single)
    want = orc.sir_sweep(c["n"], c["mean_degree"], c["gamma"], c["init_frac"], betas[pick], seeds[pick], 120)
    assert np.array_equal(single, want)


def test_nccl_plumbing_single_rank(orc, monkeypatch):
    # one-rank NCCL communicator from amber_nccl_unique_id: dlopen of torch's NCCL,
    # ncclCommInitRank, grouped ncclSend/ncclRecv of the bucket counts, ncclAllReduce
    # of the overflow flag and of the metrics -- the NCCL calls the multi-GPU run makes
    from paper_2601_16292_b200 import nccl_unique_id
    monkeypatch.setenv("AMBER_TEST_FORCE_EXCHANGE", "1")
    n, seed = 70_001, 12
    m = Model("wealth", n, wealth_params(counter_bits=2), seed, unique_id=nccl_unique_id())
    m.step(15)
    assert m.get_option("exchange") == 2  # P2P: IPC export + ncclAllGather of the handles + barrier all-reduces
    ref, tot, _, _ = orc.wealth_run(np.ones(n, np.int32), seed, 0, 15)
    assert np.array_equal(m.read_column("wealth"), ref)
    assert np.array_equal(m.metrics("total_wealth"), tot)
    assert m.digest("wealth") == orc.digest(ref)
    assert m.get_option("replays") > 0


def sharded_sir(world, cfg):
    uid = loopback_id()
    p = sir_params(cfg["mean_degree"], cfg["beta"], cfg["gamma"], cfg["init_frac"])
    return [Model("sir", cfg["n"], p, cfg["seed"], rank=r, world=world, unique_id=uid) for r in range(world)]


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("apl", [0, 4, 8])
def test_sharded_sir_equals_oracle(orc, world, apl):
    # NEXT-3: id-range shards, pull against the all-gathered I bitmap every step;
    # apl 4: 128-agent chunks that reach past a shard's end (masked)
    cfg = dict(n=50_003, mean_degree=10.0, beta=0.05, gamma=0.1, init_frac=0.01, seed=7)
    steps = 40
    ref_m = Model("sir", cfg["n"], sir_params(cfg["mean_degree"], cfg["beta"], cfg["gamma"], cfg["init_frac"]),
                  cfg["seed"])
    rp, col = oracle_graph(orc, cfg, ref_m)
    ref_m.close()
    st = orc.sir_init(cfg["n"], 500, cfg["seed"])
    ref, counts, dig = orc.sir_run(rp, col, st, cfg["seed"], cfg["beta"], cfg["gamma"], 0, steps, digests=True)
    ms = sharded_sir(world, cfg)
    infos = [m.column_info("state") for m in ms]
    assert infos[0][2] == 0 and sum(i[3] for i in infos) == cfg["n"]
    for a, b in zip(infos, infos[1:]):
        assert a[2] + a[3] == b[2] and a[3] % 32 == 0  # contiguous, 32-aligned slices
    for m in ms:
        m.set_option("digest", 1)
        m.set_option("apl", apl)
    par(ms, lambda m: (m.step(1), m.step(steps - 1)))
    x = np.concatenate(par(ms, lambda m: m.read_column("state")))
    assert np.array_equal(x, ref)
    for name_k, name in enumerate("SIR"):
        for v in par(ms, lambda m: m.metrics(name)):
            assert np.array_equal(v, counts[:, name_k]), name  # global counts on every rank
    for v in par(ms, lambda m: m.metrics("digest")):
        assert np.array_equal(v, dig.astype(np.uint64))
    assert all(d == orc.digest(ref) for d in par(ms, lambda m: m.digest("state")))


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("direction", [0, 2])
def test_sharded_sir_push_equals_oracle(orc, world, direction):
    # sharded push steps (direction 2: every step; 0: the global-count rule):
    # pushers walk their rows against the all-gathered S bitmap, remote targets
    # are all-to-all'd to their owners, the step finalises from the hit bits
    cfg = dict(n=50_003, mean_degree=10.0, beta=0.05, gamma=0.1, init_frac=0.01, seed=7)
    steps = 40
    ref_m = Model("sir", cfg["n"], sir_params(cfg["mean_degree"], cfg["beta"], cfg["gamma"], cfg["init_frac"]),
                  cfg["seed"])
    rp, col = oracle_graph(orc, cfg, ref_m)
    ref_m.close()
    st = orc.sir_init(cfg["n"], 500, cfg["seed"])
    ref, counts, dig = orc.sir_run(rp, col, st, cfg["seed"], cfg["beta"], cfg["gamma"], 0, steps, digests=True)
    ms = sharded_sir(world, cfg)
    for m in ms:
        m.set_option("digest", 1)
        m.set_option("direction", direction)
    par(ms, lambda m: (m.step(3), m.step(steps - 3)))
    x = np.concatenate(par(ms, lambda m: m.read_column("state")))
    assert np.array_equal(x, ref)
    for name_k, name in enumerate("SIR"):
        for v in par(ms, lambda m: m.metrics(name)):
            assert np.array_equal(v, counts[:, name_k]), name
    for v in par(ms, lambda m: m.metrics("digest")):
        assert np.array_equal(v, dig.astype(np.uint64))


def test_sharded_v2_full_size_vs_oracle_golden():
    # the V2 variant (SIR on G(1e8, 5e8)) sharded over 8 virtual ranks with the
    # direction rule (push steps through the hit-bitmap exchange, then pull):
    # per-step global S, I, R and the final state digest against the
    # oracle-written golden (tests/golden/v2_sir_oracle.txt)
    import os
    from paper_2601_16292_b200.workloads import V2_SIR_SCALE as cfg
    path = os.path.join(os.path.dirname(__file__), "golden", "v2_sir_oracle.txt")
    if not os.path.exists(path):
        pytest.skip("golden file not generated (tools/make_oracle_goldens.py v2)")
    lines = [ln.split() for ln in open(path) if not ln.startswith("#")]
    want = np.array([[int(v) for v in ln] for ln in lines[1:]], dtype=np.uint64)
    ms = sharded_sir(8, cfg)
    par(ms, lambda m: (m.step(3), m.step(cfg["steps"] - 3)))
    for k, name in enumerate("SIR"):
        for v in par(ms, lambda m: m.metrics(name)):
            assert np.array_equal(v.astype(np.uint64), want[:, 1 + k]), name
    assert all(d == int(want[-1, 4]) for d in par(ms, lambda m: m.digest("state")))
    par(ms, lambda m: m.close())


def test_sharded_sir_local_rows_and_column_write(orc):
    cfg = dict(n=20_000, mean_degree=6.0, beta=0.1, gamma=0.2, init_frac=0.005, seed=11)
    full = Model("sir", cfg["n"], sir_params(cfg["mean_degree"], cfg["beta"], cfg["gamma"], cfg["init_frac"]),
                 cfg["seed"])
    rp, col = oracle_graph(orc, cfg, full)
    full.step(8)
    mid = orc.sir_run(rp, col, orc.sir_init(cfg["n"], orc.round_count(cfg["init_frac"] * cfg["n"]), cfg["seed"]),
                      cfg["seed"], cfg["beta"], cfg["gamma"], 0, 8)[0]
    assert np.array_equal(full.read_column("state"), mid)
    ms = sharded_sir(2, cfg)
    for m in ms:  # local rows: offsets from 0, global neighbour ids
        _, _, lo, ln = m.column_info("state")
        lrp, lcol = m.read_column("row_ptr"), m.read_column("col_idx")
        assert np.array_equal(lrp, rp[lo:lo + ln + 1] - rp[lo])
        assert np.array_equal(lcol, col[rp[lo]:rp[lo + ln]])
    # restore a mid-run state into the shards, continue sharded
    def restore(m):
        _, _, lo, ln = m.column_info("state")
        m.write_column("state", mid[lo:lo + ln])
        m.set_step(8)
        m.step(12)
    par(ms, restore)
    x = np.concatenate(par(ms, lambda m: m.read_column("state")))
    assert np.array_equal(x, orc.sir_run(rp, col, mid, cfg["seed"], cfg["beta"], cfg["gamma"], 8, 12)[0])


def test_sir_nccl_plumbing_single_rank(orc, monkeypatch):
    # the sharded SIR path over a one-rank NCCL communicator: ncclAllGather of the
    # I bitmap every step, ncclAllReduce of the metrics and the digest
    from paper_2601_16292_b200 import nccl_unique_id
    monkeypatch.setenv("AMBER_TEST_FORCE_EXCHANGE", "1")
    cfg = dict(n=30_001, mean_degree=8.0, beta=0.06, gamma=0.1, init_frac=0.01, seed=3)
    m = Model("sir", cfg["n"], sir_params(cfg["mean_degree"], cfg["beta"], cfg["gamma"], cfg["init_frac"]),
              cfg["seed"], unique_id=nccl_unique_id())
    rp, col = oracle_graph(orc, cfg, m)
    m.step(25)
    st = orc.sir_init(cfg["n"], 300, cfg["seed"])
    ref, counts, _ = orc.sir_run(rp, col, st, cfg["seed"], cfg["beta"], cfg["gamma"], 0, 25)
    assert np.array_equal(m.read_column("state"), ref)
    assert np.array_equal(m.metrics("I"), counts[:, 1])
    assert m.digest("state") == orc.digest(ref)


BKEYS = ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")


def sharded_boids(world, cfg):
    uid = loopback_id()
    p = boids_params(*[cfg[k] for k in BKEYS])
    return [Model("boids", cfg["n"], p, cfg["seed"], rank=r, world=world, unique_id=uid) for r in range(world)]


def boids_state(ms):
    # collective column reads: every rank returns the whole id-ordered column
    cols = []
    for c in ("pos_x", "pos_y", "vel_x", "vel_y"):
        got = par(ms, lambda m: m.read_column(c))
        assert all(np.array_equal(g.view(np.uint32), got[0].view(np.uint32)) for g in got)
        cols.append(got[0])
    return cols


@pytest.mark.parametrize("world", [2, 3, 5])
def test_sharded_boids_equals_oracle(orc, world):
    # NEXT-3: x-slabs of cell columns, migration + halo exchange every step;
    # exact fixed-point sums -> bit-identical to the unsharded oracle
    cfg = dict(n=6000, L=200.0, R=10.0, rs=2.0, wc=0.01, wa=0.125, ws=0.05, vmax=2.0, dt=1.0, seed=3)
    steps = 25
    P = orc.boids_params(**{k: cfg[k] for k in BKEYS})
    ref = orc.boids_run(orc.boids_init(cfg["n"], cfg["L"], cfg["seed"]), P, steps)
    ms = sharded_boids(world, cfg)
    own0 = par(ms, lambda m: m.get_option("own_agents"))
    assert sum(own0) == cfg["n"]
    for m in ms:
        m.set_option("digest", 1)
    par(ms, lambda m: (m.step(1), m.step(steps - 1)))
    got = boids_state(ms)
    want = ref[0]
    for a, b in zip(got, want):
        assert np.array_equal(a.view(np.uint32), np.asarray(b, np.float32).view(np.uint32))
    assert sum(par(ms, lambda m: m.get_option("own_agents"))) == cfg["n"]  # agents migrated, none lost
    # global observables agree on every rank and with one GPU
    one = Model("boids", cfg["n"], boids_params(*[cfg[k] for k in BKEYS]), cfg["seed"])
    one.set_option("digest", 1)
    one.step(steps)
    for v in par(ms, lambda m: m.metrics("digest")):
        assert np.array_equal(v, one.metrics("digest"))
    for v in par(ms, lambda m: m.metrics("mean_speed")):
        assert np.allclose(v, one.metrics("mean_speed"), rtol=1e-12, atol=0)
    dg = par(ms, lambda m: m.digest("pos_x"))
    assert all(d == one.digest("pos_x") for d in dg)


@pytest.mark.parametrize("world,sy", [(2, 4), (3, 3), (5, 2)])
def test_sharded_boids_y_subrows_equal_oracle(orc, monkeypatch, world, sy):
    # y sub-rows of the slab grid (AMBER_BOIDS_SX; default 4 above 2^22 agents):
    # shorter stencil runs, same neighbours -> bit-identical, incl. wrapped rows
    monkeypatch.setenv("AMBER_BOIDS_SX", str(sy))
    cfg = dict(n=6000, L=200.0, R=10.0, rs=2.0, wc=0.01, wa=0.125, ws=0.05, vmax=2.0, dt=1.0, seed=3)
    steps = 20
    P = orc.boids_params(**{k: cfg[k] for k in BKEYS})
    ref = orc.boids_run(orc.boids_init(cfg["n"], cfg["L"], cfg["seed"]), P, steps)
    ms = sharded_boids(world, cfg)
    par(ms, lambda m: (m.step(3), m.step(steps - 3)))
    for a, b in zip(boids_state(ms), ref[0]):
        assert np.array_equal(a.view(np.uint32), np.asarray(b, np.float32).view(np.uint32))
    assert sum(par(ms, lambda m: m.get_option("own_agents"))) == cfg["n"]


def test_sharded_boids_large_equals_one_gpu(monkeypatch):
    # 2e6 agents at the V3 density over 4 slabs with y sub-rows against the
    # one-GPU model with x-subdivided rows (itself bit-exact vs the oracle in
    # test_gpu_boids.py): every position/velocity bit-identical after 6 steps
    monkeypatch.setenv("AMBER_BOIDS_SX", "4")
    n = 2_000_000
    cfg = dict(n=n, L=float(np.sqrt(n / 0.1)), R=10.0, rs=2.0, wc=0.01, wa=0.125, ws=0.05, vmax=2.0, dt=1.0, seed=9)
    one = Model("boids", n, boids_params(*[cfg[k] for k in BKEYS]), cfg["seed"])
    one.step(6)
    want = [one.read_column(c) for c in ("pos_x", "pos_y", "vel_x", "vel_y")]
    ms = sharded_boids(4, cfg)
    par(ms, lambda m: (m.step(2), m.step(4)))
    for a, b in zip(boids_state(ms), want):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    par(ms, lambda m: m.close())
    one.close()


def test_sharded_boids_column_write_and_single_rank_nccl(orc, monkeypatch):
    cfg = dict(n=3000, L=150.0, R=10.0, rs=2.0, wc=0.01, wa=0.125, ws=0.05, vmax=2.0, dt=1.0, seed=9)
    one = Model("boids", cfg["n"], boids_params(*[cfg[k] for k in BKEYS]), cfg["seed"])
    one.step(5)
    mid = [one.read_column(c) for c in ("pos_x", "pos_y", "vel_x", "vel_y")]
    one.step(10)
    want = [one.read_column(c) for c in ("pos_x", "pos_y", "vel_x", "vel_y")]
    ms = sharded_boids(3, cfg)  # fresh shards, state restored from the id-ordered columns

    def restore(m):
        for c, v in zip(("pos_x", "pos_y", "vel_x", "vel_y"), mid):
            m.write_column(c, v)
        m.set_step(5)
        m.step(10)
    par(ms, restore)
    for a, b in zip(boids_state(ms), want):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    # one-rank NCCL communicator: ncclSend/ncclRecv of the migration and halo
    # buffers (self exchange), ncclAllGather of the metrics, ncclAllReduce of columns
    from paper_2601_16292_b200 import nccl_unique_id
    monkeypatch.setenv("AMBER_TEST_FORCE_EXCHANGE", "1")
    m = Model("boids", cfg["n"], boids_params(*[cfg[k] for k in BKEYS]), cfg["seed"], unique_id=nccl_unique_id())
    assert m.get_option("slab_columns") == m.get_option("cells_per_side")
    m.step(15)
    for c, b in zip(("pos_x", "pos_y", "vel_x", "vel_y"), want):
        assert np.array_equal(m.read_column(c).view(np.uint32), b.view(np.uint32))
