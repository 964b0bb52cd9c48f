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

from paper_2601_16292_b200 import Model, loopback_id, shard_range, sir_params, sweep, wealth_params
from paper_2601_16292_b200.workloads import C5_SWEEP, sweep_replicates


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


def test_sharded_overflow_replay_is_collective(orc):
    # 2-bit counters overflow on some shard nearly every window: all shards replay
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
    ref, tot, _, _ = orc.wealth_run(np.ones(n, np.int32), seed, 0, 15)
    assert np.array_equal(m.read_column("wealth"), ref)
    assert np.array_equal(m.metrics("total_wealth"), tot)
    assert m.digest("wealth") == orc.digest(ref)
    assert m.get_option("replays") > 0
