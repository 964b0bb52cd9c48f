"""GPU parity: wealth transfer (C-ABI path) vs the CPU oracle, bit-exact (W1-W3).

All calls go through libamber.so (include/amber.h) via the thin binding.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2601_16292_b200 import Model, wealth_params
from paper_2601_16292_b200.workloads import C1_WEALTH_SMALL, C4_WEALTH_SCALE


def make(n, seed, **kw):
    p = wealth_params(w0=kw.pop("w0", 1), amount=kw.pop("amount", 1),
                      exclude_self=kw.pop("exclude_self", 0), counter_bits=kw.pop("bits", 0))
    return Model("wealth", n, p, seed, **kw)


def test_c1_every_step_bit_exact(orc):
    cfg = C1_WEALTH_SMALL
    m = make(cfg["n"], cfg["seed"])
    m.set_option("digest", 1)
    w = np.full(cfg["n"], cfg["w0"], np.int32)
    for t in range(cfg["steps"]):
        m.step(1)
        w = orc.wealth_step(w, cfg["seed"], t)
        assert np.array_equal(m.read_column("wealth"), w), f"step {t}"
    _, tot, act, dig = orc.wealth_run(np.full(cfg["n"], 1, np.int32), cfg["seed"], 0, cfg["steps"],
                                      digests=True)
    assert np.array_equal(m.metrics("total_wealth"), tot)
    assert np.array_equal(m.metrics("active"), act)
    assert np.array_equal(m.metrics("digest"), dig.astype(np.uint64))
    assert m.digest("wealth") == orc.digest(w)
    assert m.step_count == cfg["steps"]


@pytest.mark.parametrize("bits", [2, 4, 8, 16, 32])
@pytest.mark.parametrize("n", [1, 7, 513, 5003])
def test_counter_widths_and_ragged_sizes(orc, bits, n):
    # 2-bit counters overflow often: exercises the exact detection + replay path
    m = make(n, 1234, bits=bits)
    m.set_option("persistent", 0)  # the multi-CTA counter path (small N would use one CTA)
    m.step(60)
    w, tot, act, _ = orc.wealth_run(np.full(n, 1, np.int32), 1234, 0, 60)
    assert np.array_equal(m.read_column("wealth"), w)
    assert np.array_equal(m.metrics("total_wealth"), tot)
    assert np.array_equal(m.metrics("active"), act)
    if bits == 2 and n >= 513:
        assert m.get_option("replays") > 0


@pytest.mark.parametrize("n", [1, 2, 1000, 16384])
def test_small_single_cta_path_equals_counter_path(orc, n):
    a = make(n, 42)  # n <= 16384: one CTA runs all steps in shared memory
    b = make(n, 42)
    b.set_option("persistent", 0)
    a.step(37)
    a.step(63)
    b.step(100)
    w = orc.wealth_run(np.full(n, 1, np.int32), 42, 0, 100)[0]
    assert np.array_equal(a.read_column("wealth"), w)
    assert np.array_equal(b.read_column("wealth"), w)
    assert np.array_equal(a.metrics("active"), b.metrics("active"))


def test_chunked_stepping_and_geometry_invariance(orc):
    n, seed = 40_000, 77
    ref = orc.wealth_run(np.full(n, 1, np.int32), seed, 0, 30)[0]
    a = make(n, seed)
    for _ in range(30):
        a.step(1)
    b = make(n, seed)
    b.set_option("block", 64)
    b.set_option("grid", 3)
    b.step(13)
    b.step(17)
    c = make(n, seed)
    c.set_option("block", 128)
    c.step(30)
    for m in (a, b, c):
        assert np.array_equal(m.read_column("wealth"), ref)


@pytest.mark.parametrize("amount,exclude_self,w0", [(1, 1, 1), (3, 0, 5), (2, 1, 7), (1, 0, 0)])
def test_variants(orc, amount, exclude_self, w0):
    n, seed = 3001, 9
    m = make(n, seed, amount=amount, exclude_self=exclude_self, w0=w0)
    m.step(25)
    w = orc.wealth_run(np.full(n, w0, np.int32), seed, 0, 25, amount=amount,
                       exclude_self=exclude_self)[0]
    assert np.array_equal(m.read_column("wealth"), w)


def test_two_agents_exclude_self_fixed_point():
    m = make(2, 5, exclude_self=1)
    m.step(100)
    assert m.read_column("wealth").tolist() == [1, 1]


def test_checkpoint_resume(orc):
    n, seed = 10_000, 3
    full = make(n, seed)
    full.step(100)
    a = make(n, seed)
    a.step(50)
    saved, s = a.read_column("wealth"), a.step_count
    b = make(n, seed)
    b.write_column("wealth", saved)
    b.set_step(s)
    b.step(50)
    assert np.array_equal(b.read_column("wealth"), full.read_column("wealth"))
    assert b.digest("wealth") == full.digest("wealth")


def test_user_written_state_and_device_io(orc):
    import torch
    n, seed = 4096, 21
    rng = np.random.default_rng(0)
    w0 = rng.integers(0, 4, n).astype(np.int32)
    m = make(n, seed)
    m.write_column("wealth", torch.from_numpy(w0).cuda())
    m.step(10)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    m.read_column("wealth", out)
    w = orc.wealth_run(w0, seed, 0, 10)[0]
    assert np.array_equal(out.cpu().numpy(), w)


def test_c4_full_size_prefix(orc):
    # BASELINE config 4 at full N = 1e8, bench launch configuration; first 2 steps
    # compared element by element with the oracle, then conservation to step 50.
    cfg = C4_WEALTH_SCALE
    n = cfg["n"]
    m = make(n, cfg["seed"])
    w = np.full(n, 1, np.int32)
    for t in range(2):
        m.step(1)
        w = orc.wealth_step(w, cfg["seed"], t)
        got = m.read_column("wealth")
        assert np.array_equal(got, w), f"step {t}"
    m.step(48)
    tot = m.metrics("total_wealth")
    assert (tot == n).all() and len(tot) == 50
    assert m.get_option("replays") == 0


def test_errors_are_reported():
    from paper_2601_16292_b200 import AmberError
    with pytest.raises(AmberError):
        make(10, 1, bits=3)
    m = make(10, 1)
    with pytest.raises(AmberError):
        m.read_column("nope")
    with pytest.raises(AmberError):
        m.read_column("wealth", np.zeros(3, np.int32))


def test_small_metrics_ring_and_per_step_reads(orc):
    # metrics_capacity 16: overflow-check windows close every few steps; per-step
    # reads (as bench.py's end-to-end loop does) see exactly that step's record
    n, seed = 300_000, 27
    m = make(n, seed, bits=2)  # 2-bit counters: replays happen inside the windows
    m.set_option("metrics_capacity", 16)
    w = np.ones(n, np.int32)
    for t in range(40):
        m.step(1)
        act = m.metrics("active")
        w_next, tot, a, _ = orc.wealth_run(w, seed, t, 1)
        assert act[-1] == a[0], t
        m.reset_metrics()
        w = w_next
    assert np.array_equal(m.read_column("wealth"), w)
    assert m.get_option("replays") > 0


def test_c4_all_1000_steps_vs_oracle_golden():
    # BASELINE config 4 at full size, all 1,000 steps, in the bench configuration
    # (default scatter, one fused launch per step): the per-step D1 digest of the
    # whole column, total wealth and active count against the oracle's values
    # (tests/golden/c4_wealth_oracle.txt, tools/make_oracle_goldens.py, oracle/ only)
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "c4_wealth_oracle.txt")
    if not os.path.exists(path):
        pytest.skip("golden file not generated (tools/make_oracle_goldens.py c4, ~1 h of CPU)")
    rows = np.array([[int(x) for x in ln.split()] for ln in open(path) if not ln.startswith("#")], dtype=object)
    cfg = C4_WEALTH_SCALE
    m = make(cfg["n"], cfg["seed"])
    m.set_option("digest", 1)
    m.step(cfg["steps"])
    dig = m.metrics("digest")
    assert len(dig) == cfg["steps"]
    assert [int(x) for x in dig] == [int(x) for x in rows[:, 1]]
    assert [int(x) for x in m.metrics("total_wealth")] == [int(x) for x in rows[:, 2]]
    assert [int(x) for x in m.metrics("active")] == [int(x) for x in rows[:, 3]]


def test_injected_counter_fault_is_caught_and_replayed(orc):
    # fault injection: one extra count in a pending counter makes the
    # decoded counts exceed the increments issued (got != sent); the window is
    # replayed from its pinned state with exact counters -- result bit-exact,
    # total wealth conserved at every step
    n, seed = 300_000, 3
    m = make(n, seed)
    m.step(5)
    assert m.get_option("replays") == 0
    m.set_option("inject_counter_fault", 12_345)
    m.step(5)
    w, tot, act, _ = orc.wealth_run(np.ones(n, np.int32), seed, 0, 10)
    assert np.array_equal(m.read_column("wealth"), w)
    assert m.get_option("replays") >= 1
    # the replayed window (steps 5..9) keeps its records; the ring's earlier ones
    # are cleared with it
    assert np.array_equal(m.metrics("total_wealth"), tot[5:]) and np.array_equal(m.metrics("active"), act[5:])
