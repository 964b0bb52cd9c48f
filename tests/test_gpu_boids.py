"""GPU parity: Boids (C3) vs the oracle.  Under the float contract (B3-B7) the
GPU step is expected to equal the oracle bit for bit; the tests assert BJ's
tolerances (1e-4 relative per agent after 1 step, 1e-3 on the ensemble
statistics after 100 steps) and report the exact-match fraction."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2601_16292_b200 import Model, boids_params
from paper_2601_16292_b200.workloads import C3_BOIDS

KEYS = ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")


def make(cfg, **kw):
    return Model("boids", cfg["n"], boids_params(*[cfg[k] for k in KEYS]), cfg["seed"], **kw)


def state(m):
    return tuple(m.read_column(c) for c in ("pos_x", "pos_y", "vel_x", "vel_y"))


def oinit(orc, cfg, m):
    """The ORACLE's initial state (B1) for cfg, after checking the device's is
    bit-identical; the oracle is never stepped from device-produced state."""
    ref = orc.boids_init(cfg["n"], cfg["L"], cfg["seed"])
    for a, b in zip(state(m), ref):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    return ref


def oparams(orc, cfg):
    return orc.boids_params(**{k: cfg[k] for k in KEYS})


def test_init_bit_exact(orc):
    cfg = C3_BOIDS
    m = make(cfg)
    ref = orc.boids_init(cfg["n"], cfg["L"], cfg["seed"])
    for a, b in zip(state(m), ref):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_c3_one_step_tolerance_and_exact(orc):
    cfg = C3_BOIDS
    m = make(cfg)
    st0 = oinit(orc, cfg, m)
    m.step(1)
    got = state(m)
    ref = orc.boids_step(st0, oparams(orc, cfg))
    L = cfg["L"]
    dpx = (got[0] - ref[0] + L / 2) % L - L / 2
    dpy = (got[1] - ref[1] + L / 2) % L - L / 2
    assert (np.abs(dpx) <= 1e-4 * np.maximum(np.abs(ref[0]), 1)).all()
    assert (np.abs(dpy) <= 1e-4 * np.maximum(np.abs(ref[1]), 1)).all()
    for k in (2, 3):
        assert (np.abs(got[k] - ref[k]) <= 1e-4 * np.maximum(np.abs(ref[k]), 1e-3)).all()
    exact = np.mean([np.array_equal(a.view(np.uint32), b.view(np.uint32)) for a, b in zip(got, ref)])
    assert exact == 1.0  # bit-exact under the float contract


def test_c3_one_step_brute_force_sample(orc):
    # full N, bench configuration: 300 agents checked against the O(N) brute-force scan
    cfg = C3_BOIDS
    m = make(cfg)
    st0 = oinit(orc, cfg, m)
    m.step(1)
    got = state(m)
    ids = np.random.default_rng(1).choice(cfg["n"], 300, replace=False)
    px, py, vx, vy, nn = orc.boids_step_sample(st0, oparams(orc, cfg), ids)
    assert np.array_equal(got[0][ids], px) and np.array_equal(got[1][ids], py)
    assert np.array_equal(got[2][ids], vx) and np.array_equal(got[3][ids], vy)
    assert 20 < nn.mean() < 45  # ~ rho*pi*R^2 = 31.4 neighbours


def test_c3_hundred_steps_ensemble(orc):
    cfg = C3_BOIDS
    m = make(cfg)
    st0 = oinit(orc, cfg, m)
    m.step(cfg["steps"])
    ms_g, po_g = m.metrics("mean_speed"), m.metrics("polarisation")
    ref, ms_o, po_o = orc.boids_run(st0, oparams(orc, cfg), cfg["steps"])
    assert abs(ms_g[-1] - ms_o[-1]) <= 1e-3 * ms_o[-1]
    assert abs(po_g[-1] - po_o[-1]) <= 1e-3
    got = state(m)
    match = np.mean([np.array_equal(a.view(np.uint32), b.view(np.uint32)) for a, b in zip(got, ref)])
    assert match == 1.0


def test_dense_flock(orc):
    # strong cohesion packs agents into few cells (long candidate runs per lane);
    # results must still be exact
    cfg = dict(C3_BOIDS, n=6000, L=100.0, R=10.0, rs=0.5, wc=0.5, wa=0.5, ws=0.0, vmax=2.0, seed=9)
    m = make(cfg)
    st = oinit(orc, cfg, m)
    P = oparams(orc, cfg)
    m.step(40)
    for _ in range(40):
        st = orc.boids_step(st, P)
    for a, b in zip(state(m), st):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("kw", [dict(L=15.0, R=7.0, rs=2.0), dict(L=64.0, R=7.5, rs=3.0),
                                dict(L=200.0, R=10.0, wa=1.0, wc=0.3, ws=0.4, vmax=0.5)])
def test_small_boxes_and_params(orc, kw):
    cfg = dict(C3_BOIDS, n=1500, seed=5, **kw)
    m = make(cfg)
    st = oinit(orc, cfg, m)
    m.step(15)
    P = oparams(orc, cfg)
    for _ in range(15):
        st = orc.boids_step(st, P)
    for a, b in zip(state(m), st):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_geometry_invariance_and_io(orc):
    cfg = dict(C3_BOIDS, n=20_000, L=450.0)
    a = make(cfg)
    a.step(10)
    b = make(cfg)
    b.set_option("block", 64)
    b.set_option("grid", 7)
    b.step(4)
    b.step(6)
    for x, y in zip(state(a), state(b)):
        assert np.array_equal(x, y)
    for lanes in (8, 16):
        d = make(cfg)
        d.set_option("lanes", lanes)
        d.step(10)
        for x, y in zip(state(a), state(d)):
            assert np.array_equal(x, y)
    c = make(cfg)
    c.step(3)
    s = orc.boids_run(oinit(orc, cfg, make(cfg)), oparams(orc, cfg), 3)[0]
    for x, y in zip(state(c), s):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    c.write_column("vel_x", s[2] * 0.5)
    assert np.array_equal(c.read_column("vel_x"), (s[2] * 0.5).astype(np.float32))
    assert c.digest("pos_x") == orc.digest(s[0])


@pytest.mark.parametrize("n", [1, 2, 7])
def test_tiny_populations(orc, n):
    # degenerate cases: a single agent (no neighbours: straight line with wrap), pairs
    cfg = dict(C3_BOIDS, n=n, L=40.0, seed=13)
    m = make(cfg)
    st = oinit(orc, cfg, m)
    m.step(30)
    P = oparams(orc, cfg)
    for _ in range(30):
        st = orc.boids_step(st, P)
    for a, b in zip(state(m), st):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("L,sx", [(3000.0, "1"), (30_000.0, "1"), (3000.0, "4")])
def test_large_grid_device_scan_and_edges(orc, monkeypatch, L, sx):
    # > 2^16 cells: the hand-written chunked cell scan (at L = 30,000: 9e6 cells,
    # > 1,024 chunks, so the chunk-offset pass loops); sparse agents, so most
    # stencils touch the box edges' wrapped rows/columns as well as interior runs
    monkeypatch.setenv("AMBER_BOIDS_SX", sx)
    cfg = dict(C3_BOIDS, n=30_000, L=L, seed=17)
    m = make(cfg)
    assert m.get_option("cells_per_side") ** 2 > (1 << 16)
    st = oinit(orc, cfg, m)
    m.step(12)
    P = oparams(orc, cfg)
    for _ in range(12):
        st = orc.boids_step(st, P)
    for a, b in zip(state(m), st):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_fused_counts_across_calls_options_and_writes(orc):
    # the group step counts the next step's cells (small N): the counts must stay
    # valid across step calls, option switches (lanes) and column
    # writes -- every step against the oracle, bit for bit
    cfg = dict(C3_BOIDS, n=6_001, L=250.0, seed=29)
    m = make(cfg)
    P = oparams(orc, cfg)
    st = oinit(orc, cfg, m)
    plan = [(2, {}), (1, {"lanes": 4}), (2, {"lanes": 8}), (1, {"lanes": 16}), (2, {"lanes": 4}),
            ("write", None), (3, {"lanes": 4}), (1, {"lanes": 8})]
    for k, opts in plan:
        if k == "write":
            vx = (st[2] * np.float32(0.75)).astype(np.float32)
            m.write_column("vel_x", vx)
            st = (st[0], st[1], vx, st[3])
            continue
        for key, v in opts.items():
            m.set_option(key, v)
        m.step(k)
        for _ in range(k):
            st = orc.boids_step(st, P)
        for a, b in zip(state(m), st):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert m.metrics("mean_speed").shape[0] >= 1


def test_quantised_velocity_stencil_paths(orc):
    # the pre-quantised-velocity stencil (QV: q24(v) carried as int32 in the
    # sorted records) and the float-velocity stencil give the same integers (B3)
    cfg = dict(C3_BOIDS, n=20_000, L=450.0)
    a = make(cfg)
    assert a.get_option("qv") == 1
    a.step(10)
    b = make(cfg)
    b.set_option("qv", 0)
    assert b.get_option("qv") == 0
    b.step(10)
    for x, y in zip(state(a), state(b)):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    # a written velocity beyond the int32 range of q24 (|v| >= 128): the next step
    # runs the float stencil, the clamp brings every velocity back below vmax, and
    # the steps after it run QV again -- each step equal to the oracle
    c = make(cfg)
    st = oinit(orc, cfg, c)
    vx = (st[2] * np.float32(300.0)).astype(np.float32)
    c.write_column("vel_x", vx)
    st = (st[0], st[1], vx, st[3])
    assert c.get_option("qv") == 0
    P = oparams(orc, cfg)
    for k in range(4):
        c.step(1)
        st = orc.boids_step(st, P)
        for x, y in zip(state(c), st):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), k
        assert c.get_option("qv") == 1
    # vmax >= 64: velocities may leave the QV range, the float stencil always runs
    d = make(dict(cfg, vmax=80.0, L=2000.0))
    assert d.get_option("qv") == 0


@pytest.mark.parametrize("sx", ["1", "2", "3", "4", "8"])
def test_x_subdivided_cells(orc, monkeypatch, sx):
    # rows of R-high cells split into sx columns in x (stencil runs (2 + 1/sx) cs
    # wide): the same bits for every sx, and the oracle's, incl. the wrapped edges
    monkeypatch.setenv("AMBER_BOIDS_SX", sx)
    for kw in (dict(n=20_000, L=450.0), dict(n=6000, L=100.0, rs=0.5, wc=0.5, wa=0.5, ws=0.0), dict(n=3000, L=50.0)):
        cfg = dict(C3_BOIDS, seed=21, **kw)
        m = make(cfg)
        assert m.get_option("x_subdivision") == int(sx)
        st = oinit(orc, cfg, m)
        m.step(8)
        P = oparams(orc, cfg)
        for _ in range(8):
            st = orc.boids_step(st, P)
        for x, z in zip(state(m), st):
            assert np.array_equal(x.view(np.uint32), z.view(np.uint32))


def test_v3_full_size_region_vs_oracle(orc):
    # the SURVEY 8(d) variant V3 at its full size (N = 1e8, L = 31,623) in the
    # bench's launch configuration (QV records, x-subdivided rows, 40-register
    # stencil): the oracle builds the whole initial population itself (B1),
    # the device's must equal it; then 3 steps of the oracle on the agents of a
    # 304 x 304 window around (10000, 10000) -- a 200 x 200 core plus a margin
    # 3 (R + 2 vmax) + R wider than any dependency of the core's agents -- and
    # every core agent's state after 3 device steps must equal the oracle's
    from paper_2601_16292_b200.workloads import V3_BOIDS_SCALE as cfg
    m = make(cfg)
    ref0 = orc.boids_init(cfg["n"], cfg["L"], cfg["seed"])
    for a, b in zip(state(m), ref0):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    K, x0, W = 3, 10_000.0, 200.0
    M = K * (cfg["R"] + 2 * cfg["vmax"] * cfg["dt"]) + cfg["R"]
    px, py = ref0[0], ref0[1]
    win = np.nonzero((px >= x0 - M) & (px < x0 + W + M) & (py >= x0 - M) & (py < x0 + W + M))[0]
    core = (px[win] >= x0) & (px[win] < x0 + W) & (py[win] >= x0) & (py[win] < x0 + W)
    assert core.sum() > 3000
    sub = tuple(c[win] for c in ref0)
    P = oparams(orc, cfg)
    for _ in range(K):
        sub = orc.boids_step(sub, P)
    m.step(1)
    m.step(K - 1)
    got = state(m)
    for g, o in zip(got, sub):
        assert np.array_equal(g[win[core]].view(np.uint32), o[core].view(np.uint32))


def test_pdl_off_and_on_both_equal_the_oracle(orc, tmp_path):
    # the scatter-scan and stencil kernels are launched with programmatic
    # dependent launch and wait on the device for their predecessor; with
    # AMBER_PDL=0 (fixed per process) they launch normally.  Both must equal the
    # oracle at every checked step.
    import os
    import subprocess
    import sys
    cfg = dict(C3_BOIDS, n=20_000, L=450.0, seed=41)
    steps = 12
    out = tmp_path / "cols.npz"
    code = (
        "import numpy as np, sys\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_2601_16292_b200 import Model, boids_params\n"
        f"m = Model('boids', {cfg['n']}, boids_params(*{[cfg[k] for k in KEYS]!r}), {cfg['seed']})\n"
        f"m.step({steps})\n"
        f"np.savez({str(out)!r}, *[m.read_column(c) for c in ('pos_x', 'pos_y', 'vel_x', 'vel_y')])\n")
    env = dict(os.environ, AMBER_PDL="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    m = make(cfg)
    st = oinit(orc, cfg, m)
    P = oparams(orc, cfg)
    m.step(steps)
    for _ in range(steps):
        st = orc.boids_step(st, P)
    off = np.load(out)
    for k, (a, b) in enumerate(zip(state(m), st)):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), "PDL on"
        assert np.array_equal(off[f"arr_{k}"].view(np.uint32), b.view(np.uint32)), "PDL off"
