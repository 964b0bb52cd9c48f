"""Pins for the oracle's Boids step (contract B1-B8; BJ config 3).

The paper has no flocking model (BJ substitutes Boids for its Random Walk),
so the rules are DESIGN.md readings; the pins check the oracle against the
plain brute-force definition, scipy's periodic KD-tree (library neighbour
query), closed-form special cases, a hand-worked two-agent case, and a
double-precision evaluation of the same rules.
"""
import numpy as np
import pytest
from scipy.spatial import cKDTree

from paper_2601_16292_b200.workloads import C3_BOIDS


def params(orc, **kw):
    base = dict(L=1000.0, R=10.0, rs=2.0, wc=0.01, wa=0.125, ws=0.05, vmax=2.0, dt=1.0)
    base.update(kw)
    return orc.boids_params(**base)


def dense_state(orc, n, L, seed):
    return orc.boids_init(n, L, seed)


def test_init_ranges(orc):
    L = 1000.0
    px, py, vx, vy = orc.boids_init(50_000, L, 3)
    assert (px >= 0).all() and (px < L).all() and (py >= 0).all() and (py < L).all()
    sp = np.sqrt(vx.astype(np.float64) ** 2 + vy.astype(np.float64) ** 2)
    assert np.abs(sp - 1).max() < 3e-7  # speed 1 within float rounding (B1)
    ang = np.arctan2(vy, vx)
    hist, _ = np.histogram(ang, bins=8, range=(-np.pi, np.pi))
    assert (np.abs(hist - 50_000 / 8) < 5 * np.sqrt(50_000 / 8)).all()  # uniform angle
    assert abs(px.mean() - L / 2) < 5 * L / np.sqrt(12 * 50_000)


@pytest.mark.parametrize("kw", [{}, {"R": 37.0, "rs": 9.0}, {"L": 64.0, "R": 7.5, "rs": 3.0},
                                {"wa": 1.0, "wc": 0.3, "ws": 0.4, "vmax": 0.5}])
def test_binned_equals_brute_force(orc, kw):
    # B pin (i): cell-list step == O(N^2) definition, bit for bit, over many steps
    P = params(orc, **kw)
    st = dense_state(orc, 2000, P.L, 11)
    for _ in range(12):
        a = orc.boids_step(st, P, brute=False)
        b = orc.boids_step(st, P, brute=True)
        for x, y in zip(a, b):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
        st = a


def test_neighbour_counts_match_periodic_kdtree(orc):
    # B2 pinned by scipy.spatial.cKDTree(boxsize=L).query_ball_point (inclusive radius)
    P = params(orc, L=200.0)
    px, py, vx, vy = orc.boids_init(3000, P.L, 5)
    ids = np.arange(0, 3000, 7)
    *_, nn = orc.boids_step_sample((px, py, vx, vy), P, ids)
    pts = np.stack([px, py], 1).astype(np.float64)
    tree = cKDTree(pts, boxsize=P.L)
    for k, i in enumerate(ids):
        cand = tree.query_ball_point(pts[i], r=P.R)
        d = np.array([np.hypot(*((pts[j] - pts[i] + P.L / 2) % P.L - P.L / 2)) for j in cand])
        borderline = np.abs(d - P.R) < 1e-3
        lo = len(cand) - 1 - borderline.sum()
        assert lo <= nn[k] <= len(cand) - 1 + 1e-9 + borderline.sum()


def test_zero_weights_is_free_flight(orc):
    # B pin (ii): p' = wrap(p + v dt) exactly, v unchanged
    P = params(orc, wc=0.0, wa=0.0, ws=0.0, dt=1.0)
    px, py, vx, vy = orc.boids_init(5000, P.L, 8)
    npx, npy, nvx, nvy = orc.boids_step((px, py, vx, vy), P)
    assert np.array_equal(nvx, vx) and np.array_equal(nvy, vy)
    ex = (px + vx).astype(np.float32)
    ex = np.where(ex < 0, ex + np.float32(P.L), ex).astype(np.float32)
    ex = np.where(ex >= P.L, ex - np.float32(P.L), ex).astype(np.float32)
    assert np.array_equal(npx, ex)


def test_isolated_agents_move_straight_with_wrap(orc):
    # B pin (iii): agents farther than R apart fly straight and wrap
    P = params(orc, L=100.0)
    px = np.array([0.5, 50.0, 99.5], np.float32)
    py = np.array([50.0, 0.2, 99.0], np.float32)
    vx = np.array([-1.0, 0.6, 0.8], np.float32)
    vy = np.array([0.0, -0.8, 0.6], np.float32)
    a = orc.boids_step((px, py, vx, vy), P)
    assert np.allclose(a[0], [99.5, 50.6, 0.3], atol=1e-4)
    assert np.allclose(a[1], [50.0, 99.4, 99.6], atol=1e-4)
    assert np.array_equal(a[2], vx) and np.array_equal(a[3], vy)
    assert ((a[0] >= 0) & (a[0] < P.L) & (a[1] >= 0) & (a[1] < P.L)).all()


def test_alignment_only_gives_neighbour_mean(orc):
    # B pin (iv): w_a = 1, others 0 -> v' = mean neighbour velocity (fixed-point quantum)
    P = params(orc, L=60.0, wc=0.0, ws=0.0, wa=1.0, vmax=10.0)
    st = orc.boids_init(400, P.L, 4)
    px, py, vx, vy = st
    out = orc.boids_step(st, P, brute=True)
    pts = np.stack([px, py], 1).astype(np.float64)
    tree = cKDTree(pts, boxsize=P.L)
    for i in range(0, 400, 13):
        nb = [j for j in tree.query_ball_point(pts[i], r=P.R) if j != i]
        if nb:
            assert abs(out[2][i] - vx[nb].astype(np.float64).mean()) < 1e-6
            assert abs(out[3][i] - vy[nb].astype(np.float64).mean()) < 1e-6


def test_two_agent_worked_example(orc):
    # hand-worked: two agents 1 apart, at rest -> v0' = (wc*1 - ws*1, 0) = (-0.04, 0)
    P = params(orc, L=100.0)
    st = (np.array([10.0, 11.0], np.float32), np.array([20.0, 20.0], np.float32),
          np.zeros(2, np.float32), np.zeros(2, np.float32))
    px, py, vx, vy = orc.boids_step(st, P)
    assert abs(vx[0] - (-0.04)) < 1e-7 and abs(vx[1] - 0.04) < 1e-7
    assert vy[0] == 0.0 and vy[1] == 0.0
    assert abs(px[0] - 9.96) < 1e-5 and abs(px[1] - 11.04) < 1e-5


def test_speed_clamp_and_box(orc):
    # B pin (v): |v'| <= vmax (+1 ulp), p' in [0, L)
    P = params(orc, L=80.0, wc=0.5, ws=0.5, vmax=1.5)
    st = orc.boids_init(3000, P.L, 2)
    for _ in range(5):
        st = orc.boids_step(st, P)
        sp = np.hypot(st[2].astype(np.float64), st[3].astype(np.float64))
        assert sp.max() <= 1.5 * (1 + 2e-7)
        assert (st[0] >= 0).all() and (st[0] < P.L).all()
        assert (st[1] >= 0).all() and (st[1] < P.L).all()


def test_float_contract_close_to_real_arithmetic(orc):
    # B pin (vi): one float32 step stays within the B8 one-step tolerance of the
    # same rules evaluated in double precision
    P = params(orc, L=300.0)
    st = orc.boids_init(3000, P.L, 13)
    f32 = orc.boids_step(st, P, brute=True)
    f64 = orc.boids_step_f64(st, P)
    dp = (f32[0] - f64[0] + P.L / 2) % P.L - P.L / 2
    assert (np.abs(dp) <= 1e-4 * np.maximum(np.abs(f64[0]), 1)).all()
    assert (np.abs(f32[2] - f64[2]) <= 1e-4 * np.maximum(np.abs(f64[2]), 1e-3)).all()


def test_metrics_definitions(orc):
    vx = np.array([1.0, 0.0, -3.0], np.float32)
    vy = np.array([0.0, 2.0, 4.0], np.float32)
    ms, po = orc.boids_metrics(vx, vy)
    assert abs(ms - (1 + 2 + 5) / 3) < 1e-15
    ux, uy = 1 + 0 - 0.6, 0 + 1 + 0.8
    assert abs(po - np.hypot(ux, uy) / 3) < 1e-15


def test_c3_short_run_statistics(orc):
    # sanity: C3 initial state, two steps; speeds bounded and polarisation small
    cfg = C3_BOIDS
    P = params(orc, **{k: cfg[k] for k in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")})
    st = orc.boids_init(cfg["n"], cfg["L"], cfg["seed"])
    _, ms, po = orc.boids_run(st, P, 2)
    assert 0.5 < ms[-1] <= 2.0 and po[-1] < 0.05


def test_init_equals_curand_reformulation(orc, curand_host):
    # B1 bit for bit: positions from 32-bit lanes 2i, 2i+1 of tag 0x20 (R4, R8);
    # velocity by rejection in the unit disc with counter (lo32 i, hi32 i,
    # attempt, 0x21), words 0 and 1; every draw from cuRAND's Philox routine,
    # every float op a numpy float32 op (IEEE single rounding, no FMA)
    n, L = 20_000, np.float32(1000.0)
    for seed in (3, (7 << 32) | 3):
        px, py, vx, vy = orc.boids_init(n, float(L), seed)
        i = np.arange(n, dtype=np.uint64)
        u01 = lambda w: (np.asarray(w, np.uint32) >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
        assert np.array_equal(px, L * u01(curand_host.lane32(seed, 0x20, 2 * i, 0)))
        assert np.array_equal(py, L * u01(curand_host.lane32(seed, 0x20, 2 * i + 1, 0)))
        wx, wy = np.full(n, np.nan, np.float32), np.full(n, np.nan, np.float32)
        todo, attempt, retried = np.arange(n, dtype=np.uint64), 0, 0
        key = [[seed & 0xFFFFFFFF, seed >> 32]]
        while todo.size:
            ctr = np.stack([(todo & np.uint64(0xFFFFFFFF)).astype(np.uint32), (todo >> np.uint64(32)).astype(np.uint32),
                            np.full(todo.size, attempt, np.uint32), np.full(todo.size, 0x21, np.uint32)], 1)
            w = curand_host.blocks(ctr, key)
            a = np.float32(2.0) * u01(w[:, 0]) - np.float32(1.0)
            b = np.float32(2.0) * u01(w[:, 1]) - np.float32(1.0)
            s2 = a * a + b * b
            ok = (s2 > 0) & (s2 <= 1)
            s = np.sqrt(s2[ok])
            wx[todo[ok]], wy[todo[ok]] = a[ok] / s, b[ok] / s
            todo, attempt = todo[~ok], attempt + 1
            retried += int(todo.size)
        assert retried > 0.15 * n  # about 1 - pi/4 of the agents need a second attempt
        assert np.array_equal(vx.view(np.uint32), wx.view(np.uint32))
        assert np.array_equal(vy.view(np.uint32), wy.view(np.uint32))
