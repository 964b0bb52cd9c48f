"""Pins for the oracle's Random Walk (Sec. 5.1.1 l.205, Sec. 5.3 l.272;
DESIGN.md K1-K3).  Expected values: the plain definition evaluated with numpy
float32 arithmetic on draws from cuRAND's Philox routine, closed-form
statistics of the uniform velocity law, and boundary special cases."""
import numpy as np
import pytest

TAG_POS, TAG_VEL = 0x30, 0x31


def u01(x):
    return (np.asarray(x, np.uint32) >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)


def numpy_walk(px, py, L, vmax, seed, t, curand_host):
    n = px.size
    i = np.arange(n, dtype=np.uint64)
    ux = u01(curand_host.lane32(seed, TAG_VEL, 2 * i, t))
    uy = u01(curand_host.lane32(seed, TAG_VEL, 2 * i + 1, t))
    f2, f1, vm = np.float32(2), np.float32(1), np.float32(vmax)
    vx = (f2 * ux - f1) * vm
    vy = (f2 * uy - f1) * vm
    hi = np.nextafter(np.float32(L), np.float32(0))
    x = np.clip(px + vx, np.float32(0), hi).astype(np.float32)
    y = np.clip(py + vy, np.float32(0), hi).astype(np.float32)
    return x, y


def test_init_matches_draws(orc, curand_host):
    n, L, seed = 1000, 100.0, 7
    px, py = orc.walk_init(n, L, seed)
    i = np.arange(n, dtype=np.uint64)
    assert np.array_equal(px, np.float32(L) * u01(curand_host.lane32(seed, TAG_POS, 2 * i, 0)))
    assert np.array_equal(py, np.float32(L) * u01(curand_host.lane32(seed, TAG_POS, 2 * i + 1, 0)))


def test_steps_equal_definition(orc, curand_host):
    n, L, vmax, seed = 3001, 50.0, 3.0, 11
    px, py = orc.walk_init(n, L, seed)
    for t in range(15):
        ref = numpy_walk(px, py, L, vmax, seed, t, curand_host)
        px, py = orc.walk_step(px, py, L, vmax, seed, t)
        assert np.array_equal(px, ref[0]) and np.array_equal(py, ref[1])


def test_zero_speed_and_box(orc):
    px, py = orc.walk_init(2000, 10.0, 3)
    a, b, md = orc.walk_run(px, py, 10.0, 0.0, 3, 0, 5)
    assert np.array_equal(a, px) and np.array_equal(b, py) and (md == 0).all()
    a, b, _ = orc.walk_run(px, py, 10.0, 25.0, 3, 0, 20)  # huge steps: every agent pinned to the walls
    hi = np.nextafter(np.float32(10.0), np.float32(0))
    assert ((a >= 0) & (a <= hi) & (b >= 0) & (b <= hi)).all()
    assert 0.7 < np.isin(a, [0.0, hi]).mean() < 0.9  # P(|v| pushes past a wall) = 1 - L/(2 vmax) = 0.8


def test_velocity_law_closed_form(orc):
    # interior agents, one step: mean displacement = vmax * E|U|, U uniform on [-1,1]^2,
    # E|U| = (sqrt(2) + asinh(1)) / 3 = 0.765196...; per-component variance vmax^2/3
    n, L, vmax = 200_000, 1e6, 1.0
    px = np.full(n, L / 2, np.float32)
    py = np.full(n, L / 2, np.float32)
    a, b, md = orc.walk_run(px, py, L, vmax, 5, 0, 1)
    e_abs = (np.sqrt(2) + np.arcsinh(1.0)) / 3
    sd = 0.41 / np.sqrt(n)
    assert abs(md[0] - e_abs) < 5 * sd
    dx = a.astype(np.float64) - L / 2
    assert abs(dx.mean()) < 5 * np.sqrt(1 / 3 / n)
    assert abs(dx.var() - 1 / 3) < 0.01
