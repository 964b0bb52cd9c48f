"""GPU parity: Random Walk (NEXT-2; Sec. 5.1.1 l.205) vs the oracle, bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2601_16292_b200 import Model, walk_params
from paper_2601_16292_b200.workloads import WALK_PAPER, WALK_SCALE


def make(cfg, **kw):
    return Model("walk", cfg["n"], walk_params(cfg["L"], cfg["vmax"]), cfg["seed"], **kw)


def test_paper_size_every_step(orc):
    cfg = WALK_PAPER
    m = make(cfg)
    px, py = orc.walk_init(cfg["n"], cfg["L"], cfg["seed"])
    assert np.array_equal(m.read_column("pos_x"), px) and np.array_equal(m.read_column("origin_y"), py)
    x, y, md = orc.walk_run(px, py, cfg["L"], cfg["vmax"], cfg["seed"], 0, cfg["steps"])
    for t in range(cfg["steps"]):
        m.step(1)
    assert np.array_equal(m.read_column("pos_x"), x) and np.array_equal(m.read_column("pos_y"), y)
    got = m.metrics("mean_displacement")
    assert np.allclose(got, md, rtol=1e-6, atol=0)


@pytest.mark.parametrize("n,vmax", [(1, 1.0), (3, 2.0), (5, 0.0), (1001, 40.0), (65_539, 0.5)])
def test_sizes_and_boundaries(orc, n, vmax):
    cfg = dict(n=n, L=30.0, vmax=vmax, seed=9)
    m = make(cfg)
    m.step(7)
    m.step(13)
    px, py = orc.walk_init(n, 30.0, 9)
    x, y, _ = orc.walk_run(px, py, 30.0, vmax, 9, 0, 20)
    assert np.array_equal(m.read_column("pos_x"), x) and np.array_equal(m.read_column("pos_y"), y)


def test_checkpoint_and_geometry(orc):
    cfg = dict(WALK_PAPER, n=50_000)
    a = make(cfg)
    a.step(30)
    b = make(cfg)
    b.set_option("block", 64)
    b.set_option("grid", 3)
    b.step(10)
    sx, sy = b.read_column("pos_x"), b.read_column("pos_y")
    c = make(cfg)
    c.write_column("pos_x", sx)
    c.write_column("pos_y", sy)
    c.set_step(10)
    c.step(20)
    for m in (b, c):
        if m is b:
            m.step(20)
        assert np.array_equal(m.read_column("pos_x"), a.read_column("pos_x"))


def test_scale_first_step(orc):
    cfg = WALK_SCALE
    m = make(cfg)
    m.step(1)
    px, py = orc.walk_init(cfg["n"], cfg["L"], cfg["seed"])
    x, y = orc.walk_step(px, py, cfg["L"], cfg["vmax"], cfg["seed"], 0)
    assert np.array_equal(m.read_column("pos_x"), x) and np.array_equal(m.read_column("pos_y"), y)
