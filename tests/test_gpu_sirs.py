"""GPU parity: SIR in continuous space (NEXT-1: the paper's SIR benchmark,
PAPER.md Sec. 5.1.1 l.203 + Listing 2) vs the oracle, bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2601_16292_b200 import Model, sir_space_params
from paper_2601_16292_b200.workloads import SIRS_PAPER, SIRS_SCALE

KEYS = ("L", "r", "p_infect", "p_recover", "init_frac")


def make(cfg, **kw):
    return Model("sir_space", cfg["n"], sir_space_params(*[cfg[k] for k in KEYS]), cfg["seed"], **kw)


def k_inf(cfg):
    import oracle
    return oracle.round_count(cfg["init_frac"] * cfg["n"])


def test_paper_size_bit_exact(orc):
    cfg = SIRS_PAPER
    m = make(cfg)
    px, py, st = orc.sirs_init(cfg["n"], cfg["L"], k_inf(cfg), cfg["seed"])
    assert np.array_equal(m.read_column("pos_x"), px) and np.array_equal(m.read_column("pos_y"), py)
    assert np.array_equal(m.read_column("state"), st)
    rp, col = orc.sirs_contacts(px, py, cfg["r"])
    assert np.array_equal(m.read_column("row_ptr"), rp) and np.array_equal(m.read_column("col_idx"), col)
    ref, counts = orc.sirs_run(rp, col, st, cfg["seed"], cfg["p_infect"], cfg["p_recover"], 0, cfg["steps"])
    m.step(40)
    m.step(60)
    assert np.array_equal(m.read_column("state"), ref)
    for k, nm in enumerate("SIR"):
        assert np.array_equal(m.metrics(nm), counts[:, k])


@pytest.mark.parametrize("n,L,r", [(1, 10.0, 1.0), (50, 5.0, 2.0), (2000, 30.0, 7.9), (3000, 100.0, 0.5)])
def test_sizes_and_radii(orc, n, L, r):
    cfg = dict(n=n, L=L, r=r, p_infect=0.3, p_recover=0.1, init_frac=0.02, seed=4)
    m = make(cfg)
    px, py, st = orc.sirs_init(n, L, k_inf(cfg), 4)
    rp, col = orc.sirs_contacts(px, py, r, cap=n * n + 1)
    assert np.array_equal(m.read_column("col_idx"), col)
    ref, _ = orc.sirs_run(rp, col, st, 4, 0.3, 0.1, 0, 25)
    m.step(25)
    assert np.array_equal(m.read_column("state"), ref)


def test_scale_contacts_all_rows_and_steps(orc):
    # N = 1e7 at the paper's density: the oracle builds positions, initial state
    # and the whole contact graph itself (its grid search, pinned against the
    # all-pairs definition on CPU); the device's columns must equal them
    # entirely; then 20 steps of the oracle on ITS graph vs the device
    cfg = SIRS_SCALE
    m = make(cfg)
    px, py, st = orc.sirs_init(cfg["n"], cfg["L"], k_inf(cfg), cfg["seed"])
    assert np.array_equal(m.read_column("pos_x"), px) and np.array_equal(m.read_column("pos_y"), py)
    assert np.array_equal(m.read_column("state"), st)
    rp, col = orc.sirs_contacts_grid(px, py, cfg["L"], cfg["r"])
    assert np.array_equal(m.read_column("row_ptr"), rp)
    assert np.array_equal(m.read_column("col_idx"), col)
    ref, counts = orc.sirs_run(rp, col, st, cfg["seed"], cfg["p_infect"], cfg["p_recover"], 0, 20)
    m.step(20)
    assert np.array_equal(m.read_column("state"), ref)
    assert np.array_equal(m.metrics("I")[-20:], counts[:, 1])
