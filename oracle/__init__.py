"""CPU oracle for the AMBER hot path -- TEST INFRASTRUCTURE ONLY.

This package wraps ``oracle/amber_oracle.c`` (plain, single-threaded C that
follows the paper's synchronous-update definition step by step; see the C
file's header and DESIGN.md "Contract").  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it.  The product package
``paper_2601_16292_b200`` never imports it and shares no code with it.

Functions whose parity is not pinned by the paper or by mathematics say so in
their docstring ("parity unpinned"); every other one is pinned by a
``tests/test_oracle_*.py`` case listed in DESIGN.md.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "amber_oracle.c")
HDR = os.path.join(HERE, "amber_oracle.h")
LIB = os.environ.get("AMBER_ORACLE_LIB") or os.path.join(HERE, "liboracle.so")  # (sanitizer builds: tests)

TAG_WEALTH_RECV = 0x01
TAG_SIR_TX = 0x10
TAG_SIR_REC = 0x11
TAG_SIR_INIT = 0x12
TAG_GRAPH = 0x13
TAG_BOIDS_POS = 0x20
TAG_BOIDS_VEL = 0x21
TAG_WALK_POS = 0x30
TAG_WALK_VEL = 0x31
TAG_SIRS_POS, TAG_SIRS_TX, TAG_SIRS_INIT, TAG_SIRS_REC = 0x40, 0x41, 0x42, 0x43
S, I, R = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile liboracle.so with the contract's float flags (B7)."""
    stale = (not os.path.exists(LIB)) or any(
        os.path.getmtime(p) > os.path.getmtime(LIB) for p in (SRC, HDR))
    if force or stale:
        cmd = ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-Wall", "-o", LIB, SRC, "-lm"]
        subprocess.check_call(cmd)
    return LIB


class BoidsParams(C.Structure):
    _fields_ = [(k, C.c_float) for k in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        u32p, u64p, i32p, i64p = (C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_int32), C.POINTER(C.c_int64))
        u8p, f32p, f64p = C.POINTER(C.c_uint8), C.POINTER(C.c_float), C.POINTER(C.c_double)
        sig = {
            "orc_philox4x32_10": (None, [u32p, u32p, u32p]),
            "orc_lane64": (C.c_uint64, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32]),
            "orc_lane32": (C.c_uint32, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32]),
            "orc_mulhi64": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "orc_bernoulli_threshold": (C.c_uint64, [C.c_double]),
            "orc_u01": (C.c_float, [C.c_uint32]),
            "orc_round_count": (C.c_int64, [C.c_double]),
            "orc_mix64": (C.c_uint64, [C.c_uint64]),
            "orc_digest_bits32": (C.c_uint64, [u32p, C.c_int64, C.c_int64]),
            "orc_digest_u8": (C.c_uint64, [u8p, C.c_int64, C.c_int64]),
            "orc_wealth_receiver": (C.c_int64, [C.c_uint64, C.c_int64, C.c_int64, C.c_uint32,
                                                C.c_int]),
            "orc_wealth_step": (C.c_int, [C.c_int64, C.c_int32, C.c_int, C.c_uint64, C.c_uint32,
                                          i32p, i32p]),
            "orc_wealth_run": (C.c_int, [C.c_int64, C.c_int32, C.c_int, C.c_uint64, C.c_uint32,
                                         C.c_int64, i32p, i64p, i64p, u64p]),
            "orc_er_draw": (None, [C.c_uint64, C.c_int64, C.c_int64, i64p, i64p]),
            "orc_er_graph": (C.c_int64, [C.c_int64, C.c_int64, C.c_uint64, i32p, i32p]),
            "orc_sir_init": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, u8p]),
            "orc_sir_tx_word": (C.c_uint32, [C.c_uint64, C.c_int64, C.c_int64, C.c_uint32]),
            "orc_sir_step": (None, [C.c_int64, i32p, i32p, C.c_uint64, C.c_uint32, C.c_uint64,
                                    C.c_uint64, u8p, u8p]),
            "orc_sir_run": (C.c_int, [C.c_int64, i32p, i32p, C.c_uint64, C.c_double, C.c_double,
                                      C.c_uint32, C.c_int64, u8p, i64p, u64p]),
            "orc_sir_replicate": (C.c_int64, [C.c_int64, C.c_double, C.c_double, C.c_double,
                                              C.c_double, C.c_uint64, C.c_int64]),
            "orc_sir_sweep": (C.c_int, [C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int64,
                                        f64p, u64p, C.c_int64, f64p]),
            "orc_boids_init": (None, [C.c_int64, C.c_float, C.c_uint64, f32p, f32p, f32p, f32p]),
            "orc_boids_step_brute": (None, [C.c_int64, C.POINTER(BoidsParams)] + [f32p] * 8),
            "orc_boids_step_brute_sample": (None, [C.c_int64, C.POINTER(BoidsParams)] + [f32p] * 4
                                            + [C.c_int64, i64p] + [f32p] * 4 + [i64p]),
            "orc_boids_step_binned": (C.c_int, [C.c_int64, C.POINTER(BoidsParams)] + [f32p] * 8),
            "orc_boids_metrics": (None, [C.c_int64, f32p, f32p, f64p, f64p]),
            "orc_boids_run": (C.c_int, [C.c_int64, C.POINTER(BoidsParams), C.c_int64] + [f32p] * 4
                              + [f64p, f64p]),
            "orc_boids_step_brute_f64": (None, [C.c_int64, C.POINTER(BoidsParams)] + [f64p] * 8),
            "orc_sirs_init": (C.c_int, [C.c_int64, C.c_float, C.c_int64, C.c_uint64, f32p, f32p, u8p]),
            "orc_sirs_contacts": (C.c_int64, [C.c_int64, f32p, f32p, C.c_float, i32p, i32p, C.c_int64]),
            "orc_sirs_contacts_grid": (C.c_int64, [C.c_int64, f32p, f32p, C.c_float, C.c_float, i32p, i32p,
                                                   C.c_int64]),
            "orc_sirs_step": (None, [C.c_int64, i32p, i32p, C.c_uint64, C.c_uint32, C.c_uint64,
                                     C.c_uint64, u8p, u8p]),
            "orc_sirs_run": (C.c_int, [C.c_int64, i32p, i32p, C.c_uint64, C.c_double, C.c_double,
                                       C.c_uint32, C.c_int64, u8p, i64p]),
            "orc_walk_init": (None, [C.c_int64, C.c_float, C.c_uint64, f32p, f32p]),
            "orc_walk_step": (None, [C.c_int64, C.c_float, C.c_float, C.c_uint64, C.c_uint32, f32p, f32p,
                                     f32p, f32p]),
            "orc_walk_run": (C.c_int, [C.c_int64, C.c_float, C.c_float, C.c_uint64, C.c_uint32,
                                       C.c_int64, f32p, f32p, f32p, f32p, f64p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _check(rc):
    if rc < 0:
        raise RuntimeError(f"oracle error {rc}")
    return rc


# ----------------------------------------------------------------- RNG (R1-R8)
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32).copy()
    k = np.asarray(key, dtype=np.uint32).copy()
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(out, C.c_uint32))
    return out


def lane64(seed, tag, u, t):
    return int(lib().orc_lane64(seed, tag, u, t))


def lane32(seed, tag, u, t):
    return int(lib().orc_lane32(seed, tag, u, t))


def mulhi64(x, n):
    return int(lib().orc_mulhi64(x, n))


def bernoulli_threshold(p):
    return int(lib().orc_bernoulli_threshold(p))


def u01(x):
    return float(lib().orc_u01(x))


def round_count(x):
    return int(lib().orc_round_count(x))


def mix64(z):
    return int(lib().orc_mix64(z))


def digest(col, id0=0):
    """D1 digest of a column (int32/uint32/float32 by bit pattern, uint8 zero-extended)."""
    col = np.ascontiguousarray(col)
    if col.dtype == np.uint8:
        return int(lib().orc_digest_u8(_p(col, C.c_uint8), col.size, id0))
    bits = col.view(np.uint32)
    return int(lib().orc_digest_bits32(_p(bits, C.c_uint32), bits.size, id0))


# ---------------------------------------------------------------- wealth (W)
def wealth_receiver(seed, n, i, t, exclude_self=0):
    return int(lib().orc_wealth_receiver(seed, n, i, t, exclude_self))


def wealth_step(w, seed, t, amount=1, exclude_self=0):
    w = np.ascontiguousarray(w, dtype=np.int32)
    out = np.empty_like(w)
    _check(lib().orc_wealth_step(w.size, amount, exclude_self, seed, t, _p(w, C.c_int32),
                                 _p(out, C.c_int32)))
    return out


def wealth_run(w, seed, t0, steps, amount=1, exclude_self=0, digests=False):
    """Returns (w_after, total[steps], active[steps], digest[steps] or None)."""
    w = np.ascontiguousarray(w, dtype=np.int32).copy()
    tot = np.zeros(max(steps, 1), dtype=np.int64)
    act = np.zeros(max(steps, 1), dtype=np.int64)
    dig = np.zeros(max(steps, 1), dtype=np.uint64) if digests else None
    _check(lib().orc_wealth_run(w.size, amount, exclude_self, seed, t0, steps, _p(w, C.c_int32),
                                _p(tot, C.c_int64), _p(act, C.c_int64),
                                _p(dig, C.c_uint64) if digests else None))
    return w, tot[:steps], act[:steps], (dig[:steps] if digests else None)


# ------------------------------------------------------------ graph (G1-G4)
def er_draw(seed, n, e):
    u, v = C.c_int64(), C.c_int64()
    lib().orc_er_draw(seed, n, e, C.byref(u), C.byref(v))
    return u.value, v.value


def er_graph(n, m, seed):
    """Returns (row_ptr int32[n+1], col int32[2M'], M')."""
    row_ptr = np.zeros(n + 1, dtype=np.int32)
    col = np.zeros(max(2 * m, 1), dtype=np.int32)
    mu = _check(lib().orc_er_graph(n, m, seed, _p(row_ptr, C.c_int32), _p(col, C.c_int32)))
    return row_ptr, col[: 2 * mu].copy(), int(mu)


# ---------------------------------------------------------------- SIR (S1-S6)
def sir_init(n, k, seed):
    st = np.zeros(n, dtype=np.uint8)
    _check(lib().orc_sir_init(n, k, seed, _p(st, C.c_uint8)))
    return st


def sir_tx_word(seed, a, b, t):
    return int(lib().orc_sir_tx_word(seed, a, b, t))


def sir_step(row_ptr, col, state, seed, t, beta, gamma):
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
    col = np.ascontiguousarray(col if len(col) else np.zeros(1, np.int32), dtype=np.int32)
    state = np.ascontiguousarray(state, dtype=np.uint8)
    out = np.empty_like(state)
    lib().orc_sir_step(state.size, _p(row_ptr, C.c_int32), _p(col, C.c_int32), seed, t,
                       bernoulli_threshold(beta), bernoulli_threshold(gamma),
                       _p(state, C.c_uint8), _p(out, C.c_uint8))
    return out


def sir_run(row_ptr, col, state, seed, beta, gamma, t0, steps, digests=False):
    """Returns (state_after, counts[steps,3], digest[steps] or None)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
    col = np.ascontiguousarray(col if len(col) else np.zeros(1, np.int32), dtype=np.int32)
    st = np.ascontiguousarray(state, dtype=np.uint8).copy()
    counts = np.zeros((max(steps, 1), 3), dtype=np.int64)
    dig = np.zeros(max(steps, 1), dtype=np.uint64) if digests else None
    _check(lib().orc_sir_run(st.size, _p(row_ptr, C.c_int32), _p(col, C.c_int32), seed, beta,
                             gamma, t0, steps, _p(st, C.c_uint8), _p(counts, C.c_int64),
                             _p(dig, C.c_uint64) if digests else None))
    return st, counts[:steps], (dig[:steps] if digests else None)


def sir_replicate(n, mean_degree, beta, gamma, init_frac, seed, steps):
    return _check(int(lib().orc_sir_replicate(n, mean_degree, beta, gamma, init_frac, seed,
                                              steps)))


def sir_sweep(n, mean_degree, gamma, init_frac, betas, seeds, steps):
    betas = np.ascontiguousarray(betas, dtype=np.float64)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = np.zeros(betas.size, dtype=np.float64)
    _check(lib().orc_sir_sweep(n, mean_degree, gamma, init_frac, betas.size,
                               _p(betas, C.c_double), _p(seeds, C.c_uint64), steps,
                               _p(out, C.c_double)))
    return out


# -------------------------------------------------------------- Boids (B1-B8)
def boids_params(L=1000.0, R=10.0, rs=2.0, wc=0.01, wa=0.125, ws=0.05, vmax=2.0, dt=1.0):
    return BoidsParams(L, R, rs, wc, wa, ws, vmax, dt)


def boids_init(n, L, seed):
    arrs = [np.zeros(n, dtype=np.float32) for _ in range(4)]
    lib().orc_boids_init(n, L, seed, *[_p(a, C.c_float) for a in arrs])
    return tuple(arrs)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def boids_step(state, P, brute=False):
    px, py, vx, vy = (_f32(a) for a in state)
    outs = [np.empty_like(px) for _ in range(4)]
    args = [px.size, C.byref(P)] + [_p(a, C.c_float) for a in (px, py, vx, vy, *outs)]
    if brute:
        lib().orc_boids_step_brute(*args)
    else:
        _check(lib().orc_boids_step_binned(*args))
    return tuple(outs)


def boids_step_sample(state, P, ids):
    """Brute-force one step for the listed agents only; returns (px,py,vx,vy,n_neigh)."""
    px, py, vx, vy = (_f32(a) for a in state)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    outs = [np.empty(ids.size, dtype=np.float32) for _ in range(4)]
    nn = np.zeros(ids.size, dtype=np.int64)
    lib().orc_boids_step_brute_sample(px.size, C.byref(P),
                                      *[_p(a, C.c_float) for a in (px, py, vx, vy)],
                                      ids.size, _p(ids, C.c_int64),
                                      *[_p(a, C.c_float) for a in outs], _p(nn, C.c_int64))
    return (*outs, nn)


def boids_metrics(vx, vy):
    vx, vy = _f32(vx), _f32(vy)
    ms, po = C.c_double(), C.c_double()
    lib().orc_boids_metrics(vx.size, _p(vx, C.c_float), _p(vy, C.c_float), C.byref(ms),
                            C.byref(po))
    return ms.value, po.value


def boids_run(state, P, steps):
    """Returns (state_after, mean_speed[steps], polarisation[steps])."""
    arrs = [_f32(a).copy() for a in state]
    ms = np.zeros(max(steps, 1), dtype=np.float64)
    po = np.zeros(max(steps, 1), dtype=np.float64)
    _check(lib().orc_boids_run(arrs[0].size, C.byref(P), steps,
                               *[_p(a, C.c_float) for a in arrs], _p(ms, C.c_double),
                               _p(po, C.c_double)))
    return tuple(arrs), ms[:steps], po[:steps]


def boids_step_f64(state, P):
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in state]
    outs = [np.empty_like(arrs[0]) for _ in range(4)]
    lib().orc_boids_step_brute_f64(arrs[0].size, C.byref(P),
                                   *[_p(a, C.c_double) for a in (*arrs, *outs)])
    return tuple(outs)


# ------------------------------------------------------------ Random Walk (K)
def walk_init(n, L, seed):
    px, py = np.zeros(n, np.float32), np.zeros(n, np.float32)
    lib().orc_walk_init(n, L, seed, _p(px, C.c_float), _p(py, C.c_float))
    return px, py


def walk_step(px, py, L, vmax, seed, t):
    px, py = _f32(px), _f32(py)
    ox, oy = np.empty_like(px), np.empty_like(py)
    lib().orc_walk_step(px.size, L, vmax, seed, t, _p(px, C.c_float), _p(py, C.c_float),
                        _p(ox, C.c_float), _p(oy, C.c_float))
    return ox, oy


def walk_run(px, py, L, vmax, seed, t0, steps, origin=None):
    """Returns (px, py, mean_displacement[steps]) ; origin defaults to the input positions."""
    px, py = _f32(px).copy(), _f32(py).copy()
    ox, oy = (px.copy(), py.copy()) if origin is None else (_f32(origin[0]), _f32(origin[1]))
    md = np.zeros(max(steps, 1), np.float64)
    _check(lib().orc_walk_run(px.size, L, vmax, seed, t0, steps, _p(px, C.c_float), _p(py, C.c_float),
                              _p(ox, C.c_float), _p(oy, C.c_float), _p(md, C.c_double)))
    return px, py, md[:steps]


# ------------------------------------------------- SIR in continuous space (C)
def sirs_init(n, L, k, seed):
    px, py = np.zeros(n, np.float32), np.zeros(n, np.float32)
    st = np.zeros(n, np.uint8)
    _check(lib().orc_sirs_init(n, L, k, seed, _p(px, C.c_float), _p(py, C.c_float), _p(st, C.c_uint8)))
    return px, py, st


def sirs_contacts(px, py, r, cap=None):
    px, py = _f32(px), _f32(py)
    n = px.size
    cap = cap or max(64 * n, 1)
    rp = np.zeros(n + 1, np.int32)
    col = np.zeros(cap, np.int32)
    a = _check(int(lib().orc_sirs_contacts(n, _p(px, C.c_float), _p(py, C.c_float), r, _p(rp, C.c_int32),
                                           _p(col, C.c_int32), cap)))
    return rp, col[:a].copy()


def sirs_contacts_grid(px, py, L, r, cap=None):
    """Same lists as sirs_contacts, found through a uniform grid (large n)."""
    px, py = _f32(px), _f32(py)
    n = px.size
    cap = cap or max(64 * n, 1)
    rp = np.zeros(n + 1, np.int32)
    col = np.zeros(cap, np.int32)
    a = _check(int(lib().orc_sirs_contacts_grid(n, _p(px, C.c_float), _p(py, C.c_float), L, r, _p(rp, C.c_int32),
                                                _p(col, C.c_int32), cap)))
    return rp, col[:a].copy()


def sirs_step(rp, col, st, seed, t, p_inf, p_rec):
    rp = np.ascontiguousarray(rp, np.int32)
    col = np.ascontiguousarray(col if len(col) else np.zeros(1, np.int32), np.int32)
    st = np.ascontiguousarray(st, np.uint8)
    out = np.empty_like(st)
    lib().orc_sirs_step(st.size, _p(rp, C.c_int32), _p(col, C.c_int32), seed, t, bernoulli_threshold(p_inf),
                        bernoulli_threshold(p_rec), _p(st, C.c_uint8), _p(out, C.c_uint8))
    return out


def sirs_run(rp, col, st, seed, p_inf, p_rec, t0, steps):
    rp = np.ascontiguousarray(rp, np.int32)
    col = np.ascontiguousarray(col if len(col) else np.zeros(1, np.int32), np.int32)
    st = np.ascontiguousarray(st, np.uint8).copy()
    counts = np.zeros((max(steps, 1), 3), np.int64)
    _check(lib().orc_sirs_run(st.size, _p(rp, C.c_int32), _p(col, C.c_int32), seed, p_inf, p_rec, t0, steps,
                              _p(st, C.c_uint8), _p(counts, C.c_int64)))
    return st, counts[:steps]
