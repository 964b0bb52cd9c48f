#!/usr/bin/env python
"""SURVEY 8(d) roofline variants V2 (SIR, N = 1e8) and V3 (Boids, N = 1e8) on
one B200 through the public API: CUDA-event step time, per-kernel device time
from the library's event profiler, algorithmic bytes per step, and the
properties that hold at any size (S + I + R = N, S non-increasing, R
non-decreasing; Boids speed clamp).  One JSON object per variant on stdout.
  python tools/measure_scale.py [v2] [v3]
"""
import json
import os
import sys

# load every kernel at context creation: lazy module loading inside a timed
# region would be counted as step time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_16292_b200 import Model, boids_params, sir_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def timed(m, k):
    m.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    m.step(k)
    e1.record(m.stream)
    m.synchronize()
    ms = e0.elapsed_time(e1)
    prof = m.profile_results()
    m.profile(False)
    return ms, prof


def warm_sir():
    # first use of each step kernel loads its module (CUDA lazy loading, ~0.1 s):
    # keep that out of the timed regions
    for pers in (0, 1):
        w = Model("sir", 5000, sir_params(10.0, 0.05, 0.1, 0.01), 1)
        w.set_option("persistent", pers)
        w.step(3)
        w.synchronize()
        w.close()


def v2():
    c = W.V2_SIR_SCALE
    warm_sir()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = Model("sir", c["n"], sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"]), c["seed"])
    m.synchronize()
    build_s = time.perf_counter() - t0
    _, _, _, arcs = m.column_info("col_idx")
    kbar = arcs / c["n"]
    m.set_option("persistent", 0)  # one pull launch per step: per-step kernel times
    ms, prof = timed(m, c["steps"])
    S, I, R = (m.metrics(x).astype(np.int64) for x in ("S", "I", "R"))
    assert ((S + I + R) == c["n"]).all() and (np.diff(S) <= 0).all() and (np.diff(R) >= 0).all()
    # algorithmic bytes of step t: state read + written (2 B/agent) plus the
    # rows of the smaller side the direction-optimizing step traverses: row_ptr pair (8 B),
    # columns (4 B/arc) and one neighbour-state byte per arc
    s_prev = np.concatenate([[c["n"] - round(c["init_frac"] * c["n"])], S[:-1]])
    i_prev = np.concatenate([[round(c["init_frac"] * c["n"])], I[:-1]])
    side = np.minimum(s_prev, i_prev).astype(np.float64)
    alg = 2.0 * c["n"] + side * (8.0 + 5.0 * kbar)
    kern = {name: (cnt, tot) for name, cnt, tot in prof}
    step_ms = ms / c["steps"]
    m2 = Model("sir", c["n"], sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"]), c["seed"])
    ms_p, prof_p = timed(m2, c["steps"])  # default persistent cooperative launch
    assert m2.digest("state") == m.digest("state")
    out = dict(variant="V2 SIR G(1e8, 5e8) x20 (SURVEY 8(d) added roofline variant)", n=c["n"], arcs=arcs,
               build_s=build_s, steps=c["steps"], ms_per_step=step_ms, ms_per_step_persistent=ms_p / c["steps"],
               agent_updates_per_s=c["n"] * c["steps"] / (ms_p / 1e3),
               alg_bytes_per_step=float(alg.mean()),
               roofline={"bound": "hbm", "achieved": float(alg.sum() / (ms_p / 1e3) / 1e9), "peak": HBM,
                         "unit": "GB/s", "frac": float(alg.sum() / (ms_p / 1e3) / 1e9 / HBM),
                         "timing": "default persistent cooperative launch (direction-optimizing), CUDA events",
                         "alg_rule": "2 B/agent + (8 + 5*kbar) B per agent of the smaller of S, I"},
               kernels=prof, kernels_persistent=prof_p, S=S.tolist(), I=I.tolist(), R=R.tolist())
    m.close()
    m2.close()
    return out


def v3():
    c = W.V3_BOIDS_SCALE
    bp = boids_params(*[c[k] for k in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = Model("boids", c["n"], bp, c["seed"])
    m.synchronize()
    build_s = time.perf_counter() - t0
    m.step(1)
    ms, prof = timed(m, c["steps"] - 1)
    vx, vy = m.read_column("vel_x"), m.read_column("vel_y")
    sp = np.sqrt(vx.astype(np.float64) ** 2 + vy.astype(np.float64) ** 2)
    assert sp.max() <= c["vmax"] * (1 + 1e-6)
    px = m.read_column("pos_x")
    assert px.min() >= 0 and px.max() < c["L"]
    alg = 48.0 * c["n"]  # 32 B state in/out + ~16 B binning per agent-update
    step_ms = ms / (c["steps"] - 1)
    out = dict(variant="V3 Boids N=1e8 L=31623 x10 (SURVEY 8(d) added roofline variant)", n=c["n"],
               build_s=build_s, steps=c["steps"] - 1, ms_per_step=step_ms,
               agent_updates_per_s=c["n"] / (step_ms / 1e3),
               hbm_alg={"achieved": alg / (step_ms / 1e3) / 1e9, "peak": HBM, "unit": "GB/s",
                        "frac": alg / (step_ms / 1e3) / 1e9 / HBM, "alg_bytes_per_agent": 48},
               mean_speed=m.metrics("mean_speed").tolist(), kernels=prof)
    m.close()
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["v2", "v3"]
    for w in which:
        print(json.dumps({"v2": v2, "v3": v3}[w]()), flush=True)
