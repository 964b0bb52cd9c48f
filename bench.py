#!/usr/bin/env python
"""bench.py -- agent-updates/s of the AMBER hot path on B200 (driver contract).

Default workload (BASELINE.json config 4, the metric's "1/2/4/8 B200" config):
wealth transfer, N = 1e8 agents, int32 wealth, Philox seed 11.  One "step" is
one synchronous step of the whole population (one fused kernel launch on one
GPU; plus the cross-shard exchange when sharded).  The state (400 MB) is
larger than L2, so no L2 flush is needed between timed steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl amber|reference]
                  [--workload c4|c1|c2|c3|c5] [--no-cpu-baseline]

For N > 1 the driver launches it under torchrun (one rank per GPU over NCCL);
agents are sharded by contiguous id ranges and the timed region is the max
over ranks of the device time.  `--impl reference` times the CPU oracle (the
reference arm for this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys

# load every kernel at context creation: lazy module loading inside a timed
# region would be counted as step time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "agent-updates/sec per step (1/2/4/8 B200) and % of HBM roofline vs CPU oracle"
UNIT = "agent-updates/s"
# random 32-bit L2 atomics, any target set that fits L2 (measured on this pool's B200,
# tools/red_ceiling.cu -> profiles/r01_red_ceiling.txt): the scatter's binding roof
RED_CEILING = 1.85e11
# the fused roof of the C4 step: the same 800 MB column stream and 0.587*N random
# REDs into 4-bit packed L2-resident counters in ONE kernel, with a hash in
# place of Philox and no apply (tools/red_stream_ceiling.cu ->
# profiles/r02_red_stream_ceiling.txt, best grid): ms per N = 1e8 step
STREAM_RED_ROOF_MS = 0.3855
# the Boids stencil's own instruction sequence over shared-memory-staged candidates
# (memory latency hidden) at full residency, candidate visits per second
# (tools/alu_ceiling.cu -> profiles/r02_alu_ceiling.txt): pre-quantised-velocity
# form (the default, option qv) and float-velocity form
STENCIL_CEILING = {1: 9.337e11, 0: 7.928e11}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def host_info():
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.idx = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.05)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, pw, mx, reasons = [], [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        # "under load": samples drawing more than a third of the busiest sample's power
        hi = max(pw) if pw else 0.0
        load = [c for c, p in zip(sm, pw) if p >= hi / 3] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "samples_under_load": len(load), "power_w_max": hi,
                "window": "nvidia-smi every 20 ms over the whole GPU arm (warm-up, timed repetitions, "
                          "e2e, other configs)"}


# ------------------------------------------------------------------ oracle
def cpu_baseline_wealth(n_total, seed, steps=2):
    """Oracle (as it stands, single-threaded C) on the config's FULL population
    (N = 1e8: ~5 s per step on one core) for `steps` synchronous steps.
    Returns the cpu_baseline object."""
    import numpy as np

    import oracle
    w = np.ones(n_total, np.int32)
    t0 = time.perf_counter()
    oracle.wealth_run(w, seed, 0, steps)
    dt = time.perf_counter() - t0
    return {"value": n_total * steps / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"wealth N={n_total:.0e} (the whole config population) x {steps} steps from the "
                      f"initial state, seed {seed}, single thread, {dt:.1f}s"}


def run_reference_small(args, oracle, np):
    """--impl reference --workload c1|c2|c3|c5: the oracle on the host, the
    inputs built by the oracle itself (graphs, initial states), one JSON line
    with the same unit as the GPU arm's line for that workload."""
    from paper_2601_16292_b200 import workloads as W
    w = args.workload
    model, ncpu = host_info()
    keys = ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")
    if w == "c1":
        c = W.C1_WEALTH_SMALL
        fn, units, sample = (lambda: oracle.wealth_run(np.ones(c["n"], np.int32), c["seed"], 0, c["steps"]),
                             c["n"] * c["steps"], f"wealth N={c['n']} x {c['steps']} steps (the whole config)")
    elif w == "c2":
        c = W.C2_SIR
        m_draws, k_inf = oracle.round_count(c["n"] * c["mean_degree"] / 2.0), oracle.round_count(c["init_frac"] * c["n"])
        rp, col, _ = oracle.er_graph(c["n"], m_draws, c["seed"])
        st = oracle.sir_init(c["n"], k_inf, c["seed"])
        fn, units, sample = (lambda: oracle.sir_run(rp, col, st, c["seed"], c["beta"], c["gamma"], 0, c["steps"]),
                             c["n"] * c["steps"], f"SIR N={c['n']} x {c['steps']} steps (the whole config)")
    elif w == "c3":
        c = W.C3_BOIDS
        P = oracle.boids_params(**{k: c[k] for k in keys})
        s0 = oracle.boids_init(c["n"], c["L"], c["seed"])
        fn, units, sample = (lambda: oracle.boids_run(s0, P, 3), c["n"] * 3,
                             f"Boids N={c['n']}, first 3 of {c['steps']} steps (sparse phase; later steps denser)")
    elif w == "c5":
        c = W.C5_SWEEP
        betas, seeds = W.sweep_replicates(c)
        pick = np.arange(0, len(betas), 256)
        fn, units, sample = (lambda: oracle.sir_sweep(c["n"], c["mean_degree"], c["gamma"], c["init_frac"],
                                                      betas[pick], seeds[pick], c["steps"]),
                             c["n"] * c["steps"] * len(pick),
                             f"{len(pick)} of {len(betas)} replicates spanning all betas, nominal updates")
    else:
        print(json.dumps({"impl": "reference", "workload": w, "unavailable": "no oracle leg for this workload"}))
        return 0
    for _ in range(min(args.warmup, 1)):
        fn()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn()
    v = units * args.steps / (time.perf_counter() - t0)
    line = {"impl": "reference", "workload": w, "value": v, "unit": "agent-updates/s",
            "cpu_baseline": {"value": v, "unit": "agent-updates/s", "cores": 1, "kind": "oracle",
                             "sample": f"{sample}; host {model}, {ncpu} cpus"}}
    if w == "c5":  # replicates are independent: also the all-core aggregate (one process per core)
        import multiprocessing as mp
        jobs = [(c["n"], c["mean_degree"], c["gamma"], c["init_frac"], float(betas[k]), int(seeds[k]), c["steps"])
                for k in np.arange(0, len(betas), 32)]
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(ncpu) as pool:
            pool.map(_sweep_one, jobs, chunksize=1)
        va = c["n"] * c["steps"] * len(jobs) / (time.perf_counter() - t0)
        line["cpu_baseline_all_cores"] = {"value": va, "unit": "agent-updates/s", "cores": ncpu, "kind": "oracle",
                                          "sample": f"{len(jobs)} of {len(betas)} replicates, one process per core"}
    print(json.dumps(line), flush=True)
    return 0


def _sweep_one(job):
    import numpy as np

    import oracle
    n, kbar, gamma, init_frac, beta, seed, steps = job
    return oracle.sir_sweep(n, kbar, gamma, init_frac, np.array([beta]), np.array([seed], np.uint64), steps)[0]


C4_L2 = "state (400 MB int32 column) larger than L2; no flush"


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores (bounded sample)."""
    import numpy as np

    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    oracle.build()
    if args.workload != "c4":
        return run_reference_small(args, oracle, np)
    from paper_2601_16292_b200.workloads import C4_WEALTH_SCALE as cfg
    # size the per-step sample so warmup + steps stay within ~2-3 minutes
    n_probe = 2_000_000
    w = np.ones(n_probe, np.int32)
    t0 = time.perf_counter()
    oracle.wealth_step(w, cfg["seed"], 0)
    per_agent = (time.perf_counter() - t0) / n_probe
    budget = 150.0
    n_s = int(max(100_000, min(cfg["n"], budget / (per_agent * max(args.steps + args.warmup, 1)))))
    w = np.ones(n_s, np.int32)
    for t in range(args.warmup):
        w = oracle.wealth_step(w, cfg["seed"], t)
    t0 = time.perf_counter()
    w, _, _, _ = oracle.wealth_run(w, cfg["seed"], args.warmup, args.steps)
    dt = time.perf_counter() - t0
    v = n_s * args.steps / dt
    model, ncpu = host_info()
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "C4 wealth transfer (BASELINE config 4)", "n_agents": cfg["n"],
                       "seed": cfg["seed"], "l2": C4_L2},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"wealth N={n_s} x {args.steps} steps per timed region "
                                       f"(of N={cfg['n']}); host {model}, {ncpu} cpus"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ traffic record
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")


def source_sha(files):
    """sha256 over the CUDA sources a kernel is built from: its .cu and every
    header it includes (transitively, `#include "..."` from csrc/ or include/)."""
    import hashlib
    import re
    csrc = os.path.join(ROOT, "paper_2601_16292_b200", "csrc")
    inc = os.path.join(ROOT, "include")
    seen, todo = set(), list(files)
    while todo:
        f = todo.pop()
        if f in seen:
            continue
        seen.add(f)
        path = os.path.join(csrc, f) if os.path.exists(os.path.join(csrc, f)) else os.path.join(inc, f)
        with open(path, encoding="utf-8", errors="replace") as fh:
            todo += re.findall(r'^\s*#\s*include\s+"([^"]+)"', fh.read(), re.M)
    h = hashlib.sha256()
    for f in sorted(seen):
        path = os.path.join(csrc, f) if os.path.exists(os.path.join(csrc, f)) else os.path.join(inc, f)
        with open(path, "rb") as fh:
            h.update(f.encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def traffic_record(kernel):
    """ncu DRAM bytes per launch of `kernel` from profiles/traffic.json (written by
    tools/traffic_record.py from one `ncu --set full` capture), with the commit it
    was taken at and whether the kernel's sources are unchanged since."""
    if not os.path.exists(TRAFFIC_FILE):
        return None, None
    rec = json.load(open(TRAFFIC_FILE)).get(kernel)
    if not rec:
        return None, None
    cur = source_sha(rec["sources"])
    return rec["dram_bytes_per_launch"], {"file": "profiles/traffic.json", "ncu_report": rec.get("report"),
                                          "commit": rec.get("commit"), "source_sha": rec.get("source_sha"),
                                          "source_matches_current": cur == rec.get("source_sha")}


# ------------------------------------------------------------ the other configs
def _timed(m, k, torch):
    """Device time of m.step(k) (one call), CUDA events on the model stream."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m.synchronize()
    e0.record(m.stream)
    m.step(k)
    e1.record(m.stream)
    m.synchronize()
    return e0.elapsed_time(e1)


def _oracle_rate(fn, units):
    t0 = time.perf_counter()
    fn()
    return units / (time.perf_counter() - t0)


def bench_configs(hbm):
    """BASELINE configs 1, 2, 3, 5 and the SURVEY 8(d) roofline variants V2, V3 on
    this GPU (unprofiled CUDA-event time of the config's steps) with the oracle
    timed beside each on this host (single thread; C5 also one process per core),
    the binding roof and the ncu summary it comes from.  One dict per config."""
    import numpy as np
    import torch

    import oracle
    from paper_2601_16292_b200 import Model, boids_params, sir_params, sweep, wealth_params
    from paper_2601_16292_b200 import workloads as W
    oracle.build()
    bkeys = ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")
    out = {}
    _, ncpu = host_info()

    # C1: wealth N = 1e3, 100 steps (one single-CTA launch for all steps)
    c = W.C1_WEALTH_SMALL
    m = Model("wealth", c["n"], wealth_params(), c["seed"])
    m.step(c["steps"])
    m.set_step(0)
    m.write_column("wealth", np.ones(c["n"], np.int32))
    ms = _timed(m, c["steps"], torch)
    ok = bool(np.array_equal(m.read_column("wealth"), oracle.wealth_run(np.ones(c["n"], np.int32), c["seed"], 0,
                                                                         c["steps"])[0]))
    m.close()
    orate = _oracle_rate(lambda: oracle.wealth_run(np.ones(c["n"], np.int32), c["seed"], 0, c["steps"]),
                         c["n"] * c["steps"])
    out["c1"] = {"workload": "C1 wealth N=1e3 x100 (BASELINE config 1)", "ms_per_step": ms / c["steps"],
                 "value": c["n"] * c["steps"] / (ms / 1e3), "unit": UNIT, "bit_exact_vs_oracle": ok,
                 "roof": {"bound": "latency", "why": "1,000 agents: one CTA, one barrier per step",
                          "evidence": "DESIGN.md 5 (wealth_small_kernel)"},
                 "oracle": {"value": orate, "unit": UNIT, "cores": 1, "sample": "the whole config"}}

    # C2: SIR on G(1e5, 5e5), 200 steps (one persistent cooperative launch)
    c = W.C2_SIR
    sp = sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"])
    m = Model("sir", c["n"], sp, c["seed"])
    ms = _timed(m, c["steps"], torch)
    mm, kk = oracle.round_count(c["n"] * c["mean_degree"] / 2.0), oracle.round_count(c["init_frac"] * c["n"])
    rp, col, _ = oracle.er_graph(c["n"], mm, c["seed"])
    st0 = oracle.sir_init(c["n"], kk, c["seed"])
    t0 = time.perf_counter()
    ref, rcounts, _ = oracle.sir_run(rp, col, st0, c["seed"], c["beta"], c["gamma"], 0, c["steps"])
    orate = c["n"] * c["steps"] / (time.perf_counter() - t0)
    ok = bool(np.array_equal(m.read_column("state"), ref))
    ok = ok and bool(np.array_equal(m.metrics("I"), rcounts[:, 1]))
    m.close()
    # steps whose input has no infected agent are the identity: the persistent
    # launch records them without a pass (SIR step)
    ident = int((rcounts[:-1, 1] == 0).sum())
    out["c2"] = {"workload": "C2 SIR G(1e5, 5e5) x200 (BASELINE config 2)", "ms_per_step": ms / c["steps"],
                 "value": c["n"] * c["steps"] / (ms / 1e3), "unit": UNIT, "bit_exact_vs_oracle": ok,
                 "identity_steps": ident,
                 "note": f"{ident} of the {c['steps']} steps start with no infected agent (the epidemic is over): "
                         "the identity, recorded without a pass; value counts every step",
                 "roof": {"bound": "latency", "why": "4.6 MB, L2-resident; per-step grid barrier (1.2-1.6 us) + "
                          "the bitmap -> row -> probe chain",
                          "evidence": "profiles/r01_c2_sir_persistent_ncu.txt, profiles/r01_grid_sync_probe.txt"},
                 "oracle": {"value": orate, "unit": UNIT, "cores": 1, "sample": "the whole config (graph build "
                            "excluded, as on the GPU)"}}

    # C3: Boids N = 1e5, 100 steps
    c = W.C3_BOIDS
    bp = boids_params(*[c[k] for k in bkeys])
    m = Model("boids", c["n"], bp, c["seed"])
    m.step(1)
    ms = _timed(m, c["steps"] - 1, torch)
    per = ms / (c["steps"] - 1)
    roof3 = boids_roof(m, per, "C3")
    m.close()
    P = oracle.boids_params(**{k: c[k] for k in bkeys})
    s0 = oracle.boids_init(c["n"], c["L"], c["seed"])
    orate = _oracle_rate(lambda: oracle.boids_run(s0, P, 3), c["n"] * 3)
    out["c3"] = {"workload": "C3 Boids N=1e5 x100 (BASELINE config 3)", "ms_per_step": per,
                 "value": c["n"] / (per / 1e3), "unit": UNIT,
                 "roof": roof3,
                 "oracle": {"value": orate, "unit": UNIT, "cores": 1,
                            "sample": "first 3 steps on the full population (sparse phase)"}}

    # C5: 4,096 SIR replicates x 300 steps
    c = W.C5_SWEEP
    betas, seeds = W.sweep_replicates(c)
    sp0 = sir_params(c["mean_degree"], 0.0, c["gamma"], c["init_frac"])
    sweep(c["n"], sp0, betas[:64], seeds[:64], 5)  # warm (module load)
    res, st = sweep(c["n"], sp0, betas, seeds, c["steps"], with_stats=True)
    upd = c["n"] * c["steps"] * len(betas)
    pick = np.arange(0, len(betas), 256)
    want = oracle.sir_sweep(c["n"], c["mean_degree"], c["gamma"], c["init_frac"], betas[pick], seeds[pick],
                            c["steps"])
    t0 = time.perf_counter()
    oracle.sir_sweep(c["n"], c["mean_degree"], c["gamma"], c["init_frac"], betas[pick], seeds[pick], c["steps"])
    orate = c["n"] * c["steps"] * len(pick) / (time.perf_counter() - t0)
    import multiprocessing as mp
    jobs = [(c["n"], c["mean_degree"], c["gamma"], c["init_frac"], float(betas[k]), int(seeds[k]), c["steps"])
            for k in np.arange(0, len(betas), 32)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(ncpu) as pool:
        pool.map(_sweep_one, jobs, chunksize=1)
    orate_all = c["n"] * c["steps"] * len(jobs) / (time.perf_counter() - t0)
    out["c5"] = {"workload": "C5 sweep 4096 x SIR N=1e4 x300 (BASELINE config 5)",
                 "ms_total": st["step_ms"], "ms_per_step": st["step_ms"] / c["steps"],
                 "value": upd / (st["step_ms"] / 1e3), "unit": UNIT + " (nominal: replicates x N x steps)",
                 "active_updates": st["active_updates"], "build_ms": st["build_ms"],
                 "sampled_replicates_bit_exact_vs_oracle": bool(np.array_equal(res[pick], want)),
                 "roof": {"bound": "issue", "why": "graphs and states resident in shared memory for all 300 steps; "
                          "HBM only for the one-time load", "evidence": "profiles/r02_sweep_ncu.txt"},
                 "oracle": {"value": orate, "unit": UNIT, "cores": 1,
                            "sample": f"{len(pick)} of {len(betas)} replicates spanning all betas"},
                 "oracle_all_cores": {"value": orate_all, "unit": UNIT, "cores": ncpu,
                                      "sample": f"{len(jobs)} replicates, one process per core"}}

    # V2: SIR on G(1e8, 5e8), 20 steps (SURVEY 8(d) added roofline variant)
    c = W.V2_SIR_SCALE
    sp = sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"])
    m = Model("sir", c["n"], sp, c["seed"])
    arcs = m.column_info("col_idx")[3]
    ms = _timed(m, c["steps"], torch)
    S, I = (m.metrics(x).astype(np.float64) for x in ("S", "I"))
    m.close()
    k0 = oracle.round_count(c["init_frac"] * c["n"])
    s_prev = np.concatenate([[c["n"] - k0], S[:-1]])
    i_prev = np.concatenate([[k0], I[:-1]])
    alg = 2.0 * c["n"] * c["steps"] + float((np.minimum(s_prev, i_prev) * (8.0 + 5.0 * arcs / c["n"])).sum())
    ach = alg / (ms / 1e3) / 1e9
    # the binding roof: one random L2 probe per traversed arc.  Traversed arcs
    # per step estimated from the previous step's counts and the kernel's
    # direction rule at 8 agents per lane (push iff 10 I < 9 S: the I agents'
    # rows, else the S agents'), ignoring the pull's early exits (so the floor
    # is an upper estimate of the probe work); rate = random 4-byte loads from
    # an L2-resident array (tools/scatter_probe.cu, profiles/r01_scatter_probe.txt)
    kbar = arcs / c["n"]
    walked = np.where(10.0 * i_prev < 9.0 * s_prev, i_prev, s_prev) * kbar
    probe_rate = 2.776e11
    floor_ms = float(walked.sum()) / probe_rate * 1e3
    n_o = 1_000_000
    rp, col, _ = oracle.er_graph(n_o, oracle.round_count(n_o * c["mean_degree"] / 2.0), c["seed"])
    st0 = oracle.sir_init(n_o, oracle.round_count(c["init_frac"] * n_o), c["seed"])
    orate = _oracle_rate(lambda: oracle.sir_run(rp, col, st0, c["seed"], c["beta"], c["gamma"], 0, c["steps"]),
                         n_o * c["steps"])
    out["v2"] = {"workload": "V2 SIR G(1e8, 5e8) x20 (SURVEY 8(d) roofline variant)",
                 "ms_per_step": ms / c["steps"], "value": c["n"] * c["steps"] / (ms / 1e3), "unit": UNIT,
                 "roof": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                          "alg_rule": "2 B/agent + (8 + 5 kbar) B per agent of the smaller of S, I",
                          "binding": "random L2 neighbour-bitmap probes, one per traversed arc",
                          "evidence": "profiles/r02_v2_sir_ncu.txt, profiles/r02_v2_push_step_ncu.txt, profiles/r02_v2_steps.json"},
                 "probe_roof": {"bound": "l2_random_loads", "arcs_walked_per_step_est": float(walked.sum()) / c["steps"],
                                "peak_loads_per_s": probe_rate, "floor_ms_per_step": floor_ms / c["steps"],
                                "frac": floor_ms / ms if ms > 0 else None,
                                "peak_source": "tools/scatter_probe.cu ldg_rand (profiles/r01_scatter_probe.txt)",
                                "note": "arcs walked estimated from the per-step S/I counts and the direction rule"},
                 "oracle": {"value": orate, "unit": UNIT, "cores": 1,
                            "sample": f"the same model at N={n_o:.0e} (mean degree 10), 20 steps"}}

    # V3: Boids N = 1e8, L = 31,623 (density 0.1), 10 steps
    c = W.V3_BOIDS_SCALE
    m = Model("boids", c["n"], boids_params(*[c[k] for k in bkeys]), c["seed"])
    m.step(1)
    ms = _timed(m, c["steps"] - 1, torch)
    per = ms / (c["steps"] - 1)
    roofv3 = boids_roof(m, per, "V3")
    m.close()
    n_o = 1_000_000
    P = oracle.boids_params(**{**{k: c[k] for k in bkeys}, "L": 3162.3})
    s0 = oracle.boids_init(n_o, 3162.3, c["seed"])
    orate = _oracle_rate(lambda: oracle.boids_run(s0, P, 1), n_o)
    out["v3"] = {"workload": "V3 Boids N=1e8 L=31623 x10 (SURVEY 8(d) roofline variant)", "ms_per_step": per,
                 "value": c["n"] / (per / 1e3), "unit": UNIT, "roof": roofv3,
                 "oracle": {"value": orate, "unit": UNIT, "cores": 1,
                            "sample": f"N={n_o:.0e} at the same density (L=3162.3), first step"}}
    return out


def boids_roof(m, ms_per_step, which):
    """Boids binding roof: the stencil kernel's ALU/issue ceiling.  One more
    (profiled) step gives the stencil kernel's device time and the candidate
    visits of its pass (option stencil_candidates); achieved = visits / time,
    peak = the measured ceiling of the same instruction sequence."""
    qv = m.get_option("qv")
    m.profile(True)
    m.step(1)
    m.synchronize()
    prof = {k: t / n for k, n, t in m.profile_results()}
    m.profile(False)
    cand = m.get_option("stencil_candidates")
    st_ms = prof.get("boids_step", 0.0)
    # the profiled step is the one AFTER the timed ones: flocks cluster as the run
    # goes on, so it can cost more than the timed average; its share is taken
    # against its own kernels' total, not against ms_per_step
    prof_step_ms = sum(prof.values())
    ach = cand / (st_ms / 1e3) if st_ms > 0 else 0.0
    peak = STENCIL_CEILING[qv]
    return {"bound": "alu", "kernel": "boids_group_kernel", "achieved": ach, "peak": peak,
            "unit": "candidate-visits/s", "frac": ach / peak, "candidates_per_step": cand,
            "stencil_ms": st_ms, "profiled_step_kernels_ms": prof_step_ms,
            "stencil_share_of_step": st_ms / prof_step_ms if prof_step_ms > 0 else None,
            "profiled_step": "the step after the timed ones, each kernel timed by events (PDL off)",
            "kernel_ms": prof, "peak_source": "profiles/r02_alu_ceiling.txt (tools/alu_ceiling.cu, "
                                               f"{'pre-quantised' if qv else 'float'}-velocity stencil)",
            "why": "FP32 + int64 fixed-point stencil; memory latency hidden in the ceiling",
            "evidence": ("profiles/r02_v3_boids_group_final_ncu.txt" if which == "V3"
                         else "profiles/r02_c3_boids_group_ncu.txt")}


# ------------------------------------------------------------------ GPU arm
def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    return world, rank, local, pg


def barrier_sync(pg, torch):
    torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()


def max_over_ranks(pg, torch, v, device="cuda"):
    """Max of a host scalar over all ranks (the driver's timing rule)."""
    if pg is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def bench_wealth(args):
    import numpy as np
    import torch

    from paper_2601_16292_b200 import Model, nccl_unique_id, wealth_params
    from paper_2601_16292_b200.workloads import C4_WEALTH_SCALE as cfg

    world, rank, local, pg = dist_setup(args)
    uid = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(obj, src=0)
        uid = obj[0]
    n = cfg["n"]
    m = Model("wealth", n, wealth_params(w0=cfg["w0"], amount=cfg["amount"],
                                         exclude_self=cfg["exclude_self"],
                                         counter_bits=args.counter_bits), cfg["seed"],
              device=local, rank=rank, world=world, unique_id=uid)
    _, _, off, n_loc = m.column_info("wealth")
    stream = m.stream
    clocks = ClockSampler(local)
    clocks.start()  # sampled over the whole GPU arm, so the record is never empty
    for _ in range(args.warmup):
        m.step(1)
    m.synchronize()
    # PAPER.md l.213 protocol: repetitions of the K-step region, the first 2
    # discarded as warm-up, the median of the next 5 reported; each repetition
    # is K steps between a barrier + synchronize on both sides, device time by
    # CUDA events on the model stream, max over ranks
    reps_ms, prof, act_hist = [], [], []
    for rep in range(args.warmup_reps + args.reps):
        timed = rep >= args.warmup_reps
        if timed:
            m.reset_metrics()
            m.profile(True)
        barrier_sync(pg, torch)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            m.step(1)
        ev1.record(stream)
        m.synchronize()
        barrier_sync(pg, torch)
        if timed:
            reps_ms.append(max_over_ranks(pg, torch, ev0.elapsed_time(ev1)))
            prof.append(m.profile_results())
            m.profile(False)
            tot = m.metrics("total_wealth")
            assert (tot == n * cfg["w0"]).all(), "wealth not conserved"
            act_hist.append(m.metrics("active"))
    med = sorted(range(args.reps), key=lambda k: reps_ms[k])[args.reps // 2]
    ms, prof = reps_ms[med], prof[med]
    # scatter REDs issued in the median repetition = senders of each of its steps =
    # agents with w >= amount in the state the step starts from (the previous
    # step's `active`; the first step's from the last step of the repetition before)
    prev_last = int(act_hist[med - 1][-1]) if med > 0 else None
    act = act_hist[med]
    reds = float(act[:-1].sum()) + float(prev_last if prev_last is not None else act[0])
    launches = sum(c for _, c, _ in prof)
    dom = max(prof, key=lambda r: r[2]) if prof else ("", 0, 0.0)
    dom_avg_ms = dom[2] / max(dom[1], 1)
    value = n * args.steps / (ms / 1e3)

    # ---- end to end through the public API with host buffers -------------
    # timed: H2D of the initial column from pinned host memory, K steps each
    # followed by a D2H read of that step's observables, D2H of the final column
    host_w = torch.full((n_loc,), cfg["w0"], dtype=torch.int32).pin_memory()
    host_out = torch.empty((n_loc,), dtype=torch.int32).pin_memory()
    m.set_step(0)
    barrier_sync(pg, torch)
    t0 = time.perf_counter()
    m.write_column("wealth", host_w.numpy())
    m.reset_metrics()
    e2e_active = []
    for _ in range(args.steps):
        m.step(1)
        e2e_active.append(int(m.metrics("active")[-1]))  # this step's observable, read on the host
        m.reset_metrics()
    m.read_column("wealth", host_out.numpy())
    barrier_sync(pg, torch)
    e2e_s = max_over_ranks(pg, torch, time.perf_counter() - t0)
    # per step: the 40-byte step record (overflow check + the metric read share one copy)
    e2e = {"value": n * args.steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(n_loc * 4 / args.steps),
           "d2h_bytes_per_step": int(n_loc * 4 / args.steps + 40),
           "note": f"one {n_loc * 4 / 1e6:.0f} MB H2D of the initial column and one D2H of the final column "
                   f"per run, amortised over the run's K={args.steps} steps (the e2e rate therefore grows "
                   f"with K), plus a 40-byte host read of each step's observables"}

    hbm, kind = peaks()
    # algorithmic bytes of the method per step: the
    # column read + written once (8 B/agent) plus one 4-byte increment read and
    # written per transfer (8 B/transfer; transfers = senders, from `active`)
    transfers = reds / args.steps
    alg_bytes = 8.0 * n_loc + 8.0 * transfers
    achieved = alg_bytes / (dom_avg_ms / 1e3) / 1e9 if dom_avg_ms > 0 else 0.0
    traffic, traffic_src = traffic_record(dom[0])
    if rank == 0:
        model, ncpu = host_info()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded Philox population, BASELINE config 4)",
            # config: the workload only (the reference arm prints the same dict);
            # how this arm runs it is in parallelism / counter_bits
            "config": {"workload": "C4 wealth transfer (BASELINE config 4)", "n_agents": n,
                       "seed": cfg["seed"], "l2": C4_L2},
            "parallelism": f"id-sharded x{world}", "counter_bits": m.get_option("counter_bits"),
            "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": hbm,
                         "peak_kind": kind, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "alg_bytes_per_launch": alg_bytes,
                         "alg_bytes_rule": "8 B/agent + 8 B/transfer",
                         "transfers_per_step": transfers,
                         "avg_launch_ms": dom_avg_ms,
                         "share_of_step": dom[2] / ms if ms > 0 else None},
            "scatter": "packed-counter L2 atomics",
            "kernels": [{"name": a, "launches": b, "total_ms": c} for a, b, c in prof],
            "gpu_launches": launches,
            "timing": {"protocol": f"median of {args.reps} timed repetitions of K steps after "
                                   f"{args.warmup_reps} discarded repetitions (PAPER.md l.213) and W warm-up "
                                   f"steps; CUDA events on the model stream, max over ranks",
                       "reps_ms": reps_ms, "median_rep": med},
            "e2e": e2e,
            "clocks": None,
            "host": {"cpu": model, "cpus": ncpu},
        }
        line["stream_red_roof"] = {
            "bound": "l2_red+hbm", "kernel": dom[0], "achieved_ms": dom_avg_ms,
            "roof_ms": STREAM_RED_ROOF_MS * n_loc / 1e8, "frac": STREAM_RED_ROOF_MS * n_loc / 1e8 / dom_avg_ms
            if dom_avg_ms > 0 else None,
            "roof_source": "tools/red_stream_ceiling.cu (profiles/r02_red_stream_ceiling.txt): 800 MB column "
                           "stream + 0.587 N random REDs into packed 4-bit counters in one kernel, hash instead "
                           "of Philox, no apply -- the floor of any one-RED-per-transfer step"}
        if True:  # packed counters: one L2 RED per transfer
            line["l2_atomic_roof"] = {
                "bound": "l2_atomics", "kernel": dom[0],
                "achieved_reds_per_s": reds / (ms / 1e3) if ms > 0 else None,
                "peak_reds_per_s": RED_CEILING, "peak_kind": "measured (tools/red_ceiling.cu, "
                "profiles/r01_red_ceiling.txt)",
                "frac": (reds / (ms / 1e3)) / RED_CEILING if ms > 0 else None,
                "reds_per_step": reds / args.steps}
        m.close()
        if world == 1 and not args.no_configs:
            line["configs"] = bench_configs(hbm)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_wealth(n, cfg["seed"])
        line["clocks"] = clocks.stop()
        print(json.dumps(line), flush=True)
    else:
        m.close()
        clocks.stop()
    if pg is not None:
        pg.destroy_process_group()
    return 0


def bench_small(args):
    """Extra single-GPU measurements of the other configs (not the driver line)."""
    import numpy as np
    import torch

    from paper_2601_16292_b200 import Model, boids_params, sir_params, sweep, walk_params, wealth_params
    from paper_2601_16292_b200 import workloads as W

    out = {}
    w = args.workload
    if w in ("walk", "walk_scale"):
        c = W.CONFIGS[w]
        m = Model("walk", c["n"], walk_params(c["L"], c["vmax"]), c["seed"])
        k = c["steps"]
        m.step(2)
        m.synchronize()
        m.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(m.stream)
        m.step(k)
        e1.record(m.stream)
        m.synchronize()
        ms = e0.elapsed_time(e1)
        prof = m.profile_results()
        avg = prof[0][2] / prof[0][1]
        hbm, kind = peaks()
        ach = 24.0 * c["n"] / (avg / 1e3) / 1e9
        print(json.dumps({"workload": w, "n": c["n"], "steps": k, "ms_per_step": ms / k,
                          "value": c["n"] * k / (ms / 1e3), "unit": UNIT,
                          "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                                       "frac": ach / hbm, "alg_bytes_per_agent": 24},
                          "kernels": prof}))
        return 0
    if w == "listing1":
        # PAPER.md Listing 1 at N = 1e8: population.update("wealth", col("wealth") + 10)
        from paper_2601_16292_b200.population import Population, col
        n = 100_000_000
        p = Population({"wealth": "i32"}, capacity=n)
        p.add_agents(n, wealth=1)
        p.update("wealth", col("wealth") + 10)
        p.synchronize()
        k = 50
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(p.stream)
        for _ in range(k):
            p.update("wealth", col("wealth") + 10, count=False)  # asynchronous
        e1.record(p.stream)
        p.synchronize()
        dt = e0.elapsed_time(e1) / k / 1e3
        k += 0
        hbm, kind = peaks()
        ach = 9.0 * n / dt / 1e9  # alive mask 1 B + column read 4 B + write 4 B per row
        assert p.aggregate("sum", col("wealth")) == n * (1 + 10 * (k + 1))
        print(json.dumps({"workload": "listing1", "n": n, "ms_per_update": dt * 1e3,
                          "value": n / dt, "unit": "rows/s",
                          "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                                       "frac": ach / hbm, "alg_bytes_per_row": 9,
                                       "note": "CUDA events over 50 asynchronous update calls"}}))
        return 0
    if w == "population":
        # NEXT-4 general columnar updates (not the Listing-1 fast path): programs are
        # compiled at run time into straight-line kernels (or interpreted, AMBER_POP_JIT=0)
        from paper_2601_16292_b200.population import Population, col, rand
        n = 100_000_000
        hbm, kind = peaks()
        cases = [("wealth = max(wealth-1, 0) + 2*state where state == 0",
                  (col("wealth") - 1).max(0) + col("state") * 2, col("state") == 0, 10.0,
                  "alive 1 + state 1 + wealth 4 read + 4 written"),
                 ("wealth = max(wealth-1, 0) + (rand < 0.5) where state == 0",
                  (col("wealth") - 1).max(0) + (rand(7) < 0.5), col("state") == 0, 18.0,
                  "alive 1 + state 1 + agent id 8 (keys the draw) + wealth 4 read + 4 written")]
        res = []
        for name, e, wh, bpr, rule in cases:
            p = Population({"wealth": "i32", "state": "u8"}, capacity=n)
            p.add_agents(n, wealth=3, state=0)
            p.update("wealth", e, where=wh)
            p.synchronize()
            k = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(p.stream)
            for _ in range(k):
                p.update("wealth", e, where=wh, count=False)
            e1.record(p.stream)
            p.synchronize()
            dt = e0.elapsed_time(e1) / k / 1e3
            ach = bpr * n / dt / 1e9
            res.append({"program": name, "ms_per_update": dt * 1e3, "rows_per_s": n / dt,
                        "paths_jit_interp": p.update_paths(),
                        "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                                     "alg_bytes_per_row": bpr, "rule": rule}})
            p.close()
        print(json.dumps({"workload": "population", "n": n, "cases": res}))
        return 0
    if w in ("sirs", "sirs_scale"):
        c = W.CONFIGS[w]
        from paper_2601_16292_b200 import sir_space_params
        def make():
            return Model("sir_space", c["n"], sir_space_params(c["L"], c["r"], c["p_infect"], c["p_recover"],
                                                               c["init_frac"]), c["seed"])
        k = c["steps"]
    elif w == "c1":
        c = W.C1_WEALTH_SMALL

        def make():
            return Model("wealth", c["n"], wealth_params(), c["seed"])
        k = c["steps"]
    elif w == "c2":
        c = W.C2_SIR

        def make():
            return Model("sir", c["n"], sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"]),
                         c["seed"])
        k = c["steps"]
    elif w == "c3":
        c = W.C3_BOIDS

        def make():
            return Model("boids", c["n"], boids_params(*[c[x] for x in ("L", "R", "rs", "wc", "wa", "ws",
                                                                          "vmax", "dt")]), c["seed"])
        k = c["steps"]
    elif w == "c5":
        c = W.C5_SWEEP
        betas, seeds = W.sweep_replicates(c)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res, st = sweep(c["n"], sir_params(c["mean_degree"], 0.0, c["gamma"], c["init_frac"]), betas,
                        seeds, c["steps"], with_stats=True)
        wall = time.perf_counter() - t0
        upd = c["n"] * c["steps"] * len(betas)
        print(json.dumps({"workload": "c5", "agent_updates": upd, "step_ms": st["step_ms"],
                          "build_ms": st["build_ms"], "wall_s": wall,
                          "value": upd / (st["step_ms"] / 1e3), "unit": UNIT,
                          "active_updates": st["active_updates"]}))
        return 0
    else:
        raise SystemExit(f"unknown workload {w}")
    m = make()
    m.step(1)
    m.synchronize()
    # the timed run is unprofiled (per-kernel events between the launches of a
    # multi-kernel step would be counted as step time); the per-kernel split
    # comes from a second, profiled run of the same steps on a fresh model
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    m.step(k)
    e1.record(m.stream)
    m.synchronize()
    ms = e0.elapsed_time(e1)
    m2 = make()
    m2.step(1)
    m2.profile(True)
    m2.step(k)
    m2.synchronize()
    print(json.dumps({"workload": w, "n": c["n"], "steps": k, "ms": ms, "ms_per_step": ms / k,
                      "value": c["n"] * k / (ms / 1e3), "unit": UNIT,
                      "kernels_profiled_run": m2.profile_results()}))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="amber", choices=["amber", "reference"])
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the other configs' entries (C1-C3, C5, V2, V3)")
    ap.add_argument("--reps", type=int, default=5, help="timed repetitions of the K-step region (median)")
    ap.add_argument("--warmup-reps", type=int, default=2, help="discarded repetitions before the timed ones")
    ap.add_argument("--counter-bits", type=int, default=0,
                    help="wealth scatter (amber_wealth_params.counter_bits); 0 = library default")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.workload != "c4":
        return bench_small(args)
    return bench_wealth(args)


if __name__ == "__main__":
    sys.exit(main())
