#!/usr/bin/env python
"""Measure every BASELINE config on one B200 through the public API, with the
CPU oracle timed beside it by bench.py's reference arm (`bench.py --impl
reference --workload cX`: single thread, bounded samples; this script never
imports oracle/), and write one JSON object per config to stdout (collected
into profiles/rNN_all_configs.jsonl).

GPU timing: CUDA events on the model stream around amber_step(K) after a
warm-up call; per-kernel device time from the library's event profiler.
"""
import json
import os
import sys

# load every kernel at context creation: lazy module loading inside a timed
# region would be counted as step time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import subprocess  # noqa: E402
from paper_2601_16292_b200 import Model, boids_params, sir_params, sweep, wealth_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def timed(m, k):
    """Step time of k steps, unprofiled (per-kernel events between the launches
    of a multi-kernel step would count as step time), then the per-kernel split
    from the next k steps with the profiler on."""
    m.step(2)
    m.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    m.step(k)
    e1.record(m.stream)
    m.synchronize()
    ms = e0.elapsed_time(e1)
    m.profile(True)
    m.step(k)
    m.synchronize()
    prof = m.profile_results()
    m.profile(False)
    return ms, prof


def cpu_rate(workload):
    """The oracle's rate for a workload from bench.py's reference arm (one timed run)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", workload,
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, cwd=ROOT)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    return json.loads(line)["value"]


def main():
    out = []
    # C1
    c = W.C1_WEALTH_SMALL
    m = Model("wealth", c["n"], wealth_params(), c["seed"])
    ms, prof = timed(m, c["steps"])
    cpu = cpu_rate("c1")
    out.append(dict(config="C1 wealth N=1e3 x100", us_per_step=ms / c["steps"] * 1e3,
                    agent_updates_per_s=c["n"] * c["steps"] / ms * 1e3, kernels=prof,
                    bound="launch/latency (single-CTA, all steps one launch)", cpu_oracle_per_s=cpu))
    m.close()
    # C2
    c = W.C2_SIR
    m = Model("sir", c["n"], sir_params(c["mean_degree"], c["beta"], c["gamma"], c["init_frac"]), c["seed"])
    ms, prof = timed(m, c["steps"])
    cpu = cpu_rate("c2")
    out.append(dict(config="C2 SIR G(1e5,5e5) x200", us_per_step=ms / c["steps"] * 1e3,
                    agent_updates_per_s=c["n"] * c["steps"] / ms * 1e3, kernels=prof,
                    bound="latency (L2-resident 4.6 MB; grid barrier per step)", cpu_oracle_per_s=cpu))
    m.close()
    # C3
    c = W.C3_BOIDS
    bp = boids_params(*[c[k] for k in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")])
    m = Model("boids", c["n"], bp, c["seed"])
    ms, prof = timed(m, c["steps"])
    cpu = cpu_rate("c3")
    out.append(dict(config="C3 Boids N=1e5 x100", us_per_step=ms / c["steps"] * 1e3,
                    agent_updates_per_s=c["n"] * c["steps"] / ms * 1e3, kernels=prof,
                    bound="issue/latency (fp32+int64 stencil, L1-resident)",
                    cpu_oracle_per_s=cpu, cpu_sample="first 3 steps (sparse phase; later steps denser)"))
    m.close()
    # C4 (short run; the driver line is bench.py)
    c = W.C4_WEALTH_SCALE
    m = Model("wealth", c["n"], wealth_params(), c["seed"])
    ms, prof = timed(m, 200)
    dom = max(prof, key=lambda r: r[2])
    avg = dom[2] / dom[1]
    senders = float(m.metrics("active")[-201:-1].mean())  # transfers of each timed step
    out.append(dict(config="C4 wealth N=1e8 x200 (of 1000)", us_per_step=ms / 200 * 1e3,
                    agent_updates_per_s=c["n"] * 200 / ms * 1e3, kernels=prof,
                    hbm_frac=(8 * c["n"] + 8 * senders) / (avg / 1e3) / 1e9 / HBM,
                    alg_bytes_rule="8 B/agent + 8 B/transfer (SURVEY 8(d))",
                    bound="L2 atomics (random REDs, profiles/r01_red_ceiling.txt)"))
    m.close()
    # C5
    c = W.C5_SWEEP
    betas, seeds = W.sweep_replicates(c)
    res, stt = sweep(c["n"], sir_params(c["mean_degree"], 0.0, c["gamma"], c["init_frac"]), betas, seeds,
                     c["steps"], with_stats=True)
    cpu = cpu_rate("c5")
    out.append(dict(config="C5 sweep 4096 x N=1e4 x300", step_ms=stt["step_ms"], build_ms=stt["build_ms"],
                    agent_updates_per_s=stt["agent_updates"] / stt["step_ms"] * 1e3,
                    active_updates_per_s=stt["active_updates"] / stt["step_ms"] * 1e3,
                    bound="shared-memory latency (graphs smem-resident, early exit)",
                    cpu_oracle_per_s=cpu, cpu_sample="16 replicates spanning all betas (nominal updates)"))
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
