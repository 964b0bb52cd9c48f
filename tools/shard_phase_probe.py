#!/usr/bin/env python
"""Per-phase device times of a sharded step (C4 wealth; V2 SIR or V3 Boids with
a third argument "sir" / "boids") at G virtual ranks on ONE B200 (loopback transport: each rank's kernels run on this GPU, its own
host thread, host barriers between phases -- no kernel waits on another).

Run it under the ncu launch list so every kernel is timed alone (serialised),
which is what each rank's kernel costs on its own GPU:

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/shard_launches.csv python tools/shard_phase_probe.py 8

Without ncu it prints the loopback wall time per step (all ranks' kernels
sharing one GPU).  python tools/shard_phase_probe.py [G] [steps] [wealth|sir|boids]"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_16292_b200 import Model, boids_params, loopback_id, sir_params, wealth_params  # noqa: E402
from paper_2601_16292_b200 import workloads as W  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
kind = sys.argv[3] if len(sys.argv) > 3 else "wealth"
C = dict({"wealth": W.C4_WEALTH_SCALE, "sir": W.V2_SIR_SCALE, "boids": W.V3_BOIDS_SCALE}[kind])
if os.environ.get("PROBE_N"):  # smaller population at the same density (G copies of the sharded buffers share one GPU)
    n2 = int(float(os.environ["PROBE_N"]))
    if "L" in C:
        C["L"] = float(C["L"] * (n2 / C["n"]) ** 0.5)
    C["n"] = n2
P = {"wealth": lambda: wealth_params(),
     "sir": lambda: sir_params(C["mean_degree"], C["beta"], C["gamma"], C["init_frac"]),
     "boids": lambda: boids_params(*[C[k] for k in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")])}[kind]()


def par(ms, fn):
    err = []

    def run(m):
        try:
            fn(m)
        except Exception as e:  # pragma: no cover
            err.append(e)

    th = [threading.Thread(target=run, args=(m,)) for m in ms]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]


uid = loopback_id()
ms = [Model(kind, C["n"], P, C["seed"], rank=r, world=world, unique_id=uid) for r in range(world)]
if kind == "sir" and os.environ.get("PROBE_DIR"):  # SIR direction: 0 auto, 1 pull, 2 push
    for m in ms:
        m.set_option("direction", int(os.environ["PROBE_DIR"]))
par(ms, lambda m: (m.step(3), m.synchronize()))
t0 = time.perf_counter()
par(ms, lambda m: (m.step(steps), m.synchronize()))
dt = time.perf_counter() - t0
tots = [None] * world
name = {"wealth": "total_wealth", "sir": "I", "boids": "mean_speed"}[kind]
par(ms, lambda m: tots.__setitem__(ms.index(m), m.metrics(name)[-1]))
print(f"{kind} G={world} loopback on one GPU: {dt / steps * 1e3:.3f} ms/step wall (all ranks sharing the GPU); "
      f"last {name} {tots[0]}", flush=True)
par(ms, lambda m: m.close())
