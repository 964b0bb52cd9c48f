#!/usr/bin/env python
"""Per-phase device times of the sharded C4 wealth step at G virtual ranks on
ONE B200 (loopback transport: each rank's kernels run on this GPU, its own
host thread, host barriers between phases -- no kernel waits on another).

Run it under the ncu launch list so every kernel is timed alone (serialised),
which is what each rank's kernel costs on its own GPU:

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/shard_launches.csv python tools/shard_phase_probe.py 8

Without ncu it prints the loopback wall time per step (all ranks' kernels
sharing one GPU).  python tools/shard_phase_probe.py [G] [steps]"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_16292_b200 import Model, loopback_id, wealth_params  # noqa: E402
from paper_2601_16292_b200.workloads import C4_WEALTH_SCALE as C  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10


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
ms = [Model("wealth", C["n"], wealth_params(), C["seed"], rank=r, world=world, unique_id=uid) for r in range(world)]
par(ms, lambda m: (m.step(3), m.synchronize()))
t0 = time.perf_counter()
par(ms, lambda m: (m.step(steps), m.synchronize()))
dt = time.perf_counter() - t0
tots = [None] * world
par(ms, lambda m: tots.__setitem__(ms.index(m), int(m.metrics("total_wealth")[-1])))
print(f"G={world} loopback on one GPU: {dt / steps * 1e3:.3f} ms/step wall (all ranks sharing the GPU); "
      f"total wealth {tots[0]} (expected {C['n']})", flush=True)
par(ms, lambda m: m.close())
