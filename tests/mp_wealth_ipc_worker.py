"""Worker of tests/test_gpu_ipc.py (launched by torch.distributed.run, two
processes on ONE GPU): the sharded wealth model with its peer-memory (P2P)
exchange carried by host collectives over gloo -- CUDA IPC handles of the
bucket blocks all-gathered between the two processes, each step's receive
kernel reading the other process's buckets through the IPC mapping after a
host barrier (no kernel waits on another).  Rank 0 compares the gathered
column and the all-reduced metrics with the oracle and writes the verdict."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_16292_b200 import Model, wealth_params  # noqa: E402


def main():
    out_path, n, seed, steps, bits = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    m = Model("wealth", n, wealth_params(counter_bits=bits), seed, device=0, rank=rank, world=world,
              host_group=dist.group.WORLD)
    m.set_option("digest", 1)
    m.step(1)
    m.step(steps - 1)
    mode = m.get_option("exchange")
    replays = m.get_option("replays")
    _, _, lo, ln = m.column_info("wealth")
    w = torch.from_numpy(m.read_column("wealth").astype(np.int32))
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([ln], dtype=torch.int64))
    mx = max(int(s.item()) for s in sizes)  # gloo all_gather needs equal sizes: pad
    parts = [torch.zeros(mx, dtype=torch.int32) for _ in sizes]
    dist.all_gather(parts, torch.cat([w, torch.zeros(mx - ln, dtype=torch.int32)]))
    parts = [p_[:int(s.item())] for p_, s in zip(parts, sizes)]
    tot, act, dig = m.metrics("total_wealth"), m.metrics("active"), m.metrics("digest")
    m.close()
    if rank == 0:
        import oracle
        full = torch.cat(parts).numpy()
        ref, rtot, ract, rdig = oracle.wealth_run(np.ones(n, np.int32), seed, 0, steps, digests=True)
        res = {"exchange": int(mode), "replays": int(replays), "column_equal": bool(np.array_equal(full, ref)),
               "total_equal": bool(np.array_equal(tot, rtot)), "active_equal": bool(np.array_equal(act, ract)),
               "digest_equal": bool(np.array_equal(dig, rdig.astype(np.uint64)))}
        json.dump(res, open(out_path, "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
