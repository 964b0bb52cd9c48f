"""Multi-process (world_size 2 and 4, gloo on CPU) checks of the N>1 host logic.

The GPU data path (NCCL exchange inside libamber.so) cannot run here; these
tests cover what the ranks must agree on before any kernel runs:
  * the partition rules the library exposes (amber_shard_range / amber_sweep_range)
    tile [0, N) / [0, R) exactly, with shard boundaries on 8-agent multiples
    (R4: two-agent Philox blocks never straddle ranks);
  * the NCCL unique-id rendezvous used by bench.py (rank 0 creates, all ranks
    receive the same 128 bytes through torch.distributed);
  * bench.py's max-over-ranks timing reduction;
  * the sharded wealth step: receivers bucketed by owner rank (owner = r / shard
    size, as in the kernel), exchanged with all_to_all, applied by the owner,
    equal the unsharded oracle step bit for bit;
  * the sharded SIR step (NEXT-3): 32-aligned id ranges (amber_sir_shard_range),
    local I-bitmap words all-gathered every step, each rank pulling its own rows
    against the global bitmap with globally keyed draws, equals the unsharded
    oracle run bit for bit;
  * the sharded Boids step (NEXT-3): x-slabs of whole cell columns, agents
    migrating to the slab of their cell column and the edge columns exchanged
    as halos; each rank steps its own agents from own + halo agents only, and
    the union equals the unsharded oracle run bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surface failures to the parent
        q.put((rank, f"ERROR {type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


def run_world(world, fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        assert not (isinstance(v, str) and v.startswith("ERROR")), v
    return [out[r] for r in range(world)]


def _partitions(rank, world):
    from paper_2601_16292_b200 import shard_range, sweep_range
    res = {}
    for n in (1, 7, 1000, 100_003, 100_000_000):
        lo, hi = shard_range(n, world, rank)
        t = torch.tensor([lo, hi], dtype=torch.int64)
        g = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(g, t)
        res[n] = [tuple(x.tolist()) for x in g]
    for R in (0, 5, 4096):
        r0, r1 = sweep_range(R, world, rank)
        t = torch.tensor([r0, r1], dtype=torch.int64)
        g = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(g, t)
        res[("sweep", R)] = [tuple(x.tolist()) for x in g]
    return res


def _uid(rank, world):
    from paper_2601_16292_b200 import nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def _maxtime(rank, world):
    import bench
    return bench.max_over_ranks(dist, torch, float(rank + 1) * 1.5, device="cpu")


def _sharded_wealth(rank, world):
    import oracle
    from paper_2601_16292_b200 import shard_range
    n, seed, steps = 1003, 17, 6
    lo, hi = shard_range(n, world, rank)
    shard = ((-(-n // world) + 7) // 8) * 8
    w = np.ones(n, np.int32)[lo:hi].copy()
    for t in range(steps):
        send = [[] for _ in range(world)]
        inc = np.zeros(hi - lo, np.int64)
        for k, i in enumerate(range(lo, hi)):
            if w[k] >= 1:
                r = oracle.wealth_receiver(seed, n, i, t)
                d = min(r // shard, world - 1)
                if d == rank:
                    inc[r - lo] += 1
                else:
                    send[d].append(r)
        counts = torch.tensor([len(s) for s in send], dtype=torch.int64)
        rc = torch.zeros(world, dtype=torch.int64)
        dist.all_to_all_single(rc, counts)
        out = torch.tensor(sum(send, []), dtype=torch.int64)
        inp = torch.zeros(int(rc.sum()), dtype=torch.int64)
        dist.all_to_all_single(inp, out, rc.tolist(), counts.tolist())
        for r in inp.tolist():
            inc[r - lo] += 1
        w = (w - (w >= 1) + inc).astype(np.int32)
    g = [None] * world
    dist.all_gather_object(g, (lo, w.tolist()))
    return g


def _sharded_wealth_dense(rank, world):
    # the dense exchange (r02 default up to 8 ranks): every rank counts ALL its
    # transfers in a global per-agent array; each owner sums the ranks' arrays
    # over its shard (here an all-reduce, then the own slice) and applies them;
    # the overflow check compares the global totals of issued and decoded counts
    import oracle
    from paper_2601_16292_b200 import shard_range
    n, seed, steps = 1003, 17, 6
    lo, hi = shard_range(n, world, rank)
    shard = ((-(-n // world) + 7) // 8) * 8
    w = np.ones(n, np.int32)[lo:hi].copy()
    for t in range(steps):
        glob = np.zeros(world * shard, np.int64)
        for k, i in enumerate(range(lo, hi)):
            if w[k] >= 1:
                glob[oracle.wealth_receiver(seed, n, i, t)] += 1
        sent = int(glob.sum())
        g = torch.tensor(glob)
        dist.all_reduce(g)
        inc = g.numpy()[lo:hi]
        tot = torch.tensor([sent, int(inc.sum())], dtype=torch.int64)
        dist.all_reduce(tot)
        assert int(tot[0]) == int(tot[1])
        w = (w - (w >= 1) + inc).astype(np.int32)
    out = [None] * world
    dist.all_gather_object(out, (lo, w.tolist()))
    return out


def _sharded_sir(rank, world):
    import oracle
    from paper_2601_16292_b200 import sir_shard_range
    n, kbar, seed, beta, gamma, steps = 2003, 6.0, 5, 0.3, 0.2, 12
    rp, col, _ = oracle.er_graph(n, int(round(n * kbar / 2)), seed)
    st0 = oracle.sir_init(n, 20, seed)
    lo, hi = sir_shard_range(n, world, rank)
    shard = ((-(-n // world) + 31) // 32) * 32
    assert lo == min(rank * shard, n) and lo % 32 == 0
    x = st0[lo:hi].copy()
    T_b, T_g = oracle.bernoulli_threshold(beta), oracle.bernoulli_threshold(gamma)
    for t in range(steps):
        # local I-bitmap words (bit b of word w = agent 32w + b of the shard), all-gathered
        bits = np.zeros(shard, np.uint8)
        bits[:hi - lo] = x == 1
        words = torch.tensor(np.packbits(bits, bitorder="little").view(np.uint32).astype(np.int64))
        g = [torch.zeros_like(words) for _ in range(world)]
        dist.all_gather(g, words)
        glob = np.concatenate([w.numpy().astype(np.uint32) for w in g])
        is_i = lambda j: (glob[j >> 5] >> (j & 31)) & 1
        y = x.copy()
        for k in range(hi - lo):
            s = lo + k
            if x[k] == 0:  # pull: any I neighbour with a transmitting pair draw (S2, S3)
                for j in col[rp[s]:rp[s + 1]]:
                    if is_i(int(j)) and oracle.sir_tx_word(seed, min(s, j), max(s, j), t) < T_b:
                        y[k] = 1
                        break
            elif x[k] == 1 and oracle.lane32(seed, 0x11, s, t) < T_g:
                y[k] = 2
        x = y
    out = [None] * world
    dist.all_gather_object(out, (lo, x.tolist()))
    ref = oracle.sir_run(rp, col, st0, seed, beta, gamma, 0, steps)[0]
    return out, ref.tolist()


def _sharded_sir_push(rank, world):
    # the sharded PUSH step (r02): own infected agents walk their rows against the
    # all-gathered S bitmap, set bits of a global-size hit bitmap; block p of it
    # goes to rank p (all_to_all), the owner ORs the blocks and finalises
    import oracle
    from paper_2601_16292_b200 import sir_shard_range
    n, kbar, seed, beta, gamma, steps = 2003, 6.0, 5, 0.3, 0.2, 12
    rp, col, _ = oracle.er_graph(n, int(round(n * kbar / 2)), seed)
    st0 = oracle.sir_init(n, 20, seed)
    lo, hi = sir_shard_range(n, world, rank)
    shard = ((-(-n // world) + 31) // 32) * 32
    x = st0[lo:hi].copy()
    T_b, T_g = oracle.bernoulli_threshold(beta), oracle.bernoulli_threshold(gamma)

    def gather(mask):
        bits = np.zeros(shard, np.uint8)
        bits[:hi - lo] = mask
        words = torch.tensor(np.packbits(bits, bitorder="little").view(np.uint32).astype(np.int64))
        g = [torch.zeros_like(words) for _ in range(world)]
        dist.all_gather(g, words)
        return np.concatenate([w.numpy().astype(np.uint32) for w in g])

    for t in range(steps):
        sg = gather(x == 0)
        is_s = lambda j: (sg[j >> 5] >> (j & 31)) & 1
        hit = np.zeros(world * shard, np.uint8)  # this rank's global hit bitmap (one byte per bit here)
        for k in range(hi - lo):
            i = lo + k
            if x[k] != 1:
                continue
            for j in col[rp[i]:rp[i + 1]]:
                j = int(j)
                if is_s(j) and oracle.sir_tx_word(seed, min(i, j), max(i, j), t) < T_b:
                    hit[j] = 1
        # block p of every rank's hit bitmap to rank p (gloo has no all_to_all: an
        # all-gather of the whole bitmaps, each rank keeping the blocks for it)
        allh = [torch.zeros(world * shard, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allh, torch.tensor(hit.astype(np.int64)))
        mine = np.zeros(shard, np.uint8)
        for r in allh:
            mine |= r.numpy()[rank * shard:(rank + 1) * shard].astype(np.uint8)
        y = x.copy()
        for k in range(hi - lo):
            if x[k] == 0 and mine[k]:
                y[k] = 1
            elif x[k] == 1 and oracle.lane32(seed, 0x11, lo + k, t) < T_g:
                y[k] = 2
        x = y
    out = [None] * world
    dist.all_gather_object(out, (lo, x.tolist()))
    ref = oracle.sir_run(rp, col, st0, seed, beta, gamma, 0, steps)[0]
    return out, ref.tolist()


def _sharded_boids(rank, world):
    import oracle
    L, R, n, seed, steps = 120.0, 10.0, 800, 4, 8
    P = oracle.boids_params(L=L, R=R)
    nc = int(np.floor(L / (R * 1.001)))
    inv_cs = np.float32(nc / L)
    col0 = [q * nc // world for q in range(world + 1)]
    c_lo, c_hi = col0[rank], col0[rank + 1]

    def col_of(x):  # the kernels' cell_coord: float32 product, truncated, clamped
        return np.clip((np.asarray(x, np.float32) * inv_cs).astype(np.int64), 0, nc - 1)

    def owner(x):
        return np.searchsorted(np.array(col0[1:]), col_of(x), side="right")

    full = [np.asarray(a, np.float32) for a in oracle.boids_init(n, L, seed)]
    ids = np.arange(n)
    own = ids[owner(full[0]) == rank]
    st = {int(i): tuple(float(a[i]) for a in full) for i in own}  # id -> (x, y, vx, vy) as float32 values
    for t in range(steps):
        # migration (to the slab of the cell column) and halos (edge columns), via all_gather
        mine = [(i, v) for i, v in st.items()]
        everyone = [None] * world
        dist.all_gather_object(everyone, mine)
        st = {i: v for part in everyone for i, v in part if owner(np.float32(v[0])) == rank}
        left_col, right_col = (c_lo - 1) % nc, c_hi % nc
        halo = {i: v for part in everyone for i, v in part
                if i not in st and col_of(np.float32(v[0])) in (left_col, right_col)}
        # step own agents from own + halo agents only (a smaller population in the same box)
        loc_ids = list(st) + list(halo)
        loc = [np.array([(st.get(i) or halo[i])[k] for i in loc_ids], np.float32) for k in range(4)]
        out = oracle.boids_step_sample(loc, P, np.arange(len(st)))
        st = {i: tuple(float(out[k][j]) for k in range(4)) for j, i in enumerate(loc_ids[:len(st)])}
    everyone = [None] * world
    dist.all_gather_object(everyone, list(st.items()))
    ref = oracle.boids_run(tuple(full), P, steps)[0]
    return everyone, [np.asarray(a, np.float32).tolist() for a in ref]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_boids_slab_halo_equals_oracle(world):
    parts, ref = run_world(world, _sharded_boids)[0]
    got = dict(kv for part in parts for kv in part)
    assert sorted(got) == list(range(len(ref[0])))
    for k in range(4):
        col = np.array([got[i][k] for i in range(len(ref[0]))], np.float32)
        assert np.array_equal(col.view(np.uint32), np.array(ref[k], np.float32).view(np.uint32))


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_sir_bitmap_allgather_equals_oracle(world):
    parts, ref = run_world(world, _sharded_sir)[0]
    x = np.concatenate([np.array(v, np.uint8) for _, v in sorted(parts)])
    assert np.array_equal(x, np.array(ref, np.uint8))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sir_push_hit_blocks_equal_oracle(world):
    parts, ref = run_world(world, _sharded_sir_push)[0]
    x = np.concatenate([np.array(v, np.uint8) for _, v in sorted(parts)])
    assert np.array_equal(x, np.array(ref, np.uint8))


@pytest.mark.parametrize("world", [2, 4])
def test_partitions_tile_exactly(world):
    res = run_world(world, _partitions)[0]
    for key, parts in res.items():
        total = key[1] if isinstance(key, tuple) else key
        cur = 0
        for lo, hi in parts:
            assert lo == min(cur, total) and lo <= hi
            if not isinstance(key, tuple) and hi < total:
                assert hi % 8 == 0
            cur = hi
        assert cur == total


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_unique_id_rendezvous(world):
    ids = run_world(world, _uid)
    assert len(ids[0]) == 128 and all(x == ids[0] for x in ids)


def test_max_over_ranks():
    assert run_world(2, _maxtime) == [3.0, 3.0]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_wealth_dense_exchange_equals_oracle(world, orc):
    parts = run_world(world, _sharded_wealth_dense)[0]
    w = np.concatenate([np.array(v, np.int32) for _, v in sorted(parts)])
    ref = orc.wealth_run(np.ones(1003, np.int32), 17, 0, 6)[0]
    assert np.array_equal(w, ref)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_wealth_step_equals_oracle(world, orc):
    parts = run_world(world, _sharded_wealth)[0]
    w = np.concatenate([np.array(x, np.int32) for _, x in sorted(parts)])
    ref = orc.wealth_run(np.ones(1003, np.int32), 17, 0, 6)[0]
    assert np.array_equal(w, ref)


def _host_collectives(rank, world):
    # the binding's amber_runtime.host_allgather / host_barrier callbacks over a
    # gloo group, called through their C function pointers exactly as the
    # library calls them (send / recv raw addresses, bytes per rank)
    import ctypes as C

    from paper_2601_16292_b200.model import HostCollectives
    hc = HostCollectives(dist.group.WORLD)
    out = []
    for nbytes in (4, 64, 1000):
        send = (C.c_uint8 * nbytes)(*[(rank * 31 + k) % 256 for k in range(nbytes)])
        recv = (C.c_uint8 * (nbytes * world))()
        rc = hc.allgather(C.addressof(send), C.addressof(recv), nbytes, None)
        out.append((rc, bytes(recv)))
    out.append((hc.barrier(None), b""))
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_host_collectives_marshalling(world):
    res = run_world(world, _host_collectives)
    for rank_out in res:
        for (rc, got), nbytes in zip(rank_out[:3], (4, 64, 1000)):
            assert rc == 0
            want = b"".join(bytes((r * 31 + k) % 256 for k in range(nbytes)) for r in range(world))
            assert got == want
        assert rank_out[3][0] == 0
