"""Pythonic wrapper over the C ABI (marshalling only; every step runs in libamber.so).

PyTorch supplies the plumbing: the CUDA stream the kernels are enqueued on,
the caching allocator that owns device memory (passed to the library as
allocator hooks), device tensors for zero-copy column reads, and
torch.distributed for broadcasting the NCCL unique id.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .capi import check

_NP = {capi.AMBER_I32: np.int32, capi.AMBER_U8: np.uint8, capi.AMBER_F32: np.float32,
       capi.AMBER_I64: np.int64, capi.AMBER_F64: np.float64, capi.AMBER_U64: np.uint64}
_METRIC_DT = {"total_wealth": np.int64, "active": np.int64, "digest": np.uint64, "S": np.int64,
              "I": np.int64, "R": np.int64, "mean_speed": np.float64, "polarisation": np.float64,
              "mean_displacement": np.float64}


class TorchAllocator:
    """Allocator hooks routing the library's device allocations through the
    PyTorch caching allocator (torch owns device memory)."""

    def __init__(self, device: int):
        import torch
        self.torch = torch
        self.device = device

        def _alloc(nbytes, stream, ctx):
            try:
                return int(torch.cuda.caching_allocator_alloc(int(nbytes), self.device,
                                                              int(stream or 0)))
            except Exception:  # OOM etc.: report NULL, the library raises AMBER_E_OOM
                return None

        def _free(ptr, nbytes, stream, ctx):
            try:
                if ptr:
                    torch.cuda.caching_allocator_delete(int(ptr))
            except Exception:  # interpreter shutdown: torch already torn down
                pass

        self.alloc = capi.ALLOC_FN(_alloc)
        self.free = capi.FREE_FN(_free)


class HostCollectives:
    """amber_runtime.host_allgather / host_barrier over a torch.distributed
    process group of any backend (e.g. gloo): the caller's own host transport
    for the sharded wealth model's peer-memory exchange (argument marshalling
    only; the exchange itself is the library's CUDA IPC mapping + kernels)."""

    def __init__(self, group=None):
        import numpy as np
        import torch
        import torch.distributed as dist
        self.world = dist.get_world_size(group)

        def _allgather(send, recv, nbytes, ctx):
            try:
                src = torch.from_numpy(np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(send)).copy())
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
                dist.all_gather(outs, src, group=group)
                buf = torch.cat(outs).numpy()  # keep alive across the copy
                C.memmove(recv, buf.ctypes.data, nbytes * self.world)
                return 0
            except Exception:  # reported by the library as AMBER_E_NCCL
                return 1

        def _barrier(ctx):
            try:
                dist.barrier(group=group)
                return 0
            except Exception:
                return 1

        self.allgather = capi.HOST_ALLGATHER_FN(_allgather)
        self.barrier = capi.HOST_BARRIER_FN(_barrier)


def make_runtime(device=0, stream=None, torch_alloc=True, rank=0, world=1, unique_id=None, host_group=None):
    """Build an amber_runtime; keeps ctypes callbacks/buffers alive on the struct.
    host_group: a torch.distributed process group whose host collectives carry the
    sharded wealth exchange instead of NCCL (unique_id must then be None)."""
    rt = capi.amber_runtime()
    rt.device = device
    keep = []
    if stream is None:
        # a dedicated torch stream (not the legacy NULL stream, which the C ABI
        # reads as "library-created stream"): callers time on model.stream
        import torch
        stream = torch.cuda.Stream(device)
    keep.append(stream)
    rt.stream = C.c_void_p(int(getattr(stream, "cuda_stream", stream)))
    if torch_alloc:
        ta = TorchAllocator(device)
        rt.alloc, rt.free = ta.alloc, ta.free
        keep.append(ta)
    rt.rank, rt.world = rank, world
    if host_group is not None:
        if unique_id is not None:
            raise ValueError("give either unique_id or host_group")
        hc = HostCollectives(host_group)
        rt.host_allgather, rt.host_barrier = hc.allgather, hc.barrier
        keep.append(hc)
    elif world > 1 or unique_id is not None:
        if unique_id is None or len(unique_id) < 128:
            raise ValueError("world > 1 needs the 128-byte NCCL unique id")
        buf = C.create_string_buffer(bytes(unique_id), 128)
        keep.append(buf)
        rt.nccl_unique_id = C.cast(buf, C.c_void_p)
    rt._keep = keep
    return rt


def shard_range(n_agents: int, world: int, rank: int):
    """amber_shard_range: this rank's agent range [lo, hi) (host logic, no GPU)."""
    lo, hi = C.c_int64(), C.c_int64()
    check(capi.lib().amber_shard_range(int(n_agents), int(world), int(rank), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def sir_shard_range(n_agents: int, world: int, rank: int):
    """amber_sir_shard_range: this rank's agents [lo, hi) in a sharded SIR model (host logic)."""
    lo, hi = C.c_int64(), C.c_int64()
    check(capi.lib().amber_sir_shard_range(int(n_agents), int(world), int(rank), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def sweep_range(n_reps: int, world: int, rank: int):
    """amber_sweep_range: the replicates [r0, r1) this rank runs (host logic, no GPU)."""
    r0, r1 = C.c_int64(), C.c_int64()
    check(capi.lib().amber_sweep_range(int(n_reps), int(world), int(rank), C.byref(r0), C.byref(r1)))
    return r0.value, r1.value


def loopback_id() -> bytes:
    """amber_loopback_id: id of an in-process loopback group (virtual shards on one GPU)."""
    buf = C.create_string_buffer(128)
    check(capi.lib().amber_loopback_id(buf, 128))
    return buf.raw


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(capi.lib().amber_nccl_unique_id(buf, 128))
    return buf.raw


class Model:
    """One agent population on one GPU (or one shard of it when world > 1)."""

    KINDS = {"wealth": capi.AMBER_WEALTH, "sir": capi.AMBER_SIR_GRAPH, "boids": capi.AMBER_BOIDS,
             "walk": capi.AMBER_WALK, "sir_space": capi.AMBER_SIR_SPACE}

    def __init__(self, kind: str, n_agents: int, params, seed: int, *, device=0, stream=None,
                 torch_alloc=True, rank=0, world=1, unique_id=None, host_group=None):
        self.kind = kind
        self.lib = capi.lib()
        self.rt = make_runtime(device, stream, torch_alloc, rank, world, unique_id, host_group)
        self.stream = self.rt._keep[0]  # torch.cuda.Stream (or the caller's stream handle)
        self.params = params
        h = C.c_void_p()
        check(self.lib.amber_model_create(self.KINDS[kind], int(n_agents), C.byref(params),
                                          C.sizeof(params), int(seed), C.byref(self.rt),
                                          C.byref(h)))
        self.h = h
        self.n_agents = int(n_agents)

    # -- lifetime
    def close(self):
        if getattr(self, "h", None):
            check(self.lib.amber_model_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- stepping
    def step(self, n_steps: int = 1):
        check(self.lib.amber_step(self.h, int(n_steps)))

    def synchronize(self):
        check(self.lib.amber_synchronize(self.h))

    @property
    def step_count(self) -> int:
        v = C.c_int64()
        check(self.lib.amber_step_count(self.h, C.byref(v)))
        return v.value

    def set_step(self, s: int):
        check(self.lib.amber_set_step(self.h, int(s)))

    # -- columns
    def column_info(self, name: str):
        dt, g, off, ln = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
        check(self.lib.amber_column_info(self.h, name.encode(), C.byref(dt), C.byref(g),
                                         C.byref(off), C.byref(ln)))
        return _NP[dt.value], g.value, off.value, ln.value

    def read_column(self, name: str, out=None):
        """Host numpy array (default) or into `out` (numpy or CUDA torch tensor)."""
        dt, _, _, ln = self.column_info(name)
        if out is None:
            out = np.empty(ln, dtype=dt)
        if isinstance(out, np.ndarray):
            check(self.lib.amber_read_column(self.h, name.encode(), out.ctypes.data_as(C.c_void_p),
                                             out.nbytes, 0))
        else:  # torch tensor on the device
            check(self.lib.amber_read_column(self.h, name.encode(), C.c_void_p(out.data_ptr()),
                                             out.numel() * out.element_size(),
                                             1 if out.is_cuda else 0))
        return out

    def write_column(self, name: str, data):
        dt, _, _, ln = self.column_info(name)
        if isinstance(data, np.ndarray):
            a = np.ascontiguousarray(data, dtype=dt)
            check(self.lib.amber_write_column(self.h, name.encode(), a.ctypes.data_as(C.c_void_p),
                                              a.nbytes, 0))
        else:
            check(self.lib.amber_write_column(self.h, name.encode(), C.c_void_p(data.data_ptr()),
                                              data.numel() * data.element_size(),
                                              1 if data.is_cuda else 0))

    # -- observables
    def metrics(self, name: str):
        cap = self.get_option("metrics_capacity")
        out = np.zeros(cap, dtype=_METRIC_DT[name])
        n = C.c_int64()
        check(self.lib.amber_read_metrics(self.h, name.encode(), out.ctypes.data_as(C.c_void_p),
                                          out.nbytes, C.byref(n)))
        return out[: n.value].copy()

    def reset_metrics(self):
        check(self.lib.amber_reset_metrics(self.h))

    def digest(self, name: str) -> int:
        v = C.c_uint64()
        check(self.lib.amber_digest(self.h, name.encode(), C.byref(v)))
        return v.value

    def set_option(self, key: str, value: int):
        check(self.lib.amber_set_option(self.h, key.encode(), int(value)))

    def get_option(self, key: str) -> int:
        v = C.c_int64()
        check(self.lib.amber_get_option(self.h, key.encode(), C.byref(v)))
        return v.value

    # -- profiling (CUDA events on the model stream)
    def profile(self, enable: bool):
        check(self.lib.amber_profile_enable(self.h, 1 if enable else 0))

    def profile_results(self):
        res, i = [], 0
        name = C.create_string_buffer(128)
        while True:
            ln, ms = C.c_int64(), C.c_double()
            rc = self.lib.amber_profile_query(self.h, i, name, 128, C.byref(ln), C.byref(ms))
            if rc != 0:
                break
            res.append((name.value.decode(), ln.value, ms.value))
            i += 1
        return res


def wealth_params(w0=1, amount=1, exclude_self=0, counter_bits=0):
    return capi.amber_wealth_params(w0, amount, exclude_self, counter_bits)


def sir_params(mean_degree=10.0, beta=0.05, gamma=0.1, init_frac=0.01):
    return capi.amber_sir_params(mean_degree, beta, gamma, init_frac)


def boids_params(L=1000.0, R=10.0, rs=2.0, wc=0.01, wa=0.125, ws=0.05, vmax=2.0, dt=1.0):
    return capi.amber_boids_params(L, R, rs, wc, wa, ws, vmax, dt)


def sir_space_params(L=100.0, r=2.0, p_infect=0.1, p_recover=0.05, init_frac=0.01):
    return capi.amber_sir_space_params(L, r, p_infect, p_recover, init_frac)


def walk_params(L=100.0, vmax=1.0):
    return capi.amber_walk_params(L, vmax)


def sweep(n_agents, params, betas, seeds, n_steps, *, device=0, stream=None, torch_alloc=True,
          rank=0, world=1, unique_id=None, with_stats=False):
    """amber_sweep: final R fraction per replicate (host numpy float64)."""
    betas = np.asarray(betas, dtype=np.float64)
    seeds = np.asarray(seeds, dtype=np.uint64)
    reps = (capi.amber_replicate * max(len(betas), 1))()
    for r, (b, s) in enumerate(zip(betas, seeds)):
        reps[r].beta = float(b)
        reps[r].seed = int(s)
    out = np.zeros(len(betas), dtype=np.float64)
    rt = make_runtime(device, stream, torch_alloc, rank, world, unique_id)
    st = capi.amber_sweep_stats()
    check(capi.lib().amber_sweep(capi.AMBER_SIR_GRAPH, int(n_agents), C.byref(params),
                                 C.sizeof(params), reps, len(betas), int(n_steps), C.byref(rt),
                                 out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(st)))
    if with_stats:
        return out, dict(build_ms=st.build_ms, step_ms=st.step_ms, agent_updates=st.agent_updates,
                         active_updates=st.active_updates)
    return out
