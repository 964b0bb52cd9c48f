"""Thin ctypes binding of include/amber.h (argument marshalling only).

Every function below has the C name and signature of the C ABI; all
computation happens in libamber.so's CUDA kernels.  There is no CPU fallback:
importing this module raises if libamber.so has not been built, and every
call on a machine without a CUDA device fails with AMBER_E_CUDA from the
library itself.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AMBER_LIB_PATH") or os.path.join(PKG, "libamber.so")

AMBER_WEALTH, AMBER_SIR_GRAPH, AMBER_BOIDS, AMBER_WALK, AMBER_SIR_SPACE = 0, 1, 2, 3, 4
AMBER_I32, AMBER_U8, AMBER_F32, AMBER_I64, AMBER_F64, AMBER_U64 = range(6)
AMBER_OK = 0
ERRORS = {-1: "AMBER_E_INVALID_ARG", -2: "AMBER_E_UNKNOWN_KIND", -3: "AMBER_E_UNKNOWN_NAME",
          -4: "AMBER_E_BUFFER_TOO_SMALL", -5: "AMBER_E_CUDA", -6: "AMBER_E_NCCL", -7: "AMBER_E_OOM",
          -8: "AMBER_E_UNSUPPORTED"}

# Header symbols (tests check that the library exports every one of them).
SYMBOLS = ["amber_version", "amber_last_error", "amber_model_create", "amber_model_destroy",
           "amber_step", "amber_synchronize", "amber_step_count", "amber_set_step",
           "amber_column_info", "amber_read_column", "amber_write_column", "amber_read_metrics",
           "amber_reset_metrics", "amber_digest", "amber_set_option", "amber_get_option",
           "amber_profile_enable", "amber_profile_query", "amber_sweep", "amber_shard_range", "amber_sir_shard_range",
           "amber_sweep_range", "amber_nccl_unique_id", "amber_loopback_id",
           "amber_population_create", "amber_population_destroy", "amber_population_add_agents",
           "amber_population_remove_agents", "amber_population_compact", "amber_population_size",
           "amber_population_update", "amber_population_aggregate", "amber_population_read_column",
           "amber_population_batch_set", "amber_population_synchronize", "amber_population_set_step",
           "amber_population_update_paths"]

ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
HOST_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
HOST_BARRIER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class amber_runtime(C.Structure):
    _fields_ = [("device", C.c_int), ("stream", C.c_void_p), ("alloc", ALLOC_FN),
                ("free", FREE_FN), ("alloc_ctx", C.c_void_p), ("rank", C.c_int),
                ("world", C.c_int), ("nccl_unique_id", C.c_void_p),
                ("host_allgather", HOST_ALLGATHER_FN), ("host_barrier", HOST_BARRIER_FN),
                ("host_ctx", C.c_void_p)]


class amber_wealth_params(C.Structure):
    _fields_ = [("w0", C.c_int32), ("amount", C.c_int32), ("exclude_self", C.c_int32),
                ("counter_bits", C.c_int32)]


class amber_sir_params(C.Structure):
    _fields_ = [("mean_degree", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
                ("init_frac", C.c_double)]


class amber_boids_params(C.Structure):
    _fields_ = [(k, C.c_float) for k in ("L", "R", "rs", "wc", "wa", "ws", "vmax", "dt")]


class amber_walk_params(C.Structure):
    _fields_ = [("L", C.c_float), ("vmax", C.c_float)]


class amber_sir_space_params(C.Structure):
    _fields_ = [("L", C.c_float), ("r", C.c_float), ("p_infect", C.c_double),
                ("p_recover", C.c_double), ("init_frac", C.c_double)]


class amber_replicate(C.Structure):
    _fields_ = [("beta", C.c_double), ("seed", C.c_uint64)]


class amber_sweep_stats(C.Structure):
    _fields_ = [("build_ms", C.c_double), ("step_ms", C.c_double),
                ("agent_updates", C.c_int64), ("active_updates", C.c_int64)]


class amber_column_spec(C.Structure):
    _fields_ = [("name", C.c_char_p), ("dtype", C.c_int)]


class amber_instr(C.Structure):
    _fields_ = [("op", C.c_int32), ("arg", C.c_int32), ("value", C.c_double)]


class AmberError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


def _nccl_path():
    try:
        import nvidia  # torch's bundled NCCL: bind to the same copy torch uses
        for base in nvidia.__path__:
            p = os.path.join(base, "nccl", "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except ImportError:
        pass
    return ""


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                          "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    if not os.environ.get("AMBER_NCCL_LIB"):
        p = _nccl_path()
        if p:
            os.environ["AMBER_NCCL_LIB"] = p
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    i64p = P(C.c_int64)
    sig = {
        "amber_version": (C.c_int, []),
        "amber_last_error": (C.c_char_p, []),
        "amber_model_create": (C.c_int, [C.c_int, C.c_int64, C.c_void_p, C.c_size_t, C.c_uint64,
                                         P(amber_runtime), P(C.c_void_p)]),
        "amber_model_destroy": (C.c_int, [C.c_void_p]),
        "amber_step": (C.c_int, [C.c_void_p, C.c_int64]),
        "amber_synchronize": (C.c_int, [C.c_void_p]),
        "amber_step_count": (C.c_int, [C.c_void_p, i64p]),
        "amber_set_step": (C.c_int, [C.c_void_p, C.c_int64]),
        "amber_column_info": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_int), i64p, i64p, i64p]),
        "amber_read_column": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t, C.c_int]),
        "amber_write_column": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t, C.c_int]),
        "amber_read_metrics": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t, i64p]),
        "amber_reset_metrics": (C.c_int, [C.c_void_p]),
        "amber_digest": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_uint64)]),
        "amber_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
        "amber_get_option": (C.c_int, [C.c_void_p, C.c_char_p, i64p]),
        "amber_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
        "amber_profile_query": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.c_size_t, i64p,
                                          P(C.c_double)]),
        "amber_sweep": (C.c_int, [C.c_int, C.c_int64, C.c_void_p, C.c_size_t, P(amber_replicate),
                                  C.c_int64, C.c_int64, P(amber_runtime), P(C.c_double),
                                  P(amber_sweep_stats)]),
        "amber_shard_range": (C.c_int, [C.c_int64, C.c_int, C.c_int, i64p, i64p]),
        "amber_sweep_range": (C.c_int, [C.c_int64, C.c_int, C.c_int, i64p, i64p]),
        "amber_sir_shard_range": (C.c_int, [C.c_int64, C.c_int, C.c_int, i64p, i64p]),
        "amber_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_size_t]),
        "amber_loopback_id": (C.c_int, [C.c_void_p, C.c_size_t]),
        "amber_population_create": (C.c_int, [P(amber_column_spec), C.c_int, C.c_int64, C.c_uint64,
                                              P(amber_runtime), P(C.c_void_p)]),
        "amber_population_destroy": (C.c_int, [C.c_void_p]),
        "amber_population_add_agents": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_double), i64p]),
        "amber_population_remove_agents": (C.c_int, [C.c_void_p, i64p, C.c_int64]),
        "amber_population_compact": (C.c_int, [C.c_void_p]),
        "amber_population_size": (C.c_int, [C.c_void_p, i64p, i64p]),
        "amber_population_update": (C.c_int, [C.c_void_p, C.c_char_p, P(amber_instr), C.c_int,
                                              P(amber_instr), C.c_int, i64p]),
        "amber_population_aggregate": (C.c_int, [C.c_void_p, C.c_int, P(amber_instr), C.c_int,
                                                 P(amber_instr), C.c_int, P(C.c_double)]),
        "amber_population_read_column": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t, C.c_int]),
        "amber_population_batch_set": (C.c_int, [C.c_void_p, C.c_char_p, i64p, P(C.c_double), C.c_int64]),
        "amber_population_set_step": (C.c_int, [C.c_void_p, C.c_int64]),
        "amber_population_synchronize": (C.c_int, [C.c_void_p]),
        "amber_population_update_paths": (C.c_int, [C.c_void_p, i64p, i64p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB


def check(rc):
    if rc != AMBER_OK:
        raise AmberError(rc, lib().amber_last_error().decode(errors="replace"))
    return rc


def __getattr__(name):
    # amber_* names resolve to the raw C functions (same names as the C ABI)
    if name.startswith("amber_"):
        return getattr(lib(), name)
    raise AttributeError(name)
