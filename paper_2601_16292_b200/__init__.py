"""paper_2601_16292_b200 -- B200-native hot path of AMBER (arXiv 2601.16292).

The per-step, population-wide synchronous update of columnar agent state,
as hand-written sm_100a CUDA kernels behind the C ABI in include/amber.h
(libamber.so).  This package is the thin Python binding over that ABI; it
never imports oracle/ and has no CPU fallback.
"""
from . import capi
from .capi import AmberError
from .model import (Model, boids_params, loopback_id, make_runtime, nccl_unique_id, shard_range, sir_params, sir_shard_range,
                    sweep, sweep_range, sir_space_params, walk_params, wealth_params)

from .population import Population, agent_id, col, lit, rand, step_index

__all__ = ["Population", "col", "lit", "rand", "agent_id", "step_index", "capi", "AmberError", "Model", "wealth_params", "sir_params", "boids_params", "sweep",
           "make_runtime", "nccl_unique_id", "shard_range", "sir_shard_range", "sweep_range", "loopback_id", "walk_params", "sir_space_params"]
