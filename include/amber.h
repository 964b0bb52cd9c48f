/*
 * amber.h -- C ABI of the B200-native AMBER hot path (libamber.so).
 *
 * What it computes: the per-step, population-wide, SYNCHRONOUS update of
 * columnar (struct-of-arrays) agent state from arXiv 2601.16292 ("AMBER"):
 *   - state lives in typed columns, one entry per agent id
 *     (Sec. 3.1.2 lines 85-96: "each attribute is a column ... rows
 *     corresponding to agents identified by sequential integer IDs");
 *   - a step reads one consistent snapshot and commits all writes together
 *     (Sec. 3.4: "all agents act on a consistent state
 *     snapshot");
 *   - the three model kinds are the paper's benchmark patterns as fixed by
 *     BASELINE.json: wealth transfer (Sec. 5.1.1), SIR on a
 *     contact network (line 203 + Listing 2; network per
 *     Sec. 4.1) and flocking in continuous wrapped space (Sec. 4.1
 *     line 175; BASELINE.json config 3); replicate sweeps follow Sec. 4.2
 *     line 181 / Sec. 4.4 line 191.
 * Every random draw is a pure function of (seed, step, agent/edge id) via
 * Philox4x32-10 (DESIGN.md "Contract" R1-R8), so results are independent of
 * launch geometry, rank count and call chunking.
 *
 * Conventions (all entry points):
 *   - Return 0 (AMBER_OK) on success, a negative AMBER_E_* code otherwise;
 *     amber_last_error() then returns a thread-local message.  No C++
 *     exception crosses this boundary.
 *   - Pointers: "host" = ordinary CPU memory; "device" = CUDA device memory of
 *     the model's device.  Every function documents which it takes.
 *   - Ownership: the library owns models and all their device buffers
 *     (freed by amber_model_destroy).  Caller-supplied buffers (dst/src/params/
 *     reps/out) stay owned by the caller and are not retained after return.
 *     The CUDA stream in amber_runtime is borrowed, never destroyed.
 *   - Asynchrony: amber_step only enqueues work on the model's stream.  Any
 *     call that returns data (read_*, digest, synchronize) first waits for it.
 *     Device faults surface at the next synchronising call as AMBER_E_CUDA.
 *   - Threading: a model is single-writer; distinct models may be used from
 *     distinct threads on distinct streams.
 */
#ifndef AMBER_H
#define AMBER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMBER_ABI_VERSION 1

typedef struct amber_model amber_model; /* opaque, library-owned */

typedef enum {
    AMBER_WEALTH = 0,    /* wealth transfer; column "wealth" (int32)            */
    AMBER_SIR_GRAPH = 1, /* SIR on an Erdos-Renyi CSR graph; column "state" (u8) */
    AMBER_BOIDS = 2,     /* flocking; columns pos_x, pos_y, vel_x, vel_y (f32)  */
    AMBER_WALK = 3,      /* random walk; columns pos_x, pos_y, origin_x, origin_y (f32) */
    AMBER_SIR_SPACE = 4  /* SIR in continuous space; columns state (u8), pos_x, pos_y (f32) */
} amber_kind;

typedef enum {
    AMBER_I32 = 0,
    AMBER_U8 = 1,
    AMBER_F32 = 2,
    AMBER_I64 = 3,
    AMBER_F64 = 4,
    AMBER_U64 = 5
} amber_dtype;

enum {
    AMBER_OK = 0,
    AMBER_E_INVALID_ARG = -1,    /* bad size, NULL where not allowed, out-of-range param */
    AMBER_E_UNKNOWN_KIND = -2,
    AMBER_E_UNKNOWN_NAME = -3,   /* no such column / metric / option for this kind */
    AMBER_E_BUFFER_TOO_SMALL = -4,
    AMBER_E_CUDA = -5,           /* CUDA runtime error (message has the CUDA string) */
    AMBER_E_NCCL = -6,           /* NCCL unavailable or failed */
    AMBER_E_OOM = -7,            /* device allocation failed */
    AMBER_E_UNSUPPORTED = -8     /* valid request this build does not support */
};

/* Device allocator hook (e.g. the PyTorch caching allocator).  alloc returns
 * device memory of `bytes` usable on `stream`, or NULL on failure. */
typedef void* (*amber_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*amber_free_fn)(void* ptr, size_t bytes, void* stream, void* ctx);

/* Runtime binding.  May be NULL in every call that takes it: then device 0,
 * a library-created stream, cudaMalloc, and a single process (world = 1). */
typedef struct {
    int device;                 /* CUDA device ordinal */
    void* stream;               /* cudaStream_t (borrowed) or NULL */
    amber_alloc_fn alloc;       /* NULL -> cudaMalloc */
    amber_free_fn free;         /* must be set iff alloc is set */
    void* alloc_ctx;            /* passed back to alloc/free */
    int rank;                   /* this process's rank in [0, world) */
    int world;                  /* number of processes (one GPU each); 0 or 1 = single */
    const void* nccl_unique_id; /* 128-byte id from amber_nccl_unique_id() on rank 0,
                                   broadcast to all ranks; required iff world > 1, unless
                                   host collectives are given (below) */
    /* Optional host collectives of the caller's own transport (e.g. a gloo or MPI
     * process group).  Used only when world > 1 and nccl_unique_id is NULL, and
     * only by the sharded wealth model: its peer-memory (P2P) exchange then maps
     * the peers' bucket blocks through CUDA IPC handles all-gathered with
     * host_allgather, and orders every step with host_barrier after the stream
     * drains (no kernel ever waits on another process's kernel).  Both are
     * collective over all ranks and return 0 on success; a non-zero return fails
     * the call with AMBER_E_NCCL.  host_allgather gathers `bytes` from every rank
     * into recv (world * bytes, rank order). */
    int (*host_allgather)(const void* send, void* recv, size_t bytes, void* ctx);
    int (*host_barrier)(void* ctx);
    void* host_ctx;
} amber_runtime;

/* ---- model parameters (POD, passed as pointer + sizeof for ABI growth) ---- */

/* Wealth transfer (Sec. 5.1.1: "each agent transfer a fixed
 * amount of wealth to a randomly selected other agent at each step").
 * Step t: s_i = [w_i >= amount] on the snapshot; receiver
 * r_i = floor(x * N / 2^64), x = 64-bit Philox lane (tag 0x01, lane i, step t)
 * (exclude_self = 1: r = floor(x * (N-1) / 2^64), r += (r >= i));
 * w_i' = w_i - amount*s_i + amount*#{j : s_j and r_j = i}.   Contract W1-W2. */
typedef struct {
    int32_t w0;           /* initial wealth of every agent (>= 0) */
    int32_t amount;       /* units given per step by each sender (>= 1) */
    int32_t exclude_self; /* 0: receiver uniform over all N (BJ config 1); 1: over N-1 others */
    int32_t counter_bits; /* scatter of the transfers: {0 (default = 4), 2, 4, 8, 16, 32} =
                             per-receiver counter width for L2 atomics (narrow counters stay
                             L2-resident; an overflow is detected exactly and the step window
                             is replayed with 32-bit counters); any other value is
                             AMBER_E_INVALID_ARG */
} amber_wealth_params;

/* SIR on G(n, M) (Sec. 5.1.1, Listing 2;
 * BASELINE.json config 2).  M = round(N*mean_degree/2) endpoint draws,
 * de-duplicated (G1-G3); K = round(init_frac*N) initial infected with the
 * smallest 64-bit init keys (S1).  Step t from snapshot X: a susceptible s
 * becomes I iff some neighbour i with X[i] = I has Philox word0 of counter
 * (min(s,i), max(s,i), t, 0x10) < ceil(beta*2^32); an infected agent becomes
 * R iff its 32-bit lane (tag 0x11) < ceil(gamma*2^32).  Contract S2-S4. */
typedef struct {
    double mean_degree; /* k-bar > 0 */
    double beta;        /* per S-I edge per step, in [0, 1] */
    double gamma;       /* per I agent per step, in [0, 1] */
    double init_frac;   /* fraction initially infected, in [0, 1] */
} amber_sir_params;

/* Boids in an L x L periodic box (BASELINE.json config 3; wrapped continuous
 * space per PAPER.md Sec. 4.1).  Rules, float contract and fixed-point
 * neighbour sums: DESIGN.md "Contract" B1-B7. Requires vmax*dt < L/2, R < L/2. */
typedef struct {
    float L, R, rs, wc, wa, ws, vmax, dt;
} amber_boids_params;

/* Random Walk (Sec. 5.1.1, Sec. 5.3; DESIGN.md
 * K1-K3).  Positions uniform in [0, L)^2 (32-bit lanes 2i, 2i+1 of tag 0x30);
 * step t: v = (2u - 1) * vmax per component from lanes 2i, 2i+1 of tag 0x31,
 * p' = clip(p + v) into [0, largest float below L] (float32, no FMA).
 * Metric "mean_displacement" = mean |p - origin| (per step, double sum). */
typedef struct {
    float L;    /* box side (> 0) */
    float vmax; /* max speed per component (>= 0) */
} amber_walk_params;

/* SIR in continuous space -- the paper's SIR benchmark (Sec. 5.1.1
 * line 203, Listing 2; C1-C4).  Static positions
 * uniform in [0, L)^2 (lanes 2i, 2i+1 of tag 0x40); contacts: j != i with
 * dx*dx + dy*dy <= r*r (float, bounded box, inclusive), built once; initial
 * infected: the round(init_frac*N) smallest lane64(0x42, i) keys.  Step t: a
 * susceptible with >= 1 infected contact becomes I iff lane32(0x41, i, t) <
 * ceil(p_infect*2^32) (ONE draw, Listing 2); infected recover iff
 * lane32(0x43, i, t) < ceil(p_recover*2^32). */
typedef struct {
    float L;          /* box side (> 0) */
    float r;          /* contact radius (> 0) */
    double p_infect;  /* per exposed susceptible per step, in [0, 1] */
    double p_recover; /* per infected per step, in [0, 1] */
    double init_frac; /* fraction initially infected, in [0, 1] */
} amber_sir_space_params;

/* One replicate of a sweep (Sec. 4.2). */
typedef struct {
    double beta;   /* this replicate's transmission probability */
    uint64_t seed; /* this replicate's seed (own graph, own initial infected) */
} amber_replicate;

/* Optional timing breakdown returned by amber_sweep (all host values). */
typedef struct {
    double build_ms;        /* graph + initial-state construction on the device */
    double step_ms;         /* the stepping kernels (the hot path) */
    int64_t agent_updates;  /* n_agents * n_steps * n_reps_local (nominal) */
    int64_t active_updates; /* agent-steps executed before each replicate's I reached 0 */
} amber_sweep_stats;

/* ---------------------------------------------------------------- lifetime */

/* Library ABI version (AMBER_ABI_VERSION). */
int amber_version(void);

/* Thread-local message for the last non-zero status ("" if none). */
const char* amber_last_error(void);

/* Create a model of `kind` with n_agents agents (global count when sharded),
 * params of the kind's struct (params_size = sizeof), and a 64-bit seed
 * (Philox key, contract R2).  The initial state is built on the device
 * (W: w = w0; S: graph + initial infected; B: contract B1), step count 0.
 * When rt->world > 1 the call is collective over all ranks and the agents are
 * sharded by contiguous id ranges (see amber_column_info for this rank's
 * slice): AMBER_WEALTH (ranges of ceil(N/world) rounded up to 8; receivers
 * exchanged per step) and AMBER_SIR_GRAPH (ranges rounded up to 32 agents;
 * every rank builds the seeded graph and keeps its rows; per step a pull over
 * the local rows against the global I bitmap, then an all-gather of the
 * bitmap, N/8 bytes; results identical for any world size).  Sharded SIR
 * column "state" is the local slice, "row_ptr"/"col_idx" the local rows
 * (offsets from 0, global neighbour ids); metrics and digests are global.
 * AMBER_BOIDS: x-slabs of whole grid-cell columns (rank r owns columns
 * [r*nc/world, (r+1)*nc/world), nc = cells per side >= max(3, world)); per
 * step agents migrate to the slab of their cell column and the first / last
 * column of each slab is sent to the neighbours as halos (variable all-to-all);
 * bit-identical to one GPU (exact fixed-point sums).  Sharded Boids column
 * reads / writes / digests are collective and use the whole id-ordered column.
 * Errors: INVALID_ARG (n_agents < 1, bad params, params_size too small),
 * UNKNOWN_KIND, OOM, CUDA, NCCL, UNSUPPORTED (world > 1 for another kind). */
int amber_model_create(amber_kind kind, int64_t n_agents, const void* params, size_t params_size,
                       uint64_t seed, const amber_runtime* rt, amber_model** out);

/* Destroy a model and free its device memory (waits for its stream). NULL is a no-op. */
int amber_model_destroy(amber_model* m);

/* ---------------------------------------------------------------- stepping */

/* Enqueue n_steps >= 0 synchronous steps on the model's stream (asynchronous).
 * Per-step observables are recorded on the device after every step.
 * Collective when sharded (every rank must call it with the same n_steps). */
int amber_step(amber_model* m, int64_t n_steps);

/* Wait for all enqueued work; also runs the wealth counter-overflow check
 * (and the exact replay, if one is needed). */
int amber_synchronize(amber_model* m);

/* Current step index (number of steps applied since step 0). */
int amber_step_count(amber_model* m, int64_t* out);

/* Set the step index used by the next step's draws (checkpoint/resume;
 * together with amber_write_column this restores any saved state exactly). */
int amber_set_step(amber_model* m, int64_t step);

/* ----------------------------------------------------------------- columns */

/* Describe column `name`: dtype, global length, and this rank's slice
 * [local_off, local_off + local_len).  Any out pointer may be NULL.
 * Errors: UNKNOWN_NAME. */
int amber_column_info(amber_model* m, const char* name, amber_dtype* dtype, int64_t* global_len,
                      int64_t* local_off, int64_t* local_len);

/* Copy this rank's slice of column `name`, in agent-id order, into dst
 * (host memory if dst_on_device == 0, device memory otherwise).
 * Synchronising.  Errors: UNKNOWN_NAME, BUFFER_TOO_SMALL (dst_bytes < slice bytes). */
int amber_read_column(amber_model* m, const char* name, void* dst, size_t dst_bytes,
                      int dst_on_device);

/* Overwrite this rank's slice of column `name` from src (host or device), in
 * agent-id order (checkpoint restore / user-supplied initial state).
 * Read-only columns (row_ptr, col_idx) return INVALID_ARG. */
int amber_write_column(amber_model* m, const char* name, const void* src, size_t src_bytes,
                       int src_on_device);

/* ----------------------------------------------------------------- metrics */

/* Per-step observables recorded after each step (SPEC run_model "collect"),
 * for the most recent min(steps_recorded, capacity) steps, oldest first, as
 * host values in dst.  Names: wealth: "total_wealth" (i64), "active" (i64),
 * "digest" (u64, only if option "digest" = 1); SIR: "S", "I", "R" (i64),
 * "digest"; Boids: "mean_speed", "polarisation" (f64), "digest" (of pos_x).
 * Sharded models return global (all-rank) values.  *n_out = number of values.
 * Errors: UNKNOWN_NAME, BUFFER_TOO_SMALL. */
int amber_read_metrics(amber_model* m, const char* name, void* dst, size_t dst_bytes,
                       int64_t* n_out);

/* Forget recorded metrics (the next read starts at the next step). */
int amber_reset_metrics(amber_model* m);

/* D1 digest of a column's current value: sum_i mix64((i << 32) ^ bits32(v_i))
 * mod 2^64 over all agents (global when sharded).  Synchronising.  SIR models
 * also accept "row_ptr" and "col_idx": the same sum over the int32 CSR arrays
 * with the array index as i (the local rows of a shard, not all-reduced) --
 * lets tests compare a full-size graph with an oracle-written golden digest. */
int amber_digest(amber_model* m, const char* name, uint64_t* out);

/* Model options (int64 values): "digest" (0/1: record a per-step digest of the
 * primary column; off by default because it is a parity checksum, not a model
 * observable), "metrics_capacity" (ring size, >= 16), "block" (threads per
 * block for launch-geometry invariance tests; 0 = tuned default),
 * "grid" (persistent grid size; 0 = tuned default), "persistent"
 * (wealth/SIR: 1 = all steps of a call in one launch (single-CTA kernel for
 * wealth N <= 16384; cooperative direction-optimizing kernel for SIR),
 * 0 = one launch per step, pull only for SIR), SIR "direction" (0 = choose
 * per step, push when 4I < 3S (10I < 9S at 8 agents per lane; sharded: from the
 * global counts of the all-gathered bitmaps); 1 = always pull; 2 = push whenever
 * the previous counts are known -- identical results, for tests and probes;
 * 1 or 2 also run a single step through the cooperative kernel), SIR "apl" (agents per
 * lane of the step kernels: 0 = auto (8 above 2^22 agents, else 1), 1, 2, 4
 * or 8 -- identical results); Boids: "lanes" (4/8/16 lanes per agent in the
 * stencil, default 4 -- identical results).
 * Test hook: wealth "inject_counter_fault" = local agent k adds one count to
 * k's pending receiver counter (fault injection: the exact overflow check must
 * catch it and the replay repair it).
 * Read-only (amber_get_option): wealth "replays" (exact-replay count, after
 * the overflow check), "counter_bits", "scatter" (1: packed-counter L2
 * atomics, the one shipped scatter), "exchange" (sharded: 0 none,
 * 1 NCCL send/recv, 2 P2P peer-mapped id buckets, 3 P2P dense: every rank's
 * global packed counters summed by the owners in place; set at the first
 * step; environment AMBER_WEALTH_EXCHANGE = dense | sparse | nccl, default
 * dense up to 8 ranks when each shard's counter block is word-aligned); SIR
 * "edges"; Boids "cells_per_side", sharded Boids "own_agents" and
 * "slab_columns". */
int amber_set_option(amber_model* m, const char* key, int64_t value);
int amber_get_option(amber_model* m, const char* key, int64_t* value);

/* Per-kernel device timing (CUDA events on the model's stream) for profiling
 * and roofline reporting.  enable != 0 starts (and clears) recording.
 * query(idx) returns the idx-th kernel name with its launch count and total
 * milliseconds since enabling (synchronising); INVALID_ARG past the last. */
int amber_profile_enable(amber_model* m, int enable);
int amber_profile_query(amber_model* m, int idx, char* name, size_t name_cap, int64_t* launches,
                        double* total_ms);

/* ------------------------------------------------------------------- sweep */

/* Run n_reps independent replicates of `kind` (AMBER_SIR_GRAPH only) with
 * base params (beta taken per replicate from reps[r].beta, seed from
 * reps[r].seed), n_steps steps each, and write each replicate's final
 * R fraction (R / n_agents, an exact ratio of integers) into
 * out_final_r_frac[r] (host, n_reps doubles).  When rt->world > 1 rank g
 * runs replicates [g*n_reps/world, (g+1)*n_reps/world) and the results are
 * gathered so every rank receives all n_reps values (collective).
 * stats may be NULL.  Errors: INVALID_ARG, UNKNOWN_KIND, OOM, CUDA, NCCL. */
int amber_sweep(amber_kind kind, int64_t n_agents, const void* base_params, size_t params_size,
                const amber_replicate* reps, int64_t n_reps, int64_t n_steps,
                const amber_runtime* rt, double* out_final_r_frac, amber_sweep_stats* stats);

/* ------------------------------------------------------------ multi-GPU */

/* Host-only (no device needed): the contiguous agent range [*lo, *hi) that rank
 * `rank` of `world` owns in a sharded wealth model of n_agents:
 * shard size = ceil(n/world) rounded up to a multiple of 8 agents, so the
 * two-agent Philox blocks (contract R4) never straddle shards; trailing ranks
 * may be shorter or empty.  Errors: INVALID_ARG. */
int amber_shard_range(int64_t n_agents, int world, int rank, int64_t* lo, int64_t* hi);

/* Host-only: the agent range [*lo, *hi) of rank `rank` in a sharded
 * AMBER_SIR_GRAPH model (NEXT-3): shard size = ceil(n/world) rounded up to a
 * multiple of 32 agents, so one word of the per-step all-gathered I bitmap
 * never spans two ranks; trailing ranks may be shorter or empty.
 * Errors: INVALID_ARG. */
int amber_sir_shard_range(int64_t n_agents, int world, int rank, int64_t* lo, int64_t* hi);

/* Host-only: the replicates [*r0, *r1) that rank `rank` of `world` runs in
 * amber_sweep (blocks of ceil(n_reps/world)).  Errors: INVALID_ARG. */
int amber_sweep_range(int64_t n_reps, int world, int rank, int64_t* r0, int64_t* r1);

/* Write a fresh 128-byte NCCL unique id into out (host, out_bytes >= 128).
 * Call on rank 0 and broadcast it (e.g. with torch.distributed).
 * Errors: NCCL (libnccl.so.2 not loadable: set AMBER_NCCL_LIB to its path). */
int amber_nccl_unique_id(void* out, size_t out_bytes);

/* ------------------------------------------------- generic Population (NEXT-4) */
/* The paper's general columnar API (Sec. 3.1.2 lines 85-96 and
 * Listing 1 "population.data.with_columns((pl.col('wealth') + 10))", Sec. 3.3
 * line 155 "columnar updates for all or filtered agents ... BatchUpdateContext
 * ... applying all changes atomically", Sec. 6.2 line 284 dynamic populations)
 * on the device: typed columns (one row per agent), an alive mask, stable
 * agent ids (never reused), population-wide updates and aggregates given as
 * postfix expression programs evaluated per row by one kernel. */
typedef struct amber_population amber_population; /* opaque, library-owned */

typedef struct {
    const char* name;  /* column name (copied) */
    amber_dtype dtype; /* AMBER_I32, AMBER_I64, AMBER_F32, AMBER_F64 or AMBER_U8 */
} amber_column_spec;

/* Expression instruction (postfix / stack machine of at most 64 instructions
 * and stack depth 8, evaluated in double per row; results are stored with C
 * conversion semantics: truncation toward zero for integer columns).  arg = column index for AMBER_OP_COL, tag for
 * AMBER_OP_RAND; value = the constant for AMBER_OP_CONST. */
typedef enum {
    AMBER_OP_CONST = 0, AMBER_OP_COL = 1, AMBER_OP_ID = 2, AMBER_OP_STEP = 3,
    AMBER_OP_ADD = 10, AMBER_OP_SUB, AMBER_OP_MUL, AMBER_OP_DIV, AMBER_OP_MIN, AMBER_OP_MAX,
    AMBER_OP_NEG = 20, AMBER_OP_ABS, AMBER_OP_FLOOR, AMBER_OP_SQRT,
    AMBER_OP_LT = 30, AMBER_OP_LE, AMBER_OP_GT, AMBER_OP_GE, AMBER_OP_EQ, AMBER_OP_NE,
    AMBER_OP_AND = 40, AMBER_OP_OR, AMBER_OP_NOT,
    AMBER_OP_SELECT = 50, /* c a b -> c != 0 ? a : b */
    AMBER_OP_RAND = 60    /* uniform [0,1): (lane32(tag=arg, agent id, step) >> 8) * 2^-24 */
} amber_op;

typedef struct {
    int32_t op;
    int32_t arg;
    double value;
} amber_instr;

typedef enum { AMBER_AGG_SUM = 0, AMBER_AGG_MEAN = 1, AMBER_AGG_MIN = 2, AMBER_AGG_MAX = 3, AMBER_AGG_COUNT = 4 } amber_agg;

/* Create an empty population (0 agents) with n_cols typed columns and room for
 * `capacity` rows (grows on demand).  seed keys AMBER_OP_RAND draws.
 * Errors: INVALID_ARG (duplicate/empty names, bad dtype, n_cols < 1). */
int amber_population_create(const amber_column_spec* cols, int n_cols, int64_t capacity, uint64_t seed,
                            const amber_runtime* rt, amber_population** out);
int amber_population_destroy(amber_population* p);

/* Append n live agents; their ids are next_id .. next_id+n-1 (*first_id).
 * defaults: n_cols host doubles (initial value per column) or NULL (zeros). */
int amber_population_add_agents(amber_population* p, int64_t n, const double* defaults, int64_t* first_id);

/* Mark agents dead (host id list).  Errors: INVALID_ARG (unknown or dead id;
 * then nothing is removed). */
int amber_population_remove_agents(amber_population* p, const int64_t* ids, int64_t n);

/* Drop dead rows, keeping row order (stream compaction on the device). */
int amber_population_compact(amber_population* p);

/* *live = live agents, *rows = rows in use (live + dead before compaction). */
int amber_population_size(amber_population* p, int64_t* live, int64_t* rows);

/* Host-only counters: general-program updates (not the Listing-1 fast path)
 * run so far as runtime-compiled kernels (*n_jit: NVRTC, sm_100a; the
 * expression becomes straight-line double code) or through the columnar
 * interpreter (*n_interp: no NVRTC, a failed compile, or AMBER_POP_JIT=0 when
 * the population was created).  Both paths compute identical values. */
int amber_population_update_paths(amber_population* p, int64_t* n_jit, int64_t* n_interp);

/* Synchronous population-wide update: for every live row where `where`
 * evaluates != 0 (n_where == 0: every live row), target = expr(row), all rows
 * reading the pre-update snapshot (SPEC update_column / update_where).
 * *n_updated = rows updated (synchronising); n_updated == NULL makes the call
 * fully asynchronous on the population's stream (amber_population_synchronize).  Errors: UNKNOWN_NAME, INVALID_ARG
 * (bad program: stack underflow/overflow, unknown op, column index). */
int amber_population_update(amber_population* p, const char* target, const amber_instr* expr, int n_expr,
                            const amber_instr* where, int n_where, int64_t* n_updated);

/* Reduce expr over live rows where `where` holds (double result on the host;
 * COUNT counts the rows, SUM of an empty set is 0).  Errors: INVALID_ARG for
 * MEAN/MIN/MAX of an empty set (SPEC aggregate). */
int amber_population_aggregate(amber_population* p, int agg, const amber_instr* expr, int n_expr,
                               const amber_instr* where, int n_where, double* out);

/* Column of the LIVE agents in row order (host or device dst); "id" (I64) is
 * the implicit agent-id column.  Errors: UNKNOWN_NAME, BUFFER_TOO_SMALL. */
int amber_population_read_column(amber_population* p, const char* name, void* dst, size_t dst_bytes,
                                 int dst_on_device);

/* Atomic batch of individual writes (BatchUpdateContext): values[k] goes to
 * column `name` of agent ids[k] (host arrays).  Every id is validated first;
 * on any error nothing is written.  Duplicate ids: the last write wins. */
int amber_population_batch_set(amber_population* p, const char* name, const int64_t* ids,
                               const double* values, int64_t n);

/* Wait for all work enqueued on the population's stream. */
int amber_population_synchronize(amber_population* p);

/* Step counter read by AMBER_OP_STEP / AMBER_OP_RAND (advance it per model step). */
int amber_population_set_step(amber_population* p, int64_t step);

/* Write a 128-byte id for an in-process LOOPBACK group (testing/emulation):
 * `world` models created with this id (rank 0..world-1) on one device form a
 * sharded model whose exchanges are host barriers + device-to-device copies
 * instead of NCCL.  Each rank's calls must come from its own host thread
 * (collective calls block until every rank has made them).  Errors: INVALID_ARG. */
int amber_loopback_id(void* out, size_t out_bytes);

#ifdef __cplusplus
}
#endif
#endif /* AMBER_H */
