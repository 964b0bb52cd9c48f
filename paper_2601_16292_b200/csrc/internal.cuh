// internal.cuh -- shared host/device infrastructure of libamber.so (product path).
// Errors, runtime binding (device, stream, allocator hooks), RAII device
// buffers, per-kernel CUDA-event profiler, the model interface, and small
// device reduction helpers.  Nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "amber.h"

namespace amber {

// ---------------------------------------------------------------- errors
struct Error {
    int code;
    std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error{code, msg}; }

#define AMBER_CUDA(call)                                                                   \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            ::amber::fail(e_ == cudaErrorMemoryAllocation ? AMBER_E_OOM : AMBER_E_CUDA,    \
                          std::string(#call) + " -> " + cudaGetErrorString(e_) + " (" +   \
                              __FILE__ + ":" + std::to_string(__LINE__) + ")");            \
    } while (0)

#define AMBER_REQUIRE(cond, msg)                                                  \
    do {                                                                          \
        if (!(cond)) ::amber::fail(AMBER_E_INVALID_ARG, std::string(msg));        \
    } while (0)

// AMBER_SYNC_DEBUG=1 (environment, read once): every checked launch is followed
// by a device synchronize, so an asynchronous fault (out-of-bounds access, a
// failed AMBER_DCHECK) is reported against the kernel that caused it.
inline bool sync_debug()
{
    static const bool on = [] {
        const char* v = std::getenv("AMBER_SYNC_DEBUG");
        return v && v[0] && v[0] != '0';
    }();
    return on;
}

// Programmatic dependent launch (PDL, sm_90+): a kernel launched with
// launch_pdl may start (be scheduled, run its prologue) while the previous
// kernel on the stream still runs; pdl_wait() -- griddepcontrol.wait -- blocks
// until that kernel has completed and its writes are visible, so such kernels
// call it before their first global memory access, then pdl_trigger() to let
// their own successor be scheduled.  Without the launch attribute both are
// no-ops.  AMBER_PDL=0 launches normally (A/B measurements).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline bool pdl_on()
{
    static const bool on = [] {
        const char* e = getenv("AMBER_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
template <class... KArgs, class... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    AMBER_CUDA(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

// Check the last launch (launch-config errors surface here, faults later --
// or here, under AMBER_SYNC_DEBUG).
inline void check_launch(const char* what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(AMBER_E_CUDA, std::string("launch ") + what + ": " + cudaGetErrorString(e));
    if (sync_debug()) {
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess)
            fail(AMBER_E_CUDA, std::string("AMBER_SYNC_DEBUG: ") + what + " -> " + cudaGetErrorString(e));
    }
}

// Device-side index checks, compiled in by the bounds build (-DAMBER_BOUNDS:
// paper_2601_16292_b200/libamber_bounds.so, `python -m paper_2601_16292_b200.build
// --bounds`); the product library compiles them out.  A failed check prints the
// site and traps (the launch fails with an unspecified-launch-failure error).
#ifdef AMBER_BOUNDS
#define AMBER_DCHECK(cond, what)                                                                    \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            printf("AMBER_BOUNDS %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, what,       \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                    \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#else
#define AMBER_DCHECK(cond, what) \
    do {                         \
    } while (0)
#endif

// ---------------------------------------------------------------- runtime
struct Runtime {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    amber_alloc_fn alloc = nullptr;
    amber_free_fn release = nullptr;
    void* ctx = nullptr;
    int rank = 0, world = 1;
    int num_sms = 148;

    std::vector<void*> nccl_comms;  // communicators this runtime's stream runs collectives on

    void init(const amber_runtime* rt);
    void destroy();
    void* alloc_bytes(size_t bytes);
    void free_bytes(void* p, size_t bytes);
    // Host wait for the stream.  With NCCL communicators attached, a polling
    // wait: ncclCommGetAsyncError on each, and a host timeout
    // (AMBER_NCCL_TIMEOUT_S, default 600 s); on an asynchronous NCCL error or
    // the timeout the communicators are aborted and the call fails with
    // AMBER_E_NCCL, so one dead rank cannot hang the others forever.
    void sync();
};

// NCCL hooks for Runtime::sync (defined in dist.cu): 0 = fine, else the message.
extern int (*g_nccl_async_error)(void* comm, std::string* msg);
extern void (*g_nccl_abort)(void* comm);

// RAII device buffer allocated through the runtime's allocator.
template <class T>
struct DevBuf {
    Runtime* rt = nullptr;
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    void allocate(Runtime* r, size_t count)
    {
        reset();
        rt = r;
        n = count;
        p = count ? static_cast<T*>(rt->alloc_bytes(count * sizeof(T))) : nullptr;
    }
    void reset()
    {
        if (p && rt) rt->free_bytes(p, n * sizeof(T));
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
    void zero_async(cudaStream_t s)
    {
        if (p) AMBER_CUDA(cudaMemsetAsync(p, 0, bytes(), s));
    }
};

// ---------------------------------------------------------------- profiler
// Records a CUDA event pair around every launch of a named kernel while
// enabled (on the launching stream), so per-kernel device time can be read
// back without an external profiler.
// NVTX range for the host side of a phase (amber_* entry points and every
// named kernel launch); header-only NVTX 3, free when no tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Profiler {
    bool on = false;
    struct Kernel {
        std::string name;
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    };
    std::vector<Kernel> kernels;
    std::vector<cudaEvent_t> pool;

    cudaEvent_t get_event();
    void clear();
    void enable(bool v) { clear(); on = v; }
    template <class F>
    void launch(cudaStream_t s, const char* name, F&& f)
    {
        NvtxRange nv(name);
        if (!on) {
            f();
            return;
        }
        cudaEvent_t a = get_event(), b = get_event();
        AMBER_CUDA(cudaEventRecord(a, s));
        f();
        AMBER_CUDA(cudaEventRecord(b, s));
        Kernel* k = nullptr;
        for (auto& kk : kernels)
            if (kk.name == name) k = &kk;
        if (!k) {
            kernels.push_back(Kernel{name, {}});
            k = &kernels.back();
        }
        k->ev.emplace_back(a, b);
    }
    bool query(int idx, std::string* name, int64_t* launches, double* total_ms);
    ~Profiler();
};

// ---------------------------------------------------------------- model base
struct Model {
    Runtime rt;
    Profiler prof;
    int64_t t = 0;  // step index of the current state
    int64_t block = 0, grid = 0, persistent = 1, digest_on = 0, metrics_cap = 4096;

    virtual ~Model() = default;
    virtual void step(int64_t n) = 0;
    virtual void synchronize() { AMBER_CUDA(cudaStreamSynchronize(rt.stream)); }
    virtual bool column_info(const char* name, amber_dtype* dt, int64_t* glen, int64_t* off,
                             int64_t* len) = 0;
    virtual void read_column(const char* name, void* dst, size_t bytes, bool on_dev) = 0;
    virtual void write_column(const char* name, const void* src, size_t bytes, bool on_dev) = 0;
    virtual void read_metrics(const char* name, void* dst, size_t bytes, int64_t* n_out) = 0;
    virtual void reset_metrics() = 0;
    virtual uint64_t digest(const char* name) = 0;
    virtual void set_step(int64_t s) = 0;
    virtual bool set_option(const char* key, int64_t v);
    virtual bool get_option(const char* key, int64_t* v);
};

// Factories (one per kind, defined in the kind's .cu file).
Model* make_wealth(int64_t n, const amber_wealth_params& p, uint64_t seed, const amber_runtime* rt);
Model* make_sir(int64_t n, const amber_sir_params& p, uint64_t seed, const amber_runtime* rt);
Model* make_boids(int64_t n, const amber_boids_params& p, uint64_t seed, const amber_runtime* rt);
Model* make_walk(int64_t n, const amber_walk_params& p, uint64_t seed, const amber_runtime* rt);
Model* make_sir_space(int64_t n, const amber_sir_space_params& p, uint64_t seed, const amber_runtime* rt);
void run_sweep(int64_t n, const amber_sir_params& base, const amber_replicate* reps,
               int64_t n_reps, int64_t n_steps, const amber_runtime* rt, double* out,
               amber_sweep_stats* stats);

// Generic Population (population.cu).
struct Population;
Population* make_population(const amber_column_spec* cols, int n, int64_t cap, uint64_t seed, const amber_runtime* rt);
void destroy_population(Population* p);
int64_t population_add(Population* p, int64_t n, const double* defaults);
void population_remove(Population* p, const int64_t* ids, int64_t n);
void population_compact(Population* p);
void population_size(Population* p, int64_t* live, int64_t* rows);
void population_update_paths(Population* p, int64_t* jit, int64_t* interp);
int64_t population_update(Population* p, const char* target, const amber_instr* e, int ne, const amber_instr* w, int nw,
                          bool want_count);
void population_synchronize(Population* p);
double population_aggregate(Population* p, int agg, const amber_instr* e, int ne, const amber_instr* w, int nw);
void population_read(Population* p, const char* name, void* dst, size_t bytes, bool on_dev);
void population_batch_set(Population* p, const char* name, const int64_t* ids, const double* vals, int64_t n);
void population_set_step(Population* p, int64_t s);

// Copy helper for column I/O (host or device endpoint), on the model stream.
void copy_out(Runtime& rt, void* dst, const void* src, size_t bytes, bool dst_on_dev);
void copy_in(Runtime& rt, void* dst, const void* src, size_t bytes, bool src_on_dev);

// Metric read helper: copy the valid window of a device ring (oldest first).
template <class T>
void read_ring(Runtime& rt, const T* ring, int64_t cap, int64_t first, int64_t end, void* dst,
               size_t bytes, int64_t* n_out);

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum_f64(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum of K 64-bit counters; thread 0 adds them atomically to out[k].
// All threads of the block must call it.  blockDim.x must be a multiple of 32.
template <int K>
__device__ __forceinline__ void block_sum_atomic(unsigned long long (&v)[K],
                                                 unsigned long long* const (&out)[K])
{
    __shared__ unsigned long long red[K][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        unsigned long long s = warp_sum_u64(v[k]);
        if (lane == 0) red[k][wid] = s;
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            unsigned long long s = lane < nw ? red[k][lane] : 0ull;
            s = warp_sum_u64(s);
            if (lane == 0 && out[k] && s) atomicAdd(out[k], s);
        }
    }
    __syncthreads();
}

// splitmix64 finaliser; D1 digest term for (id, 32-bit pattern).
__device__ __forceinline__ unsigned long long mix64(unsigned long long z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned long long digest_term(unsigned long long id, uint32_t bits)
{
    return mix64((id << 32) ^ (unsigned long long)bits);
}

// Digest of a 32-bit or 8-bit column (generic reduction kernel launcher).
uint64_t device_digest_u32(Runtime& rt, const uint32_t* col, int64_t n, int64_t id0);
uint64_t device_digest_u8(Runtime& rt, const uint8_t* col, int64_t n, int64_t id0);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Shard communicator for the sharded SIR (dist.cu): NCCL or loopback.
struct ShardComm;
ShardComm* make_shard_comm(Runtime& rt, const amber_runtime* r);
void destroy_shard_comm(ShardComm* c);
void shard_allgather_u32(ShardComm* c, Runtime& rt, const uint32_t* send, uint32_t* recv, size_t count);
void shard_allreduce_u64(ShardComm* c, Runtime& rt, unsigned long long* d, size_t n);
uint64_t shard_alltoallv(ShardComm* c, Runtime& rt, const void* send, const uint32_t* d_counts, size_t cap,
                         size_t elem, void* recv, size_t recv_cap);

// Multi-GPU partitions (host logic).  Wealth: contiguous id
// ranges of ceil(n/world) rounded up to 8 agents.  Sweep: replicate blocks.
inline void shard_range(int64_t n, int world, int rank, int64_t* lo, int64_t* hi)
{
    const int64_t shard = ((ceil_div(n, world) + 7) / 8) * 8;
    *lo = std::min<int64_t>(shard * rank, n);
    *hi = std::min<int64_t>(shard * (rank + 1), n);
}

// Sharded SIR (NEXT-3): contiguous id ranges of ceil(n/world) rounded up to 32
// agents (one I-bitmap word never spans two ranks).  shard = padded local size.
inline void sir_shard_range(int64_t n, int world, int rank, int64_t* lo, int64_t* len, int64_t* shard)
{
    *shard = ((ceil_div(n, world) + 31) / 32) * 32;
    *lo = std::min<int64_t>(*shard * rank, n);
    *len = std::min<int64_t>(*shard * (rank + 1), n) - *lo;
}

inline void sweep_range(int64_t n_reps, int world, int rank, int64_t* r0, int64_t* r1)
{
    const int64_t per = ceil_div(std::max<int64_t>(n_reps, 1), world);
    *r0 = std::min<int64_t>(per * rank, n_reps);
    *r1 = std::min<int64_t>(per * (rank + 1), n_reps);
}

}  // namespace amber

struct amber_model {
    amber::Model* impl;
};

struct amber_population {
    amber::Population* impl;
};
