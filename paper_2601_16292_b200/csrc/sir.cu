// sir.cu -- SIR on Erdos-Renyi contact graphs (Sec. 5.1.1,
// Listing 2, network environment Sec. 4.1;
// DESIGN.md G1-G4, S1-S6) and the batched replicate sweep (Sec. 4.2).
//
// Setup (not the hot path): a batched graph builder makes R independent
// G(n, M) graphs at once as one global CSR over R*n vertices (radix sorts of
// packed (replicate, min, max) keys, de-duplication, both arc directions,
// degree scan), and the K initial infected per replicate (segmented sort of
// the 64-bit init keys).
//
// Hot path: the per-step synchronous update.  Model (one replicate): each
// launch is one step, pull direction, one thread per 4 agents; or, with the
// "persistent" option, one cooperative launch runs all n steps with a grid
// barrier between steps.  Sweep: one CTA per replicate at a time (dynamic work
// queue), its graph, both state buffers and row offsets resident in shared
// memory for all steps, early exit once no agent is infected.
#include <cooperative_groups.h>

#include <algorithm>
#include <cub/cub.cuh>

#include "graph.cuh"
#include "internal.cuh"
#include "philox.cuh"

namespace cg = cooperative_groups;

namespace amber {

namespace {

constexpr uint8_t kS = 0, kI = 1, kR = 2, kPad = 3;

int bits_for(int64_t n)
{
    int b = 1;
    while ((1ll << b) < n) ++b;
    return b;
}

// ---------------------------------------------------------------- graph build
struct GraphBuildArgs {
    const unsigned long long* seeds;  // [R]
    int64_t R, n, m;
    int bn;  // bits per vertex id
};

// G2: e-th draw of replicate r -> packed key (r, min, max).
__global__ void er_keys_kernel(GraphBuildArgs a, unsigned long long* keys)
{
    const int64_t total = a.R * a.m;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = k / a.m, e = k - r * a.m;
        const PhiloxKey K = philox_key_dev(a.seeds[r]);
        const uint4 w = stream_block(K, TAG_GRAPH, static_cast<unsigned long long>(e), 0u);
        const unsigned long long xu = (static_cast<unsigned long long>(w.y) << 32) | w.x;
        const unsigned long long xv = (static_cast<unsigned long long>(w.w) << 32) | w.z;
        const unsigned long long u = mulhi64(xu, static_cast<unsigned long long>(a.n));
        unsigned long long v = mulhi64(xv, static_cast<unsigned long long>(a.n - 1));
        v += (v >= u);
        const unsigned long long lo = u < v ? u : v, hi = u < v ? v : u;
        keys[k] = (static_cast<unsigned long long>(r) << (2 * a.bn)) | (lo << a.bn) | hi;
    }
}

// G3: unique edges -> two arcs each (r, src, dst); duplicates -> sentinel.
__global__ void er_arcs_kernel(GraphBuildArgs a, const unsigned long long* keys, unsigned long long* arcs)
{
    const int64_t total = a.R * a.m;
    const unsigned long long mask = (1ull << a.bn) - 1;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[k];
        const bool uniq = (k == 0) || keys[k - 1] != key;
        if (uniq) {
            const unsigned long long r = key >> (2 * a.bn), lo = (key >> a.bn) & mask, hi = key & mask;
            arcs[2 * k] = (r << (2 * a.bn)) | (lo << a.bn) | hi;
            arcs[2 * k + 1] = (r << (2 * a.bn)) | (hi << a.bn) | lo;
        } else {
            arcs[2 * k] = ~0ull;
            arcs[2 * k + 1] = ~0ull;
        }
    }
}

// Degree count over the sorted valid arcs (vertex id = r*n + src), col fill.
__global__ void er_csr_kernel(GraphBuildArgs a, const unsigned long long* arcs, int64_t n_arcs, int* deg, int32_t* col)
{
    const unsigned long long mask = (1ull << a.bn) - 1;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_arcs; p += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = arcs[p];
        const unsigned long long r = key >> (2 * a.bn), src = (key >> a.bn) & mask, dst = key & mask;
        atomicAdd(deg + r * a.n + src, 1);
        col[p] = static_cast<int32_t>(dst);
    }
}

__global__ void count_valid_kernel(const unsigned long long* arcs, int64_t total, unsigned long long* n_valid)
{
    // arcs are sorted with sentinels last: find the first sentinel (binary search by one thread)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int64_t lo = 0, hi = total;
        while (lo < hi) {
            int64_t mid = (lo + hi) / 2;
            if (arcs[mid] == ~0ull) hi = mid;
            else lo = mid + 1;
        }
        *n_valid = static_cast<unsigned long long>(lo);
    }
}

// S1: init keys (64-bit lane of SIR_INIT, step 0) and ids per replicate.
__global__ void init_keys_kernel(const unsigned long long* seeds, int64_t R, int64_t n, unsigned long long* keys,
                                 int32_t* ids, uint32_t tag)
{
    const int64_t total = R * n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = k / n, i = k - r * n;
        const PhiloxKey K = philox_key_dev(seeds[r]);
        const uint4 w = stream_block(K, tag, static_cast<unsigned long long>(i / 2), 0u);
        keys[k] = lane64_of(w, static_cast<unsigned>(i & 1));
        ids[k] = static_cast<int32_t>(i);
    }
}

__global__ void init_state_kernel(const int32_t* sorted_ids, int64_t R, int64_t n, int64_t n_pad, int64_t k_inf,
                                  uint8_t* state)
{
    const int64_t total = R * n_pad;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = k % n_pad;
        state[k] = i < n ? kS : kPad;
    }
}

__global__ void init_mark_kernel(const int32_t* sorted_ids, int64_t R, int64_t n, int64_t n_pad, int64_t k_inf,
                                 uint8_t* state)
{
    const int64_t total = R * k_inf;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = k / k_inf, j = k - r * k_inf;
        state[r * n_pad + sorted_ids[r * n + j]] = kI;
    }
}

}  // namespace

void build_graphs(Runtime& rt, const std::vector<unsigned long long>& seeds, int64_t n, int64_t m, Graphs& g)
{
    const int64_t R = static_cast<int64_t>(seeds.size());
    AMBER_REQUIRE(n >= 2 && m >= 0, "graph needs n >= 2, M >= 0");
    const int bn = bits_for(n);
    const int br = R > 1 ? bits_for(R) : 0;
    AMBER_REQUIRE(2 * bn + br <= 64, "graph too large for packed 64-bit keys");
    AMBER_REQUIRE(R * 2 * m < (1ll << 31), "graph batch exceeds 2^31 arcs; use smaller batches");
    g.R = R;
    g.n = n;
    g.m = m;
    cudaStream_t s = rt.stream;
    DevBuf<unsigned long long> d_seeds, keys, keys2, arcs, arcs2, n_valid;
    DevBuf<int> deg;
    d_seeds.allocate(&rt, std::max<int64_t>(R, 1));
    AMBER_CUDA(cudaMemcpyAsync(d_seeds.p, seeds.data(), R * 8, cudaMemcpyHostToDevice, s));
    const int64_t total = R * m;
    GraphBuildArgs a{d_seeds.p, R, n, m, bn};
    const int grid = rt.num_sms * 8;
    keys.allocate(&rt, std::max<int64_t>(total, 1));
    keys2.allocate(&rt, std::max<int64_t>(total, 1));
    if (total) {
        er_keys_kernel<<<grid, 256, 0, s>>>(a, keys.p);
        check_launch("er_keys_kernel");
        size_t tmp = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.p, keys2.p, total, 0, 2 * bn + br, s);
        DevBuf<char> t;
        t.allocate(&rt, tmp + 16);
        AMBER_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, keys.p, keys2.p, total, 0, 2 * bn + br, s));
    }
    arcs.allocate(&rt, std::max<int64_t>(2 * total, 1));
    arcs2.allocate(&rt, std::max<int64_t>(2 * total, 1));
    n_valid.allocate(&rt, 1);
    n_valid.zero_async(s);
    if (total) {
        er_arcs_kernel<<<grid, 256, 0, s>>>(a, keys2.p, arcs.p);
        check_launch("er_arcs_kernel");
        keys.reset();
        keys2.reset();
        size_t tmp = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tmp, arcs.p, arcs2.p, 2 * total, 0, 64, s);
        DevBuf<char> t;
        t.allocate(&rt, tmp + 16);
        AMBER_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, arcs.p, arcs2.p, 2 * total, 0, 64, s));
        count_valid_kernel<<<1, 32, 0, s>>>(arcs2.p, 2 * total, n_valid.p);
        check_launch("count_valid_kernel");
    }
    unsigned long long nv = 0;
    AMBER_CUDA(cudaMemcpyAsync(&nv, n_valid.p, 8, cudaMemcpyDeviceToHost, s));
    AMBER_CUDA(cudaStreamSynchronize(s));
    g.arcs = static_cast<int64_t>(nv);
    deg.allocate(&rt, R * n + 1);
    deg.zero_async(s);
    g.col.allocate(&rt, std::max<int64_t>(g.arcs, 1) + 8);
    if (g.arcs) {
        er_csr_kernel<<<grid, 256, 0, s>>>(a, arcs2.p, g.arcs, deg.p, g.col.p);
        check_launch("er_csr_kernel");
    }
    g.row_ptr.allocate(&rt, R * n + 1);
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, deg.p, g.row_ptr.p, R * n + 1, s);
    DevBuf<char> t;
    t.allocate(&rt, tmp + 16);
    AMBER_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, deg.p, g.row_ptr.p, R * n + 1, s));
    AMBER_CUDA(cudaStreamSynchronize(s));
}

// S1: initial state for R replicates (row stride n_pad, padding = kPad).
void build_init_state(Runtime& rt, const std::vector<unsigned long long>& seeds, int64_t n, int64_t n_pad,
                      int64_t k_inf, uint8_t* state, uint32_t tag)
{
    const int64_t R = static_cast<int64_t>(seeds.size());
    cudaStream_t s = rt.stream;
    DevBuf<unsigned long long> d_seeds, keys, keys2;
    DevBuf<int32_t> ids, ids2;
    DevBuf<int> offsets;
    d_seeds.allocate(&rt, R);
    AMBER_CUDA(cudaMemcpyAsync(d_seeds.p, seeds.data(), R * 8, cudaMemcpyHostToDevice, s));
    keys.allocate(&rt, R * n);
    keys2.allocate(&rt, R * n);
    ids.allocate(&rt, R * n);
    ids2.allocate(&rt, R * n);
    const int grid = rt.num_sms * 8;
    init_keys_kernel<<<grid, 256, 0, s>>>(d_seeds.p, R, n, keys.p, ids.p, tag);
    check_launch("init_keys_kernel");
    std::vector<int> h_off(R + 1);
    for (int64_t r = 0; r <= R; ++r) h_off[r] = static_cast<int>(r * n);
    offsets.allocate(&rt, R + 1);
    AMBER_CUDA(cudaMemcpyAsync(offsets.p, h_off.data(), (R + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
    // stable by construction: equal keys keep ascending id order -> (key, id) order (S1)
    size_t tmp = 0;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp, keys.p, keys2.p, ids.p, ids2.p, R * n, R, offsets.p,
                                             offsets.p + 1, 0, 64, s);
    DevBuf<char> t;
    t.allocate(&rt, tmp + 16);
    AMBER_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(t.p, tmp, keys.p, keys2.p, ids.p, ids2.p, R * n, R,
                                                        offsets.p, offsets.p + 1, 0, 64, s));
    init_state_kernel<<<grid, 256, 0, s>>>(ids2.p, R, n, n_pad, k_inf, state);
    check_launch("init_state_kernel");
    if (k_inf > 0) {
        init_mark_kernel<<<grid, 256, 0, s>>>(ids2.p, R, n, n_pad, k_inf, state);
        check_launch("init_mark_kernel");
    }
    AMBER_CUDA(cudaStreamSynchronize(s));
}

namespace {

// ---------------------------------------------------------------- step kernel
struct SirSlot {
    unsigned long long S, I, R, digest;
};

struct SirStepArgs {
    PhiloxKey key;
    const int32_t* row_ptr;  // n + 1 (replicate-local offsets)
    const int32_t* col;
    uint8_t* x[2];           // ping-pong state (n_pad, padding = kPad)
    uint32_t* ib[2];         // ping-pong I bitmaps (n_pad / 32 words): bit i = [x_i == I]
    uint32_t* sb[2];         // ping-pong S bitmaps
    int64_t n, n_pad;        // agents of this shard (all agents unsharded), padded to 32
    unsigned long long gid0; // global id of local agent 0 (sharded: the shard start; else 0)
    unsigned long long t_beta, t_gamma;
    uint32_t t0;             // first step index
    int64_t n_steps;         // steps in this launch (persistent) or 1
    int cur;                 // index of the buffers holding the state at t0
    int prev_ok;             // ring slot t0 - 1 holds the counts of the state at t0
    const SirSlot* prev0;    // else (if set) the counts of the state at t0 are here
    SirSlot* ring;
    int64_t ring_cap;
    int digest;
    uint32_t* queue;         // persistent launch: [2 parities][2 phases][kRegions] chunk counters
    int grab;                // chunks per queue grab
    int dir;                 // 0: direction-optimizing; 1: pull only; 2: push whenever possible (tests, probes)
};

constexpr int kRegions = 16;
#ifndef AMBER_SIR_COL_LD
// column loads of the step walks: streamed (evict-first).  r02 V2 A/B
// (tools/v2_run.py): __ldcs 1.268 / __ldg 1.278 / __ldcg 1.277 / __ldca 1.28-1.37 ms/step
#define AMBER_SIR_COL_LD __ldcs
#endif
#ifndef AMBER_SIR_WALK_U
#define AMBER_SIR_WALK_U 4
#endif
constexpr int kWalkU = AMBER_SIR_WALK_U;  // 32-arc batches in flight per warp (walk_rows)
#ifndef AMBER_SIR_PT
#define AMBER_SIR_PT 256
#endif
constexpr int kSirPT = AMBER_SIR_PT;  // threads per block of the persistent kernel
#ifndef AMBER_SIR_MINB
// r02 C2 A/B (tools/c2_lib_probe.py): 2 / 3 / 4 / 6 blocks per SM 4.03 / 3.72 /
// 3.77 / 4.28 us/step -- kept at 4 (the 1% of 3 is within run-to-run spread)
#define AMBER_SIR_MINB (1024 / AMBER_SIR_PT)
#endif
constexpr int kSirMinB = AMBER_SIR_MINB;  // min resident blocks per SM (register cap 64 at 256 threads)
// 8 agents per lane (large populations): 5 blocks per SM (48 registers, a few
// spills) -- more warps to cover the random neighbour probes: V2 1.53 -> 1.42
// ms/step (6 blocks, 40 registers: 1.41 with 4x the spills)
#ifndef AMBER_SIR_MINB_LARGE
#define AMBER_SIR_MINB_LARGE 5
#endif
constexpr int kSirMinBLarge = AMBER_SIR_MINB_LARGE;

// Warp chunks of 32 * APL agents: lane L holds agents APL*L .. APL*L+APL-1 of
// the chunk (one load of its state bytes; for APL = 4 one Philox block serves
// the lane's four recovery draws, R4).  APL = 4 (128-agent chunks) for large
// populations, APL = 1 where latency rules (C2: more, shorter warp tasks).
// The state buffers and bitmaps are allocated to a multiple of kChunkMax
// agents (padding = kPad).  Persistent launch (queue != nullptr): dynamic --
// the chunk range is split into kRegions contiguous regions, warp w draws
// batches of `grab` chunks from region w % kRegions with one atomic
// (per-region counters, so the atomics spread); the pull and push walks cost
// very different amounts per chunk, and static striding left most warps
// waiting at the step barrier (r01 ncu: 43% of stall samples).  Per-step
// launch: one chunk per warp, the block scheduler balances.
constexpr int kChunkMax = 256;
constexpr int kQCap = 32 + kChunkMax;  // owner queue per warp: < 32 carried + one chunk

// 29 KB per block: the rest of the SM's 256 KB stays L1, which holds the CSR
// column sectors a walk revisits across its batches.  Measured (r02, V2): a
// 42 KB struct (12 KB more per block, L1 92 -> 28 KB at five blocks per SM)
// 1.31 -> 1.93 ms/step; a 21 KB one (two packed queue words, L1 124 KB) no
// change.
struct SirSmem {
    int32_t id[kSirPT / 32][kQCap];  // owner: agent offset (pull: in the chunk; push: local agent id)
    int32_t rb[kSirPT / 32][kQCap];  // owner's row [rb, re)
    int32_t re[kSirPT / 32][kQCap];
    uint32_t h[kSirPT / 32][kChunkMax / 32];  // pull: infected bits of the chunk's agents
};

__host__ __device__ constexpr int64_t sir_chunks(int64_t n_pad, int apl) { return (n_pad + 32 * apl - 1) / (32 * apl); }

// f(a0, next): next = the base of the chunk this warp processes after a0 when
// it is already known (-1 otherwise), so the body can prefetch its inputs.
template <int APL, class F>
__device__ __forceinline__ void for_chunks(const SirStepArgs& a, uint32_t* q, F&& f, int grab = 0)
{
    if (!grab) grab = a.grab;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t nchunks = sir_chunks(a.n_pad, APL);
    if (!q || nw < kRegions) {
        for (int64_t c = gw; c < nchunks; c += nw) f(c * 32 * APL, c + nw < nchunks ? (c + nw) * 32 * APL : -1);
        return;
    }
    const int r = static_cast<int>(gw % kRegions);
    const int64_t lo = nchunks * r / kRegions, hi = nchunks * (r + 1) / kRegions;
    for (;;) {
        uint32_t c0 = 0;
        if (lane == 0) c0 = atomicAdd(q + r, static_cast<uint32_t>(grab));
        c0 = __shfl_sync(0xffffffffu, c0, 0);
        if (lo + c0 >= hi) break;
        const int64_t e = lo + c0 + grab < hi ? lo + c0 + grab : hi;
        for (int64_t c = lo + c0; c < e; ++c) f(c * 32 * APL, c + 1 < e ? (c + 1) * 32 * APL : -1);
    }
}

__device__ __forceinline__ uint32_t* queue_of(const SirStepArgs& a, uint32_t t, int phase)
{
    return a.queue ? a.queue + ((t & 1u) * 2 + phase) * kRegions : nullptr;
}

// Relaxed (no-return) bitwise reductions: red.global.or / .and.
__device__ __forceinline__ void red_or(uint32_t* p, uint32_t v)
{
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_and(uint32_t* p, uint32_t v)
{
    asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Plain (coherent) load: the bitmaps are rewritten by earlier steps of the same
// persistent launch, so the read-only (.nc) path must not be used.
// The lookups are random over the whole bitmap (12.5 MB at N = 1e8), so they
// carry an L2 evict_last hint, and the streamed CSR columns an evict-first one,
// to keep the bitmaps L2-resident.
__device__ __forceinline__ bool bit_of(const uint32_t* bits, uint32_t j)
{
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    uint32_t w;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(w) : "l"(bits + (j >> 5)), "l"(pol));
    return (w >> (j & 31u)) & 1u;
}

// The lane's APL state bytes (agents i0 .. i0+APL-1) as one word.
template <int APL>
__device__ __forceinline__ void store_states(uint8_t* y, int64_t i0, unsigned long long v)
{
    if constexpr (APL == 8) *reinterpret_cast<unsigned long long*>(y + i0) = v;
    else if constexpr (APL == 4) *reinterpret_cast<uint32_t*>(y + i0) = static_cast<uint32_t>(v);
    else if constexpr (APL == 2) *reinterpret_cast<uint16_t*>(y + i0) = static_cast<uint16_t>(v);
    else y[i0] = static_cast<uint8_t>(v);
}

// The lane's APL bits (agents a0 + APL*lane + k) of a bitmap whose word 0
// holds agents a0 .. a0+31 (a0 a multiple of 32); the lanes of a word share
// one load.
template <int APL>
__device__ __forceinline__ uint32_t lane_bits(const uint32_t* w0)
{
    const int lane = threadIdx.x & 31;
    return (w0[(APL * lane) >> 5] >> ((APL * lane) & 31)) & ((1u << APL) - 1u);
}

// Bits of the lane's agents that are real (id < n); padding is neither S nor I.
template <int APL>
__device__ __forceinline__ uint32_t lane_real(int64_t i0, int64_t n)
{
    const int64_t r = n - i0;
    return r >= APL ? (1u << APL) - 1u : (r <= 0 ? 0u : (1u << r) - 1u);
}

// Recovery draws of the lane's agents i0 .. i0+APL-1 (global ids; i0 is a
// multiple of APL): lane i & 3 of Philox block i / 4 (R4) -- one block per
// four agents of the lane when APL >= 4.  Bit k set iff agent i0 + k is in `inf`
// and recovers.
template <int APL>
__device__ __forceinline__ uint32_t recover_nib(const SirStepArgs& a, unsigned long long i0, uint32_t t, uint32_t inf)
{
    uint32_t out = 0;
#pragma unroll
    for (int b = 0; b < (APL + 3) / 4; ++b) {
        const uint32_t part = (inf >> (4 * b)) & 0xfu;
        if (!part) continue;
        const uint4 r = stream_block(a.key, TAG_SIR_REC, (i0 >> 2) + b, t);
        const uint32_t d[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int k = 4 * b; k < APL && k < 4 * b + 4; ++k) {
            const uint32_t q = static_cast<uint32_t>((i0 + k) & 3u);
            const uint32_t v = q == 0 ? d[0] : (q == 1 ? d[1] : (q == 2 ? d[2] : d[3]));
            if (((inf >> k) & 1u) && v < a.t_gamma) out |= 1u << k;
        }
    }
    return out;
}

// recover_nib for APL = 8 with the warp's Philox blocks compacted: the lanes'
// 4-agent groups holding an infected agent are listed in shared memory (ids /
// infected nibbles, scratch rb / re of the warp's queue slot, which the push
// queue does not use) and drawn 32 per round, one block per lane, instead of
// every lane running both of its blocks whenever any lane of the warp needs
// one (SIMT).  Same draws (R4: word i & 3 of block i / 4).  Push steps with
// sparse infected sets: V2 r02 ncu, recovery draws ~1/6 of a push step's
// instructions.  i0: the lane's first global id (a multiple of 8).
__device__ __forceinline__ uint32_t recover_nib8_compact(const SirStepArgs& a, unsigned long long i0, uint32_t t,
                                                         uint32_t inf, int32_t* ids, int32_t* res)
{
    const int lane = threadIdx.x & 31;
    const uint32_t p0 = inf & 0xfu, p1 = (inf >> 4) & 0xfu;
    const uint32_t m0 = __ballot_sync(0xffffffffu, p0 != 0), m1 = __ballot_sync(0xffffffffu, p1 != 0);
    const uint32_t c0 = __popc(m0), cnt = c0 + __popc(m1);
    if (!cnt) return 0u;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t r0 = __popc(m0 & lt), r1 = c0 + __popc(m1 & lt);
    const int32_t g = static_cast<int32_t>(i0 >> 2);
    if (p0) { ids[r0] = g; res[r0] = static_cast<int32_t>(p0); }
    if (p1) { ids[r1] = g + 1; res[r1] = static_cast<int32_t>(p1); }
    __syncwarp();
    for (uint32_t k = lane; k < cnt; k += 32) {
        const uint32_t part = static_cast<uint32_t>(res[k]);
        const uint4 r = stream_block(a.key, TAG_SIR_REC, static_cast<unsigned long long>(static_cast<uint32_t>(ids[k])), t);
        uint32_t out = 0;
        if ((part & 1u) && r.x < a.t_gamma) out |= 1u;
        if ((part & 2u) && r.y < a.t_gamma) out |= 2u;
        if ((part & 4u) && r.z < a.t_gamma) out |= 4u;
        if ((part & 8u) && r.w < a.t_gamma) out |= 8u;
        res[k] = static_cast<int32_t>(out);
    }
    __syncwarp();
    const uint32_t out = (p0 ? static_cast<uint32_t>(res[r0]) : 0u) | ((p1 ? static_cast<uint32_t>(res[r1]) : 0u) << 4);
    __syncwarp();  // the scratch is rewritten by the next chunk
    return out;
}

// Bit k of m (k < 4) -> byte k (0 or 1) of a 32-bit word.
static_assert(kS == 0 && kI == 1 && kR == 2, "the byte-parallel state deltas assume these codes");
__device__ __forceinline__ uint32_t spread4(uint32_t m) { return ((m & 0xfu) * 0x00204081u) & 0x01010101u; }

// Exclusive warp prefix sum; *total = the warp's sum.
__device__ __forceinline__ uint32_t warp_excl(uint32_t v, uint32_t* total)
{
    const int lane = threadIdx.x & 31;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    *total = __shfl_sync(0xffffffffu, incl, 31);
    return incl - v;
}

// Bitmap word of the lane's agents from the lanes' APL-bit nibbles: lanes
// g*(32/APL) .. (g+1)*(32/APL)-1 hold the 32 agents of word g of the chunk;
// every lane of the group gets the word.
template <int APL>
__device__ __forceinline__ uint32_t word_of(uint32_t nib)
{
    if constexpr (APL == 1) return __ballot_sync(0xffffffffu, nib & 1u);
    constexpr int G = 32 / APL;  // lanes per word
    uint32_t v = nib << ((threadIdx.x & (G - 1)) * APL);
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Appends the lane's agents in `nib` (ids id_base + k) with their CSR rows
// (kRows; else the ids only) to the warp's owner queue at qn + rank; returns
// the number the warp appended.
template <int APL, bool kRows = true>
__device__ __forceinline__ uint32_t queue_owners(SirSmem& sm, uint32_t qn, uint32_t nib, int32_t id_base,
                                                 const int32_t* r = nullptr)
{
    const int wq = threadIdx.x >> 5;
    uint32_t T;
    uint32_t k = qn + warp_excl(__popc(nib), &T);
    if (!kRows) {
        for (uint32_t m = nib; m; m &= m - 1u) sm.id[wq][k++] = id_base + __ffs(static_cast<int>(m)) - 1;
        return T;
    }
    if (nib) {
#pragma unroll
        for (int q = 0; q < APL; ++q)
            if ((nib >> q) & 1u) {
                sm.id[wq][k] = id_base + q;
                sm.rb[wq][k] = r[q];
                sm.re[wq][k] = r[q + 1];
                ++k;
            }
    }
    return T;
}

// Inputs of a pull chunk: the lane's S and I bitmap words (L2) and its CSR
// row offsets (HBM), all issued together.  (Loading them one chunk ahead
// through for_chunks' `next` measured slower: register spills at 64.)
template <int APL>
struct PullIn {
    uint32_t ws, wi;
    int32_t r[APL + 1];
};

template <int APL>
__device__ __forceinline__ void pull_load(const SirStepArgs& a, int64_t a0, const uint32_t* sb, const uint32_t* ib,
                                          PullIn<APL>& p)
{
    const int lane = threadIdx.x & 31;
    const int64_t i0 = a0 + APL * lane;
    p.ws = sb[(a0 >> 5) + ((APL * lane) >> 5)];
    p.wi = ib[((a.gid0 + static_cast<unsigned long long>(a0)) >> 5) + ((APL * lane) >> 5)];
    if constexpr (APL == 4) {
        if (i0 + 4 <= a.n) {
            const int4 v = *reinterpret_cast<const int4*>(a.row_ptr + i0);
            p.r[0] = v.x;
            p.r[1] = v.y;
            p.r[2] = v.z;
            p.r[3] = v.w;
            p.r[4] = a.row_ptr[i0 + 4];
            return;
        }
    }
#pragma unroll
    for (int q = 0; q <= APL; ++q) p.r[q] = i0 + q <= a.n ? a.row_ptr[i0 + q] : 0;
}

// Pull step for the 32 * APL agents of chunk a0: the susceptible agents,
// compacted into groups of 32 owners, walk their rows warp-cooperatively; an
// arc transmits iff the neighbour is I (bitmap, L2-resident) and the
// pair-keyed Bernoulli (S3) fires.  Writes the next state and the next bitmap
// words and adds the S/I/R counts (and digest terms) of the new states to cnt.
template <int APL>
__device__ __forceinline__ void sir_pull_chunk(const SirStepArgs& a, int64_t a0, const PullIn<APL>& in,
                                               uint8_t* __restrict__ y, const uint32_t* __restrict__ ib,
                                               uint32_t* __restrict__ ib_next, uint32_t* __restrict__ sb_next,
                                               uint32_t t, SirSmem& sm, unsigned long long (&cnt)[4])
{
    constexpr uint32_t kM = (1u << APL) - 1u;
    const int lane = threadIdx.x & 31;
    const int wq = threadIdx.x >> 5;
    const int64_t i0 = a0 + APL * lane;
    // the current state from the bitmaps (L2-resident; the state bytes are
    // only written): own I bits from the global I bitmap (sharded: ib is
    // global, gid0 a multiple of 32), S bits from the local S bitmap
    // (sharded: a chunk may reach past the shard into the next rank's bits)
    const uint32_t real = lane_real<APL>(i0, a.n);
    const uint32_t nib_s = (in.ws >> ((APL * lane) & 31)) & kM & real;
    const uint32_t nib_i = (in.wi >> ((APL * lane) & 31)) & kM & real;
    uint32_t hitnib = 0;
    if (__any_sync(0xffffffffu, nib_s != 0)) {
        if (lane < APL) sm.h[wq][lane] = 0u;
        const uint32_t T = queue_owners<APL>(sm, 0, nib_s, APL * lane, in.r);
        __syncwarp();
        for (uint32_t g0 = 0; g0 < T; g0 += 32) {
            const uint32_t nown = T - g0 < 32 ? T - g0 : 32;
            const bool mine = static_cast<uint32_t>(lane) < nown;
            const int32_t lid = mine ? sm.id[wq][g0 + lane] : 0;
            const int32_t rb = mine ? sm.rb[wq][g0 + lane] : 0, re = mine ? sm.re[wq][g0 + lane] : 0;
            const uint32_t own = nown >= 32 ? 0xffffffffu : ((1u << nown) - 1u);
            const uint32_t sid = static_cast<uint32_t>(a.gid0 + static_cast<unsigned long long>(a0 + lid));
            const uint32_t hit = walk_rows_pay<kWalkU, APL == 8>(
                [&](int32_t e) {
                    AMBER_DCHECK(e >= 0 && e < a.row_ptr[a.n], "SIR pull: arc index out of the CSR");
                    return static_cast<uint32_t>(AMBER_SIR_COL_LD(a.col + e));
                }, own, rb, re, sid,
                [&](uint32_t j) { return static_cast<uint32_t>(bit_of(ib, j)); },  // j: global id (global bitmap)
                [&](uint32_t j, int32_t, int, uint32_t s) {
                    const uint4 w = philox(make_uint4(min(s, j), max(s, j), t, TAG_SIR_TX), a.key);
                    return static_cast<unsigned long long>(w.x) < a.t_beta;
                });
            if ((hit >> lane) & 1u) atomicOr(&sm.h[wq][lid >> 5], 1u << (lid & 31));
        }
        __syncwarp();
        hitnib = (sm.h[wq][(APL * lane) >> 5] >> ((APL * lane) & 31)) & kM;
        __syncwarp();  // the next chunk rewrites the queue and h
    }
    const uint32_t recnib = recover_nib<APL>(a, a.gid0 + static_cast<unsigned long long>(i0), t, nib_i);
    const uint32_t s2 = nib_s & ~hitnib, i2 = (nib_s & hitnib) | (nib_i & ~recnib), r2 = real & ~s2 & ~i2;
    unsigned long long yw = 0;
#pragma unroll
    for (int k = 0; k < APL; ++k) {
        const unsigned long long st = (s2 >> k) & 1u ? kS : ((i2 >> k) & 1u ? kI : ((r2 >> k) & 1u ? kR : kPad));
        yw |= st << (8 * k);
    }
    store_states<APL>(y, i0, yw);
    const uint32_t wi = word_of<APL>(i2), ws = word_of<APL>(s2);
    if ((lane & (32 / APL - 1)) == 0) {
        ib_next[(a0 >> 5) + lane / (32 / APL)] = wi;
        sb_next[(a0 >> 5) + lane / (32 / APL)] = ws;
    }
    // pads (kPad) are in none of the nibbles
    cnt[0] += __popc(s2);
    cnt[1] += __popc(i2);
    cnt[2] += __popc(r2);
    if (a.digest) {
#pragma unroll
        for (int k = 0; k < APL; ++k)
            if (i0 + k < a.n) cnt[3] += digest_term(a.gid0 + static_cast<unsigned long long>(i0 + k), (yw >> (8 * k)) & 0xffu);
    }
}

template <int APL>
__device__ __forceinline__ void sir_pull_body(const SirStepArgs& a, int c, uint32_t t, SirSmem& sm,
                                              unsigned long long (&cnt)[4])
{
    for_chunks<APL>(a, queue_of(a, t, 0), [&](int64_t a0, int64_t) {
        PullIn<APL> in;
        pull_load<APL>(a, a0, a.sb[c], a.ib[c], in);
        sir_pull_chunk<APL>(a, a0, in, a.x[c ^ 1], a.ib[c], a.ib[c ^ 1], a.sb[c ^ 1], t, sm, cnt);
    });
}

template <int APL>
__global__ void __launch_bounds__(256) sir_step_kernel(const SirStepArgs a)
{
    __shared__ SirSmem sm;
    const uint32_t t = a.t0;
    unsigned long long cnt[4] = {0, 0, 0, 0};
    sir_pull_body<APL>(a, a.cur, t, sm, cnt);
    SirSlot* sl = a.ring + (t % a.ring_cap);
    unsigned long long* const outs[4] = {&sl->S, &sl->I, &sl->R, a.digest ? &sl->digest : nullptr};
    block_sum_atomic<4>(cnt, outs);
}

// Bitmaps of a state buffer (after creation or an external column write).
__global__ void sir_bits_kernel(const uint8_t* __restrict__ x, int64_t n_pad, uint32_t* __restrict__ ib,
                                uint32_t* __restrict__ sb)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t a0 = gw * 32; a0 < n_pad; a0 += nw * 32) {
        const uint8_t st = x[a0 + lane];
        const uint32_t iw = __ballot_sync(0xffffffffu, st == kI), sw = __ballot_sync(0xffffffffu, st == kS);
        if (lane == 0) {
            ib[a0 >> 5] = iw;
            sb[a0 >> 5] = sw;
        }
    }
}

// Push step (infected < susceptible).  Invariant of the back buffers
// (x, ib, sb)[c ^ 1]: they hold a state B from which the current state is
// reached by S -> I -> R moves only (the previous step's input; a copy of the
// current state after creation or a column write), so every agent that is S
// now is S in B.  One pass, no copy:
//  * owners of non-S agents write their new states into y (bytes of B) as one
//    atomic delta on the lane's word, and XOR-correct their bits of the next I
//    bitmap (B's bits -> survivors) and clear their S bits -- all on bits and
//    bytes no pusher touches (pushers only touch agents that are S now);
//  * every agent infected now pushes along its row to neighbours that are S
//    now (S bitmap) with the same pair-keyed draw as pull (S3); a transmitting
//    arc sets the neighbour's next I bit with atomicOr, whose old word makes
//    the new-infection count exact when several pushers hit the same agent;
//    the first one also clears its S bit and sets its byte to I.
// Pushers are compacted across chunks into the warp's owner queue and walked
// 32 owners at a time, so the concatenated rows fill the walk's 32-arc batches
// even when few agents are infected.
template <int APL>
__device__ __forceinline__ void sir_push_body(const SirStepArgs& a, int c, uint32_t t, SirSmem& sm, long long& rec,
                                              long long& inf, unsigned long long& dig)
{
    const int lane = threadIdx.x & 31;
    const int wq = threadIdx.x >> 5;
    const uint32_t* __restrict__ ib = a.ib[c];
    const uint32_t* __restrict__ sb = a.sb[c];
    uint32_t* ib_next = a.ib[c ^ 1];
    uint32_t* sb_next = a.sb[c ^ 1];
    uint8_t* y = a.x[c ^ 1];
    uint32_t* yw = reinterpret_cast<uint32_t*>(y);
    uint32_t qn = 0;  // queued pushers (warp-uniform; < 32 between chunks)
    auto walk = [&](uint32_t g0, uint32_t nown) {
        // rows are loaded here, 32 owners at a time, not per chunk: one row_ptr
        // round trip per walk instead of one per chunk with an infected agent
        const bool mine = static_cast<uint32_t>(lane) < nown;
        const uint32_t id = mine ? static_cast<uint32_t>(sm.id[wq][g0 + lane]) : 0u;
        const int32_t rb = mine ? a.row_ptr[id] : 0, re = mine ? a.row_ptr[id + 1] : 0;
        const uint32_t own = nown >= 32 ? 0xffffffffu : ((1u << nown) - 1u);
        walk_rows_pay<kWalkU, APL == 8>([&](int32_t e) {
                                  AMBER_DCHECK(e >= 0 && e < a.row_ptr[a.n], "SIR push: arc index out of the CSR");
                                  return static_cast<uint32_t>(AMBER_SIR_COL_LD(a.col + e));
                              }, own, rb, re, id,
                              [&](uint32_t j) {
                                  AMBER_DCHECK(j < static_cast<uint64_t>(a.n), "SIR push: neighbour id >= n");
                                  return static_cast<uint32_t>(bit_of(sb, j));
                              },
                              [&](uint32_t j, int32_t, int, uint32_t s) {
            const uint4 wd = philox(make_uint4(min(s, j), max(s, j), t, TAG_SIR_TX), a.key);
            if (static_cast<unsigned long long>(wd.x) < a.t_beta) {
                const uint32_t bit = 1u << (j & 31u);
                if (a.digest || APL != 8) {  // the old word dedups the digest delta and the count
                    const uint32_t prev = atomicOr(ib_next + (j >> 5), bit);
                    if (!(prev & bit)) {
                        atomicAnd(sb_next + (j >> 5), ~bit);
                        atomicOr(yw + (j >> 2), static_cast<uint32_t>(kI) << ((j & 3u) * 8u));
                        ++inf;
                        dig += digest_term(j, kI) - digest_term(j, kS);
                    }
                } else {
                    // large populations: three idempotent REDs, no returned word to
                    // wait for (r02 ncu: the returning atomicOr held 10% of the V2
                    // stall samples); the new infections are counted after the step
                    // (sir_count_new: one bitmap pass + one grid barrier, V2 1.42 ->
                    // 1.35 ms/step).  Small ones keep the inline count: at C2 the
                    // extra barrier per push step costs more (4.98 -> 6.8 us/step).
                    red_or(ib_next + (j >> 5), bit);
                    red_and(sb_next + (j >> 5), ~bit);
                    red_or(yw + (j >> 2), static_cast<uint32_t>(kI) << ((j & 3u) * 8u));
                }
            }
            return false;  // an infected agent tries every susceptible neighbour
        });
    };
    // moves the queue remainder (< 32) to the front after walking full groups
    auto drain = [&]() {
        uint32_t g0 = 0;
        for (; qn - g0 >= 32; g0 += 32) walk(g0, 32);
        const uint32_t rem = qn - g0;
        int32_t vi = 0;
        if (static_cast<uint32_t>(lane) < rem) vi = sm.id[wq][g0 + lane];
        __syncwarp();
        if (static_cast<uint32_t>(lane) < rem) sm.id[wq][lane] = vi;
        __syncwarp();
        qn = rem;
    };
    if (APL == 8 && !a.digest) {
        // Large populations: the chunk pass one bitmap word (32 agents) per
        // lane, 1,024 agents per warp chunk -- the per-chunk warp work (loads,
        // ballots, scans, queue bookkeeping) amortised over 4x the agents of
        // the 8-agents-per-lane pass below (r02 ncu, V2 push steps at 1-5%
        // infected: ~300 warp instructions per 256-agent chunk, 40% of the step).
        // Same draws and the same state / bitmap updates (tests: forced push
        // at 8 agents per lane, digest off).
        const int64_t words = a.n_pad >> 5;
        for_chunks<32>(a, queue_of(a, t, 1), [&](int64_t a0, int64_t) {
            const int64_t w = (a0 >> 5) + lane;
            const bool ok = w < words;
            const uint32_t Ws = ok ? sb[w] : 0u, Wi = ok ? ib[w] : 0u;
            const uint32_t Wbs = ok ? sb_next[w] : 0u, Wbi = ok ? ib_next[w] : 0u;
            const int64_t left = a.n - 32 * w;
            const uint32_t real = !ok || left <= 0 ? 0u : (left >= 32 ? 0xffffffffu : (1u << left) - 1u);
            const uint32_t nons = real & ~Ws;
            if (!__any_sync(0xffffffffu, nons != 0)) return;
            const uint32_t inf_now = Wi & real;
            // recoveries (R4: word i & 3 of block i / 4): the 4-agent groups
            // holding an infected agent, compacted over the warp (queue words
            // rb / re as scratch), drawn 32 per round
            uint32_t x = inf_now | (inf_now >> 1);
            x = (x | (x >> 2)) & 0x11111111u;
            x = (x | (x >> 3)) & 0x03030303u;
            x = (x | (x >> 6)) & 0x000f000fu;
            const uint32_t gm = (x | (x >> 12)) & 0xffu;  // bit g: group g of the word has an infected agent
            uint32_t T;
            const uint32_t off = warp_excl(__popc(gm), &T);
            uint32_t recw = 0;
            if (T) {
                uint32_t k = off;
                for (uint32_t m = gm; m; m &= m - 1u, ++k) {
                    const int g = __ffs(static_cast<int>(m)) - 1;
                    sm.rb[wq][k] = static_cast<int32_t>(8 * w + g);
                    sm.re[wq][k] = static_cast<int32_t>((inf_now >> (4 * g)) & 0xfu);
                }
                __syncwarp();
                for (uint32_t e = lane; e < T; e += 32) {
                    const uint32_t part = static_cast<uint32_t>(sm.re[wq][e]);
                    const uint4 r = stream_block(a.key, TAG_SIR_REC,
                                                 static_cast<unsigned long long>(static_cast<uint32_t>(sm.rb[wq][e])), t);
                    uint32_t o = 0;
                    if ((part & 1u) && r.x < a.t_gamma) o |= 1u;
                    if ((part & 2u) && r.y < a.t_gamma) o |= 2u;
                    if ((part & 4u) && r.z < a.t_gamma) o |= 4u;
                    if ((part & 8u) && r.w < a.t_gamma) o |= 8u;
                    sm.re[wq][e] = static_cast<int32_t>(o);
                }
                __syncwarp();
                k = off;
                for (uint32_t m = gm; m; m &= m - 1u, ++k)
                    recw |= static_cast<uint32_t>(sm.re[wq][k]) << (4 * (__ffs(static_cast<int>(m)) - 1));
                __syncwarp();  // the scratch is rewritten by the next chunk
            }
            rec += __popc(recw);
            const uint32_t surv = inf_now & ~recw;
            if (ok && nons) {
                // state bytes of the agents whose next state differs from B's
                // (new: I survivors and R; B: S, I or R), one delta per 4-agent word
                const uint32_t chg = nons & (Wbs | (Wbi & ~surv));
                uint32_t cg = chg | (chg >> 1);
                cg = (cg | (cg >> 2)) & 0x11111111u;
                cg = (cg | (cg >> 3)) & 0x03030303u;
                cg = (cg | (cg >> 6)) & 0x000f000fu;
                cg = (cg | (cg >> 12)) & 0xffu;
                const uint32_t oi = ~Wbs & Wbi, orr = ~Wbs & ~Wbi;
                for (uint32_t m = cg; m; m &= m - 1u) {
                    const int g = __ffs(static_cast<int>(m)) - 1;
                    const uint32_t c4 = chg >> (4 * g);
                    const uint32_t nw = spread4(c4 & (surv >> (4 * g))) + 2u * spread4(c4 & ~(surv >> (4 * g)));
                    const uint32_t old = spread4(c4 & (oi >> (4 * g))) + 2u * spread4(c4 & (orr >> (4 * g)));
                    atomicAdd(yw + 8 * w + g, nw - old);
                }
                // B's bits of the non-S agents -> survivors / cleared S
                const uint32_t flip = (Wbi ^ surv) & nons;
                if (flip) atomicXor(ib_next + w, flip);
                if (Wbs & nons) atomicAnd(sb_next + w, ~nons);
            }
            // pushers: queued in rounds of at most 8 per lane (queue capacity:
            // < 32 carried + 256), walked whenever 32 are queued
            uint32_t m = inf_now;
            while (__any_sync(0xffffffffu, m != 0)) {
                const uint32_t cnt = min(__popc(m), 8);
                uint32_t tot;
                uint32_t k = qn + warp_excl(cnt, &tot);
                for (uint32_t i = 0; i < cnt; ++i, m &= m - 1u)
                    sm.id[wq][k++] = static_cast<int32_t>(32 * w + __ffs(static_cast<int>(m)) - 1);
                qn += tot;
                __syncwarp();
                if (qn >= 32) drain();
            }
        }, a.grab > 4 ? a.grab / 4 : 1);
        if (qn) walk(0, qn);
        return;
    }
    for_chunks<APL>(a, queue_of(a, t, 1), [&](int64_t a0, int64_t) {
        const int64_t i0 = a0 + APL * lane;
        // current state and back state B from the bitmaps (L2-resident, four
        // independent loads): no state byte is read.  B's bits of a non-S agent
        // are only changed by this lane (pushers touch agents that are S now).
        constexpr uint32_t kM = (1u << APL) - 1u;
        const int64_t wl = (a0 >> 5) + ((APL * lane) >> 5);  // the lane's bitmap word
        const uint32_t sh = (APL * lane) & 31;
        const uint32_t Ws = sb[wl], Wi = ib[wl], Wbs = sb_next[wl], Wbi = ib_next[wl];
        const uint32_t nib_s = (Ws >> sh) & kM, nib_i = (Wi >> sh) & kM;
        const uint32_t b_s = (Wbs >> sh) & kM, b_i = (Wbi >> sh) & kM;
        const uint32_t nons = lane_real<APL>(i0, a.n) & ~nib_s;
        if (a.digest && nib_s) {
#pragma unroll
            for (int k = 0; k < APL; ++k)
                if ((nib_s >> k) & 1u) dig += digest_term(static_cast<unsigned long long>(i0 + k), kS);
        }
        if (!__any_sync(0xffffffffu, nons != 0)) return;
        // owners: recoveries and the new state of every non-S agent
        uint32_t recnib;
        if constexpr (APL == 8) recnib = recover_nib8_compact(a, static_cast<unsigned long long>(i0), t, nib_i, sm.rb[wq], sm.re[wq]);
        else recnib = recover_nib<APL>(a, static_cast<unsigned long long>(i0), t, nib_i);
        rec += __popc(recnib);
        if (APL == 8 && !a.digest) {
            // the same per-word deltas as below, byte-parallel: bit k of a
            // nibble -> byte k; codes S 0, I 1, R 2
            if (nons) {
                const uint32_t surv = nib_i & ~recnib;
                const uint32_t oi = nons & ~b_s & b_i, orr = nons & ~b_s & ~b_i;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t nw = spread4((nons & surv) >> (4 * h)) + 2u * spread4((nons & ~surv) >> (4 * h));
                    const uint32_t old = spread4(oi >> (4 * h)) + 2u * spread4(orr >> (4 * h));
                    if (nw != old) atomicAdd(yw + (i0 >> 2) + h, nw - old);
                }
            }
        } else if (nons) {
            // the lane's bytes sit in one 32-bit word (two for APL 8; i0 is a
            // multiple of APL).  One signed delta per 32-bit word, applied with a
            // 32-bit atomicAdd: exact mod 2^32 because every byte starts and ends
            // in 0..3, and the same access size as the pushers' atomicOr on
            // these words (no partially overlapping atomics).
            constexpr int kW = APL == 8 ? 2 : 1;
            uint32_t delta[kW] = {};
#pragma unroll
            for (int k = 0; k < APL; ++k)
                if ((nons >> k) & 1u) {
                    const uint32_t nw = ((nib_i & ~recnib) >> k) & 1u ? kI : kR;
                    const uint32_t old = (b_s >> k) & 1u ? kS : ((b_i >> k) & 1u ? kI : kR);
                    delta[k >> 2] += (nw - old) << (8 * (k & 3));
                    if (a.digest) dig += digest_term(static_cast<unsigned long long>(i0 + k), nw);
                }
            if constexpr (APL == 8) {
                if (delta[0]) atomicAdd(yw + (i0 >> 2), delta[0]);
                if (delta[1]) atomicAdd(yw + (i0 >> 2) + 1, delta[1]);
            } else if (delta[0]) {
                const uint32_t sh0 = static_cast<uint32_t>(i0 & 3) * 8u;
                atomicAdd(yw + (i0 >> 2), delta[0] << sh0);
            }
        }
        const uint32_t wsurv = word_of<APL>(nib_i & ~recnib), wnons = word_of<APL>(nons);
        // B's bits of the non-S agents -> survivors / cleared S (B's words
        // as loaded above: exact on the non-S bits, which only this group changes)
        if ((lane & (32 / APL - 1)) == 0 && wnons) {
            const uint32_t flip = (Wbi ^ wsurv) & wnons;
            if (flip) atomicXor(ib_next + wl, flip);
            if (Wbs & wnons) atomicAnd(sb_next + wl, ~wnons);
        }
        // pushers: queue, walk whenever 32 are queued
        if (!__any_sync(0xffffffffu, nib_i != 0)) return;
        qn += queue_owners<APL, false>(sm, qn, nib_i, static_cast<int32_t>(i0));
        __syncwarp();
        if (qn >= 32) drain();
    });
    if (qn) walk(0, qn);
}

// New infections of a push step that did not count them (no digest): agents S
// before it (back buffer sb) and I after it (current ib), summed over the grid
// into that step's ring slot (S -= new, I += new).  After a grid barrier.
__device__ __forceinline__ void sir_count_new(const SirStepArgs& a, int cur, SirSlot* slot)
{
    const uint32_t* sb_prev = a.sb[cur ^ 1];
    const uint32_t* ib_now = a.ib[cur];
    const int64_t words = a.n_pad / 32;
    unsigned long long c = 0;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
        c += __popc(__ldcg(sb_prev + w) & __ldcg(ib_now + w));
    unsigned long long v[2] = {0ull - c, c};
    unsigned long long* const outs[2] = {&slot->S, &slot->I};
    block_sum_atomic<2>(v, outs);
}

// The identity steps at the end of an epidemic (sir_persistent_kernel): records
// of the `rem` remaining steps repeat the current counts; an odd remainder
// copies the state to the other buffer set.  Out of line, so the step loop's
// register allocation does not carry it (inlined, it added spills to every
// variant).
__device__ __noinline__ void sir_identity_tail(SirSlot* ring, int64_t cap, const SirSlot* pv, uint32_t t, int64_t rem,
                                               int digest, const uint8_t* x, uint8_t* y, const uint32_t* ib,
                                               uint32_t* ib_o, const uint32_t* sb, uint32_t* sb_o, int64_t n_pad)
{
    const SirSlot v{pv->S, 0ull, pv->R, digest ? pv->digest : 0ull};
    if (blockIdx.x == 0)  // rem <= ring_cap - 1: slot t - 1 is not overwritten
        for (int64_t j = threadIdx.x; j < rem; j += blockDim.x) ring[(t + j) % cap] = v;
    if (rem & 1) {
        const int64_t g0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        const int64_t gs = static_cast<int64_t>(gridDim.x) * blockDim.x;
        const uint32_t* xs = reinterpret_cast<const uint32_t*>(x);
        uint32_t* xd = reinterpret_cast<uint32_t*>(y);
        for (int64_t i = g0; i < n_pad / 4; i += gs) xd[i] = xs[i];
        for (int64_t w = g0; w < n_pad / 32; w += gs) {
            ib_o[w] = ib[w];
            sb_o[w] = sb[w];
        }
    }
}

// All n_steps steps in one cooperative launch (grid barrier between steps).
// Direction-optimizing: step k pushes from the infected agents when they are
// fewer than 3/4 of the susceptible ones (counts of the previous step from its ring
// slot, so every block takes the same decision), otherwise it pulls.  Both
// directions give identical results (S3); the tests check it.
template <int APL>
__global__ void __launch_bounds__(kSirPT, APL == 8 ? kSirMinBLarge : kSirMinB) sir_persistent_kernel(const SirStepArgs a)
{
    __shared__ SirSmem sm;
    cg::grid_group grid = cg::this_grid();
    int cur = a.cur;
    bool uncounted = false;  // the previous step of this launch pushed without counting its new infections
    for (int64_t k = 0; k < a.n_steps; ++k) {
        const uint32_t t = a.t0 + static_cast<uint32_t>(k);
        SirSlot* sl = a.ring + (t % a.ring_cap);
        if (uncounted) {  // complete slot t-1 before anyone reads it
            sir_count_new(a, cur, a.ring + ((t + a.ring_cap - 1) % a.ring_cap));
            grid.sync();
        }
        // the counters of step t+1 were last used by step t-1 (finished at the previous barrier)
        if (a.queue && blockIdx.x == 0 && threadIdx.x < 2 * kRegions) a.queue[((t + 1) & 1u) * 2 * kRegions + threadIdx.x] = 0u;
        bool push = false;
        unsigned long long prev_s = 0, prev_i = 0, prev_r = 0;
        if (k > 0 || a.prev_ok || a.prev0) {
            const SirSlot* pv = k == 0 && a.prev0 ? a.prev0 : a.ring + ((t + a.ring_cap - 1) % a.ring_cap);
            prev_s = pv->S;
            prev_i = pv->I;
            prev_r = pv->R;
            // per traversed agent a push costs ~1.35x a pull (every arc of a
            // pusher is walked, with a draw per S neighbour; pullers stop at
            // their first transmission): V2, tools/v2_steps.py (r01).  At 8
            // agents per lane (r02 push chunk pass) ~1.1x: V2 step 15 (I/S =
            // 0.87) pushes in 2.70 ms vs 2.79 pulling, step 16 (1.09) 2.83 vs 2.40
            push = a.dir == 0 ? (APL == 8 ? 10 * prev_i < 9 * prev_s : 4 * prev_i < 3 * prev_s) : a.dir == 2;
        }
        if (prev_i == 0 && (k > 0 || a.prev_ok || (a.prev0 && !a.digest))) {
            // No infected agent: nothing can transmit or recover, so this step and
            // every later one of the launch is the identity (the epidemic is over;
            // C2: steps 124-199).  Their records repeat the current counts (and
            // digest); if an odd number of steps remains, the state is copied to
            // the other buffer set, where the host expects it after the launch
            // (both sets then hold it, which keeps the push's back-buffer invariant).
            // All blocks read the same slot after the last barrier, so all leave here.
            const SirSlot* pv = k == 0 && a.prev0 ? a.prev0 : a.ring + ((t + a.ring_cap - 1) % a.ring_cap);
            sir_identity_tail(a.ring, a.ring_cap, pv, t, a.n_steps - k, a.digest, a.x[cur], a.x[cur ^ 1], a.ib[cur],
                              a.ib[cur ^ 1], a.sb[cur], a.sb[cur ^ 1], a.n_pad);
            return;
        }
        if (push) {
            long long rec = 0, inf = 0;
            unsigned long long dig = 0;
            sir_push_body<APL>(a, cur, t, sm, rec, inf, dig);
            unsigned long long v[4] = {static_cast<unsigned long long>(-inf), static_cast<unsigned long long>(inf - rec),
                                       static_cast<unsigned long long>(rec), dig};
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                v[0] += prev_s;
                v[1] += prev_i;
                v[2] += prev_r;
            }
            unsigned long long* const outs[4] = {&sl->S, &sl->I, &sl->R, a.digest ? &sl->digest : nullptr};
            block_sum_atomic<4>(v, outs);
        } else {
            unsigned long long cnt[4] = {0, 0, 0, 0};
            sir_pull_body<APL>(a, cur, t, sm, cnt);
            unsigned long long* const outs[4] = {&sl->S, &sl->I, &sl->R, a.digest ? &sl->digest : nullptr};
            block_sum_atomic<4>(cnt, outs);
        }
        uncounted = push && !a.digest && APL == 8;
        cur ^= 1;
        grid.sync();
    }
    if (uncounted) sir_count_new(a, cur, a.ring + ((static_cast<int64_t>(a.t0) + a.n_steps - 1) % a.ring_cap));
}

// ---- sharded push step (NEXT-3) ----
// The shard's infected agents (local I words) walk their rows (local offsets,
// global neighbour ids) against the GLOBAL S bitmap of the current state, with
// the same pair-keyed draw as every other path (S3); a transmitting arc sets
// the neighbour's bit in this rank's copy of the global hit bitmap (no-return
// RED).  The remote parts of that bitmap then go to their owners (fixed-size
// all-to-all of bitmap blocks) and are OR-ed into the owners' words -- no
// per-target append, so no cursor atomics (r02: a warp-aggregated id append
// plus __fns register queues ran 200 us per rank at G = 8, V2 early steps).
struct ShardPushArgs {
    PhiloxKey key;
    const int32_t* row_ptr;    // local rows
    const int32_t* col;        // global neighbour ids
    const uint32_t* ib;        // local I words of the current state
    const uint32_t* sbg;       // global S bitmap of the current state
    uint32_t* hg;              // this rank's global hit bitmap (zeroed)
    int64_t nwords;            // local I words (npl / 32)
    uint32_t lo;
    unsigned long long t_beta;
    uint32_t t;
};

constexpr int kPushQ = 32 + 32 * 32;  // per-warp pusher queue: < 32 carried + one word (32 agents) per lane

__global__ void __launch_bounds__(256) sir_shard_push_kernel(const ShardPushArgs a)
{
    __shared__ uint32_t q[8][kPushQ];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    auto walk = [&](uint32_t g0, uint32_t nown) {
        const bool mine = static_cast<uint32_t>(lane) < nown;
        const uint32_t id = mine ? q[wq][g0 + lane] : 0u;
        const int32_t rb = mine ? a.row_ptr[id] : 0, re = mine ? a.row_ptr[id + 1] : 0;
        const uint32_t own = nown >= 32 ? 0xffffffffu : ((1u << nown) - 1u);
        walk_rows_pay<4>([&](int32_t e) { return static_cast<uint32_t>(__ldcs(a.col + e)); }, own, rb, re, a.lo + id,
                         [&](uint32_t j) { return (__ldcg(a.sbg + (j >> 5)) >> (j & 31u)) & 1u; },
                         [&](uint32_t j, int32_t, int, uint32_t s) {
            const uint4 w = philox(make_uint4(min(s, j), max(s, j), a.t, TAG_SIR_TX), a.key);
            if (static_cast<unsigned long long>(w.x) < a.t_beta) red_or(a.hg + (j >> 5), 1u << (j & 31u));
            return false;  // an infected agent tries every susceptible neighbour
        });
    };
    uint32_t qn = 0;  // queued pushers (warp-uniform, < 32 between words)
    for (int64_t w0 = warp * 32; w0 < a.nwords; w0 += nwarps * 32) {
        // one bitmap word (32 agents) per lane; set bits queued at their warp rank
        const int64_t w = w0 + lane;
        uint32_t m = w < a.nwords ? a.ib[w] : 0u;
        uint32_t tot;
        uint32_t k = qn + warp_excl(__popc(m), &tot);
        for (; m; m &= m - 1u) q[wq][k++] = static_cast<uint32_t>(32 * w) + (__ffs(static_cast<int>(m)) - 1);
        qn += tot;
        __syncwarp();
        uint32_t g0 = 0;
        for (; qn - g0 >= 32; g0 += 32) walk(g0, 32);
        const uint32_t rem = qn - g0;
        const uint32_t carry = static_cast<uint32_t>(lane) < rem ? q[wq][g0 + lane] : 0u;
        __syncwarp();
        if (static_cast<uint32_t>(lane) < rem) q[wq][lane] = carry;
        __syncwarp();
        qn = rem;
    }
    if (qn) walk(0, qn);
}

// This shard's hit words |= the blocks the other ranks sent for it (recv holds
// world blocks of `words` words; the own block is this rank's own region).
__global__ void sir_shard_or_kernel(const uint32_t* __restrict__ recv, int world, int64_t words, uint32_t* own)
{
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (int p = 0; p < world; ++p) v |= recv[p * words + w];
        own[w] |= v;
    }
}

// Finalises a sharded push step from the hit bits, one bitmap word (32 agents)
// per lane: S agents hit -> I, I agents recover with the same draws as every
// other path (lane i & 3 of block i / 4 of the recovery stream, R4), R stays R;
// writes the state bytes (32 per lane), the next I / S words and the step's
// S / I / R counts (and digest).  Replaces the pull kernel's chunk machinery
// in hits mode (r02: 47 us per rank at G = 8, V2 early steps).
__global__ void __launch_bounds__(256) sir_shard_finalize_kernel(const SirStepArgs a, const uint32_t* __restrict__ ibl,
                                                                 const uint32_t* __restrict__ sbl,
                                                                 const uint32_t* __restrict__ hits, uint8_t* __restrict__ y,
                                                                 uint32_t* __restrict__ ib_next,
                                                                 uint32_t* __restrict__ sb_next, SirSlot* slot)
{
    const int64_t words = a.n_pad >> 5;
    unsigned long long cnt[4] = {0, 0, 0, 0};
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t left = a.n - 32 * w;
        const uint32_t real = left <= 0 ? 0u : (left >= 32 ? 0xffffffffu : ((1u << left) - 1u));
        const uint32_t Ws = sbl[w] & real, Wi = ibl[w] & real, H = hits[w] & Ws;
        const unsigned long long g0 = a.gid0 + 32ull * static_cast<unsigned long long>(w);  // multiple of 32
        uint32_t rec = 0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (!((Wi >> (4 * g)) & 0xfu)) continue;
            const uint4 r = stream_block(a.key, TAG_SIR_REC, (g0 >> 2) + g, a.t0);
            uint32_t o = 0;
            if (r.x < a.t_gamma) o |= 1u;
            if (r.y < a.t_gamma) o |= 2u;
            if (r.z < a.t_gamma) o |= 4u;
            if (r.w < a.t_gamma) o |= 8u;
            rec |= (o & (Wi >> (4 * g))) << (4 * g);
        }
        const uint32_t s2 = Ws & ~H, i2 = H | (Wi & ~rec), r2 = real & ~s2 & ~i2, pad = ~real;
        uint32_t b[8];
#pragma unroll
        for (int g = 0; g < 8; ++g)
            b[g] = spread4(i2 >> (4 * g)) * kI + spread4(r2 >> (4 * g)) * kR + spread4(pad >> (4 * g)) * kPad;
        uint4* yv = reinterpret_cast<uint4*>(y + 32 * w);
        yv[0] = make_uint4(b[0], b[1], b[2], b[3]);
        yv[1] = make_uint4(b[4], b[5], b[6], b[7]);
        ib_next[w] = i2;
        sb_next[w] = s2;
        cnt[0] += __popc(s2);
        cnt[1] += __popc(i2);
        cnt[2] += __popc(r2);
        if (a.digest) {
            for (uint32_t m = real; m; m &= m - 1u) {
                const int k = __ffs(static_cast<int>(m)) - 1;
                cnt[3] += digest_term(g0 + k, (b[k >> 2] >> (8 * (k & 3))) & 0xffu);
            }
        }
    }
    unsigned long long* const outs[4] = {&slot->S, &slot->I, &slot->R, a.digest ? &slot->digest : nullptr};
    block_sum_atomic<4>(cnt, outs);
}

// Sharded graph slice: row offsets rebased to the shard's first arc.
__global__ void sir_rebase_kernel(const int32_t* __restrict__ rp, int64_t cnt, int32_t base, int32_t* __restrict__ out)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = rp[k] - base;
}

// S / I / R counts of a state from its bitmaps (after a column write or a step
// reset), accumulated into a zeroed ring slot: the next step's direction choice.
__global__ void sir_count_bits_kernel(const uint32_t* __restrict__ ib, const uint32_t* __restrict__ sb, int64_t n,
                                      SirSlot* slot)
{
    unsigned long long v[3] = {0, 0, 0};
    const int64_t words = (n + 31) / 32;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t left = n - 32 * w;
        const uint32_t real = left >= 32 ? 0xffffffffu : ((1u << left) - 1u);
        v[0] += __popc(sb[w] & real);
        v[1] += __popc(ib[w] & real);
        v[2] += __popc(~(sb[w] | ib[w]) & real);
    }
    unsigned long long* const outs[3] = {&slot->S, &slot->I, &slot->R};
    block_sum_atomic<3>(v, outs);
}

__global__ void sir_zero_slots(SirSlot* ring, int64_t cap, int64_t s0, int64_t count)
{
    for (int64_t k = threadIdx.x; k < count && k < cap; k += blockDim.x) ring[(s0 + k) % cap] = SirSlot{0, 0, 0, 0};
}

}  // namespace

// ---------------------------------------------------------------- model
class SirModel final : public Model {
public:
    int64_t n = 0, n_pad = 0, m_draws = 0, k_inf = 0;
    amber_sir_params p{};
    uint64_t seed = 0;
    PhiloxKey key{};
    Graphs g;
    DevBuf<uint8_t> x[2];
    DevBuf<uint32_t> ib[2], sb[2];  // I / S bitmaps of the two state buffers
    DevBuf<uint32_t> queue;         // persistent launch: chunk counters
    int cur = 0;
    DevBuf<SirSlot> ring;
    int64_t m_first = 0;
    bool prev_ok = false;  // ring slot t-1 holds the counts of the current state
    int dir = 0;           // "direction" option (SirStepArgs::dir)
    DevBuf<SirSlot> cnt0;  // counts of the current state after a column write / step reset
    bool cnt0_ok = false;  // cnt0 is valid (and prev_ok is not): the next launch reads it
    int apl = 0;           // "apl" option: agents per lane of the step kernels (0 = auto, 1, 2, 4)
    // sharded (world > 1, NEXT-3): this rank owns agents [lo, lo + nl) (shard =
    // multiple of 32 agents so bitmap words never straddle ranks), its CSR rows
    // (local offsets, global neighbour ids) and state; every step pulls its rows
    // against the GLOBAL I bitmap, then the shards' next bitmap words are
    // all-gathered (N/8 bytes per step in total).
    ShardComm* sc = nullptr;
    int64_t lo = 0, nl = 0, npl = 0, shard = 0;  // local agents / padded (unsharded: n, n_pad)
    int64_t nq = 0;                              // npl rounded up to whole 128-agent chunks
    DevBuf<uint32_t> ib_glob;  // world * shard / 32 words
    DevBuf<uint32_t> sb_glob;  // the same for the S bits (probed by the sharded push)
    bool glob_ok = false;      // ib_glob / sb_glob hold the current state's bits
    // sharded push step: this rank's global hit bitmap, the blocks received for the
    // own shard, the (fixed) block sizes of the all-to-all
    DevBuf<uint32_t> hg, push_cnt, push_recv;
    DevBuf<SirSlot> gcnt;      // global S / I / R of the current state (direction choice)

    SirModel(int64_t n_, const amber_sir_params& p_, uint64_t seed_, const amber_runtime* r)
    {
        rt.init(r);
        n = n_;
        p = p_;
        seed = seed_;
        key = philox_key(seed);
        AMBER_REQUIRE(n >= 2 && n < (1ll << 31), "SIR needs 2 <= n_agents < 2^31");
        AMBER_REQUIRE(p.mean_degree >= 0 && p.beta >= 0 && p.beta <= 1 && p.gamma >= 0 && p.gamma <= 1 &&
                          p.init_frac >= 0 && p.init_frac <= 1,
                      "SIR params out of range");
        m_draws = static_cast<int64_t>(std::floor(static_cast<double>(n) * p.mean_degree / 2.0 + 0.5));
        k_inf = static_cast<int64_t>(std::floor(p.init_frac * static_cast<double>(n) + 0.5));
        n_pad = ceil_div(n, 32) * 32;
        std::vector<unsigned long long> seeds{seed};
        build_graphs(rt, seeds, n, m_draws, g);
        nl = n;
        npl = n_pad;
        // AMBER_TEST_FORCE_EXCHANGE=1 with a unique id: the sharded path with one rank
        // (a one-rank NCCL communicator: exercises the all-gather/all-reduce plumbing)
        const char* force = getenv("AMBER_TEST_FORCE_EXCHANGE");
        const bool sharded = rt.world > 1 || (force && force[0] == '1' && r && r->nccl_unique_id);
        if (sharded) {
            AMBER_REQUIRE(rt.rank >= 0 && rt.rank < rt.world, "rank out of range");
            sir_shard_range(n, rt.world, rt.rank, &lo, &nl, &shard);
            npl = shard;
        }
        nq = sir_chunks(npl, kChunkMax / 32) * kChunkMax;  // the step kernels work on chunks of up to 256 agents
        for (auto& b : x) {
            b.allocate(&rt, nq);
            AMBER_CUDA(cudaMemsetAsync(b.p, kPad, nq, rt.stream));
        }
        for (int c = 0; c < 2; ++c) {
            ib[c].allocate(&rt, nq / 32);
            sb[c].allocate(&rt, nq / 32);
        }
        if (sharded) {
            // every rank builds the (seeded, deterministic) graph and initial state,
            // keeps its slice and frees the rest
            DevBuf<uint8_t> full;
            full.allocate(&rt, n_pad);
            build_init_state(rt, seeds, n, n_pad, k_inf, full.p);
            AMBER_CUDA(cudaMemsetAsync(x[0].p, kPad, npl, rt.stream));
            if (nl) AMBER_CUDA(cudaMemcpyAsync(x[0].p, full.p + lo, nl, cudaMemcpyDeviceToDevice, rt.stream));
            slice_graph();
            ib_glob.allocate(&rt, static_cast<size_t>(rt.world) * (shard / 32) + kChunkMax / 32);  // + one chunk of slack
            sb_glob.allocate(&rt, static_cast<size_t>(rt.world) * (shard / 32) + kChunkMax / 32);
            AMBER_CUDA(cudaMemsetAsync(ib_glob.p, 0, ib_glob.n * 4, rt.stream));
            AMBER_CUDA(cudaMemsetAsync(sb_glob.p, 0, sb_glob.n * 4, rt.stream));
            sc = make_shard_comm(rt, r);
            rt.sync();
        } else {
            build_init_state(rt, seeds, n, n_pad, k_inf, x[0].p);
        }
        build_bits();
        queue.allocate(&rt, 4 * kRegions);
        ring.allocate(&rt, metrics_cap);
        ring.zero_async(rt.stream);
        seed_counts(static_cast<unsigned long long>(n - k_inf), static_cast<unsigned long long>(k_inf), 0ull);
        rt.sync();
    }

    // Bitmaps of the current state; the back buffers become a copy of it (the
    // push step's invariant: every agent S now is S in the back state).
    void build_bits()
    {
        sir_bits_kernel<<<rt.num_sms * 8, 256, 0, rt.stream>>>(x[cur].p, nq, ib[cur].p, sb[cur].p);
        check_launch("sir_bits_kernel");
        AMBER_CUDA(cudaMemcpyAsync(x[cur ^ 1].p, x[cur].p, nq, cudaMemcpyDeviceToDevice, rt.stream));
        AMBER_CUDA(cudaMemcpyAsync(ib[cur ^ 1].p, ib[cur].p, nq / 8, cudaMemcpyDeviceToDevice, rt.stream));
        AMBER_CUDA(cudaMemcpyAsync(sb[cur ^ 1].p, sb[cur].p, nq / 8, cudaMemcpyDeviceToDevice, rt.stream));
        glob_ok = false;
    }

    // Sharded: keep the rows [lo, lo + nl) of the full CSR (offsets rebased to 0;
    // neighbour ids stay global).
    void slice_graph()
    {
        std::vector<int32_t> ends(2);
        AMBER_CUDA(cudaMemcpyAsync(&ends[0], g.row_ptr.p + lo, 4, cudaMemcpyDeviceToHost, rt.stream));
        AMBER_CUDA(cudaMemcpyAsync(&ends[1], g.row_ptr.p + lo + nl, 4, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        const int64_t arcs = ends[1] - ends[0];
        DevBuf<int32_t> rp, col;
        rp.allocate(&rt, nl + 1);
        col.allocate(&rt, std::max<int64_t>(arcs, 1) + 8);
        sir_rebase_kernel<<<rt.num_sms * 4, 256, 0, rt.stream>>>(g.row_ptr.p + lo, nl + 1, ends[0], rp.p);
        check_launch("sir_rebase_kernel");
        if (arcs)
            AMBER_CUDA(cudaMemcpyAsync(col.p, g.col.p + ends[0], arcs * 4, cudaMemcpyDeviceToDevice, rt.stream));
        rt.sync();
        std::swap(g.row_ptr.p, rp.p);
        std::swap(g.row_ptr.n, rp.n);
        std::swap(g.col.p, col.p);
        std::swap(g.col.n, col.n);
        g.arcs = arcs;
    }

    // Sharded: all-gather the current state's local I-bitmap words.
    void gather_bits(int c)
    {
        shard_allgather_u32(sc, rt, ib[c].p, ib_glob.p, static_cast<size_t>(shard / 32));
        shard_allgather_u32(sc, rt, sb[c].p, sb_glob.p, static_cast<size_t>(shard / 32));
        glob_ok = true;
    }

    // counts of the current state into ring slot t-1 (direction choice of the next step)
    void seed_counts(unsigned long long S, unsigned long long I, unsigned long long R)
    {
        const SirSlot v{S, I, R, 0};
        AMBER_CUDA(cudaMemcpyAsync(ring.p + (t + metrics_cap - 1) % metrics_cap, &v, sizeof(v),
                                   cudaMemcpyHostToDevice, rt.stream));
        rt.sync();
        prev_ok = true;
    }

    ~SirModel() override
    {
        if (rt.stream) cudaStreamSynchronize(rt.stream);
        g.row_ptr.reset();
        g.col.reset();
        for (auto& b : x) b.reset();
        for (int c = 0; c < 2; ++c) {
            ib[c].reset();
            sb[c].reset();
        }
        ring.reset();
        queue.reset();
        ib_glob.reset();
        sb_glob.reset();
        hg.reset();
        push_cnt.reset();
        push_recv.reset();
        gcnt.reset();
        if (sc) destroy_shard_comm(sc);
        rt.destroy();
    }

    SirStepArgs args(int64_t nsteps)
    {
        SirStepArgs a{};
        a.key = key;
        a.row_ptr = g.row_ptr.p;
        a.col = g.col.p;
        a.x[0] = x[0].p;
        a.x[1] = x[1].p;
        for (int c = 0; c < 2; ++c) {
            a.ib[c] = ib[c].p;
            a.sb[c] = sb[c].p;
        }
        a.prev_ok = prev_ok ? 1 : 0;
        a.prev0 = !prev_ok && cnt0_ok ? cnt0.p : nullptr;
        a.n = nl;
        a.n_pad = npl;
        a.gid0 = static_cast<unsigned long long>(lo);
        a.t_beta = bernoulli_threshold_host(p.beta);
        a.t_gamma = bernoulli_threshold_host(p.gamma);
        a.t0 = static_cast<uint32_t>(t);
        a.n_steps = nsteps;
        a.cur = cur;
        a.ring = ring.p;
        a.ring_cap = metrics_cap;
        a.digest = digest_on ? 1 : 0;
        a.dir = dir;
        return a;
    }

    // agents per lane of the step kernels ("apl" option; auto: 8 for large
    // populations, 1 where the step is latency-bound -- shorter warp tasks)
    int lanes_apl() const { return apl ? apl : (npl > (1ll << 22) ? 8 : 1); }

    void launch_step(int L, int blocks, int threads, const SirStepArgs& a)
    {
        if (L == 8) sir_step_kernel<8><<<blocks, threads, 0, rt.stream>>>(a);
        else if (L == 4) sir_step_kernel<4><<<blocks, threads, 0, rt.stream>>>(a);
        else if (L == 2) sir_step_kernel<2><<<blocks, threads, 0, rt.stream>>>(a);
        else sir_step_kernel<1><<<blocks, threads, 0, rt.stream>>>(a);
    }

    void step(int64_t nsteps) override
    {
        AMBER_REQUIRE(nsteps >= 0, "n_steps must be >= 0");
        AMBER_REQUIRE(t + nsteps < (1ll << 32), "step index would exceed 2^32");
        if (sc) {
            step_sharded(nsteps);
            return;
        }
        int64_t done = 0;
        while (done < nsteps) {
            // slot t-1 (counts of the current state) must survive the zeroing of [t, t+chunk)
            const int64_t chunk = std::min<int64_t>(nsteps - done, metrics_cap - 1);
            sir_zero_slots<<<1, 256, 0, rt.stream>>>(ring.p, metrics_cap, t, chunk);
            check_launch("sir_zero_slots");
            const int threads = block ? static_cast<int>(std::min<int64_t>(block, 256)) : 256;
            const int L = lanes_apl();
            if (persistent && (chunk > 1 || dir != 0)) {
                const int pthreads = block ? threads : kSirPT;
                const void* fn = L == 8 ? reinterpret_cast<const void*>(sir_persistent_kernel<8>)
                               : L == 4 ? reinterpret_cast<const void*>(sir_persistent_kernel<4>)
                               : L == 2 ? reinterpret_cast<const void*>(sir_persistent_kernel<2>)
                                        : reinterpret_cast<const void*>(sir_persistent_kernel<1>);
                int per_sm = 0;
                AMBER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, pthreads, 0));
                // latency-bound: many resident warps help, but the grid barrier
                // cost grows with the block count; 3 blocks/SM measured best (C2)
                // (C2); large populations are bound by random L2 lookups instead: full occupancy
                const int per = n_pad > (1ll << 22) ? per_sm : std::min(per_sm, std::max(1, 768 / pthreads));
                int blocks = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(per) * rt.num_sms,
                                                                ceil_div(sir_chunks(n_pad, L), std::max(1, pthreads / 32))));
                if (grid) blocks = static_cast<int>(std::min<int64_t>(grid, static_cast<int64_t>(per_sm) * rt.num_sms));
                blocks = std::max(blocks, 1);
                SirStepArgs a = args(chunk);
                queue.zero_async(rt.stream);
                a.queue = queue.p;
                const int64_t warps = static_cast<int64_t>(blocks) * pthreads / 32;
                a.grab = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(64, sir_chunks(n_pad, L) / (warps * 8))));
                if (sir_chunks(n_pad, L) <= 2 * warps) a.queue = nullptr;  // <= 2 chunks per warp: static striding
                void* kargs[] = {&a};
                prof.launch(rt.stream, "sir_persistent", [&] {
                    AMBER_CUDA(cudaLaunchCooperativeKernel(fn, blocks, pthreads, kargs, 0, rt.stream));
                });
                check_launch("sir_persistent_kernel");
                t += chunk;
                if (chunk & 1) cur ^= 1;
                prev_ok = true;
                cnt0_ok = false;
            } else {
                for (int64_t k = 0; k < chunk; ++k) {
                    SirStepArgs a = args(1);
                    int blocks = static_cast<int>(ceil_div(sir_chunks(n_pad, L), std::max(1, threads / 32)));
                    if (grid) blocks = static_cast<int>(grid);
                    prof.launch(rt.stream, "sir_step", [&] { launch_step(L, blocks, threads, a); });
                    check_launch("sir_step_kernel");
                    cur ^= 1;
                    ++t;
                }
                prev_ok = true;
                cnt0_ok = false;
            }
            done += chunk;
        }
    }

    // Sharded steps: per step either one pull launch over the local rows (reading
    // the global I bitmap) or a push phase (push_phase: the shard's infected
    // agents mark their targets in a global hit bitmap whose remote blocks go to
    // their owners) followed by the same launch finalising from the hit bits;
    // then the all-gather of the next I and S bitmap words.  Identical results
    // for any rank count and direction (pair-keyed draws, S3).
    void step_sharded(int64_t nsteps)
    {
        const int threads = block ? static_cast<int>(std::min<int64_t>(block, 256)) : 256;
        if (!glob_ok) gather_bits(cur);
        for (int64_t k = 0; k < nsteps; ++k) {
            sir_zero_slots<<<1, 32, 0, rt.stream>>>(ring.p, metrics_cap, t, 1);
            check_launch("sir_zero_slots");
            const bool push = sharded_push_now();
            SirStepArgs a = args(1);
            a.ib[cur] = ib_glob.p;  // read: global bits of state t; write: local bits of t+1
            if (push) push_phase();
            if (push) {
                const int fb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(npl / 32, 256),
                                                                                        rt.num_sms * 8)));
                prof.launch(rt.stream, "sir_shard_finalize", [&] {
                    sir_shard_finalize_kernel<<<fb, 256, 0, rt.stream>>>(a, ib[cur].p, sb[cur].p, hg.p + lo / 32,
                                                                         x[cur ^ 1].p, ib[cur ^ 1].p, sb[cur ^ 1].p,
                                                                         ring.p + (t % metrics_cap));
                });
                check_launch("sir_shard_finalize_kernel");
            } else {
                const int L = lanes_apl();
                int blocks = static_cast<int>(std::max<int64_t>(1, ceil_div(sir_chunks(npl, L), std::max(1, threads / 32))));
                if (grid) blocks = static_cast<int>(grid);
                prof.launch(rt.stream, "sir_shard_step", [&] { launch_step(L, blocks, threads, a); });
                check_launch("sir_step_kernel");
            }
            cur ^= 1;
            ++t;
            gather_bits(cur);
        }
        prev_ok = false;
    }

    // Direction of the next sharded step: push when the infected agents are
    // fewer than 0.9x the susceptible ones (the one-GPU rule at 8 agents per
    // lane), from the global counts of the current state (popcounts of the
    // all-gathered bitmaps); option "direction": 1 pull only, 2 push.
    bool sharded_push_now()
    {
        if (dir == 1) return false;
        if (dir == 2) return true;
        if (!gcnt.p) gcnt.allocate(&rt, 1);
        AMBER_CUDA(cudaMemsetAsync(gcnt.p, 0, sizeof(SirSlot), rt.stream));
        sir_count_bits_kernel<<<rt.num_sms * 2, 256, 0, rt.stream>>>(ib_glob.p, sb_glob.p, n, gcnt.p);
        check_launch("sir_count_bits_kernel");
        SirSlot h{};
        AMBER_CUDA(cudaMemcpyAsync(&h, gcnt.p, sizeof(h), cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        return 10 * h.I < 9 * h.S;
    }

    // Sharded push phase of step t: the pushers' walk into this rank's global hit
    // bitmap, the remote blocks of it to their owners (fixed-size all-to-all),
    // OR-ed into the own block.
    void push_phase()
    {
        const size_t words = static_cast<size_t>(shard / 32);
        const size_t gwords = static_cast<size_t>(rt.world) * words + kChunkMax / 32;
        if (!hg.p) {
            hg.allocate(&rt, gwords);
            push_recv.allocate(&rt, static_cast<size_t>(rt.world) * words);
            push_cnt.allocate(&rt, rt.world);
            std::vector<uint32_t> c(rt.world, static_cast<uint32_t>(words));
            AMBER_CUDA(cudaMemcpyAsync(push_cnt.p, c.data(), c.size() * 4, cudaMemcpyHostToDevice, rt.stream));
            rt.sync();
        }
        AMBER_CUDA(cudaMemsetAsync(hg.p, 0, gwords * 4, rt.stream));
        ShardPushArgs pa{};
        pa.key = key;
        pa.row_ptr = g.row_ptr.p;
        pa.col = g.col.p;
        pa.ib = ib[cur].p;
        pa.sbg = sb_glob.p;
        pa.hg = hg.p;
        pa.nwords = npl / 32;
        pa.lo = static_cast<uint32_t>(lo);
        pa.t_beta = bernoulli_threshold_host(p.beta);
        pa.t = static_cast<uint32_t>(t);
        prof.launch(rt.stream, "sir_shard_push", [&] {
            sir_shard_push_kernel<<<rt.num_sms * 8, 256, 0, rt.stream>>>(pa);
        });
        check_launch("sir_shard_push_kernel");
        shard_alltoallv(sc, rt, hg.p, push_cnt.p, words, 4, push_recv.p, static_cast<size_t>(rt.world) * words);
        prof.launch(rt.stream, "sir_shard_or", [&] {
            sir_shard_or_kernel<<<rt.num_sms * 4, 256, 0, rt.stream>>>(push_recv.p, rt.world, static_cast<int64_t>(words),
                                                                     hg.p + lo / 32);
        });
        check_launch("sir_shard_or_kernel");
    }

    // Sharded metrics / digests are global: summed over the ranks (collective).
    void global_sum(unsigned long long* h, size_t cnt)
    {
        if (!sc || !cnt) return;
        DevBuf<unsigned long long> d;
        d.allocate(&rt, cnt);
        AMBER_CUDA(cudaMemcpyAsync(d.p, h, cnt * 8, cudaMemcpyHostToDevice, rt.stream));
        shard_allreduce_u64(sc, rt, d.p, cnt);
        AMBER_CUDA(cudaMemcpyAsync(h, d.p, cnt * 8, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
    }

    // Sharded: "state" is this rank's slice [lo, lo + nl) of the global column;
    // "row_ptr" / "col_idx" are its rows (offsets from 0, global neighbour ids).
    bool column_info(const char* name, amber_dtype* dt, int64_t* glen, int64_t* off, int64_t* len) override
    {
        std::string k(name);
        int64_t L, G, O = 0;
        amber_dtype d;
        if (k == "state") { d = AMBER_U8; L = nl; G = n; O = lo; }
        else if (k == "row_ptr") { d = AMBER_I32; L = nl + 1; G = L; }
        else if (k == "col_idx") { d = AMBER_I32; L = g.arcs; G = L; }
        else return false;
        if (dt) *dt = d;
        if (glen) *glen = G;
        if (off) *off = O;
        if (len) *len = L;
        return true;
    }

    void read_column(const char* name, void* dst, size_t bytes, bool on_dev) override
    {
        std::string k(name);
        const void* src;
        size_t nb;
        if (k == "state") { src = x[cur].p; nb = nl; }
        else if (k == "row_ptr") { src = g.row_ptr.p; nb = (nl + 1) * 4; }
        else if (k == "col_idx") { src = g.col.p; nb = g.arcs * 4; }
        else fail(AMBER_E_UNKNOWN_NAME, "no column " + k);
        if (bytes < nb) fail(AMBER_E_BUFFER_TOO_SMALL, "dst too small for column " + k);
        copy_out(rt, dst, src, nb, on_dev);
    }

    void write_column(const char* name, const void* src, size_t bytes, bool on_dev) override
    {
        std::string k(name);
        if (k == "row_ptr" || k == "col_idx") fail(AMBER_E_INVALID_ARG, "column " + k + " is read-only");
        if (k != "state") fail(AMBER_E_UNKNOWN_NAME, "no column " + k);
        if (bytes < static_cast<size_t>(nl)) fail(AMBER_E_BUFFER_TOO_SMALL, "src smaller than state column");
        copy_in(rt, x[cur].p, src, nl, on_dev);
        build_bits();
        recount();
    }

    // Counts of the current state (into cnt0, not the ring: slot t-1 keeps the
    // record of step t-1), so the next step chooses its direction -- a pull
    // from a state with few infected agents costs ~15x a push at V2.  Sharded
    // steps always pull: nothing to do.
    void recount()
    {
        prev_ok = false;
        cnt0_ok = false;
        if (sc) return;
        if (!cnt0.p) cnt0.allocate(&rt, 1);
        AMBER_CUDA(cudaMemsetAsync(cnt0.p, 0, sizeof(SirSlot), rt.stream));
        sir_count_bits_kernel<<<rt.num_sms * 4, 256, 0, rt.stream>>>(ib[cur].p, sb[cur].p, nl, cnt0.p);
        check_launch("sir_count_bits_kernel");
        cnt0_ok = true;
    }

    void read_metrics(const char* name, void* dst, size_t bytes, int64_t* n_out) override
    {
        std::string k(name);
        size_t off;
        if (k == "S") off = offsetof(SirSlot, S);
        else if (k == "I") off = offsetof(SirSlot, I);
        else if (k == "R") off = offsetof(SirSlot, R);
        else if (k == "digest" && digest_on) off = offsetof(SirSlot, digest);
        else fail(AMBER_E_UNKNOWN_NAME, "no metric " + k);
        std::vector<SirSlot> h(metrics_cap);
        AMBER_CUDA(cudaMemcpyAsync(h.data(), ring.p, metrics_cap * sizeof(SirSlot), cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        const int64_t first = std::max(m_first, t - metrics_cap);
        const int64_t cnt = std::max<int64_t>(t - first, 0);
        if (bytes < static_cast<size_t>(cnt) * 8) fail(AMBER_E_BUFFER_TOO_SMALL, "metrics dst too small");
        std::vector<unsigned long long> vals(cnt);
        for (int64_t s = first; s < t; ++s)
            std::memcpy(&vals[s - first], reinterpret_cast<const char*>(&h[s % metrics_cap]) + off, 8);
        global_sum(vals.data(), vals.size());  // sharded: counts and digests of all ranks
        std::memcpy(dst, vals.data(), cnt * 8);
        if (n_out) *n_out = cnt;
    }

    void reset_metrics() override
    {
        rt.sync();
        m_first = t;
    }

    uint64_t digest(const char* name) override
    {
        const std::string k(name);
        // graph columns: D1 over the int32 bits with the array index as id (the
        // local rows of a shard; no all-reduce -- test hook for full-size graphs)
        if (k == "row_ptr")
            return device_digest_u32(rt, reinterpret_cast<const uint32_t*>(g.row_ptr.p), nl + 1, 0);
        if (k == "col_idx")
            return device_digest_u32(rt, reinterpret_cast<const uint32_t*>(g.col.p), g.arcs, 0);
        if (k != "state") fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        unsigned long long d = device_digest_u8(rt, x[cur].p, nl, lo);
        global_sum(&d, 1);
        return d;
    }

    void set_step(int64_t s) override
    {
        AMBER_REQUIRE(s >= 0 && s < (1ll << 32), "step out of range");
        rt.sync();
        t = s;
        m_first = s;
        recount();
    }

    bool set_option(const char* key, int64_t v) override
    {
        std::string k(key);
        if (k == "metrics_capacity") {
            AMBER_REQUIRE(v >= 16, "metrics_capacity must be >= 16");
            rt.sync();
            metrics_cap = v;
            ring.allocate(&rt, metrics_cap);
            ring.zero_async(rt.stream);
            m_first = t;
            prev_ok = false;
            return true;
        }
        if (k == "block") AMBER_REQUIRE(v <= 256, "SIR kernels are built for <= 256 threads per block");
        if (k == "apl") {
            AMBER_REQUIRE(v == 0 || v == 1 || v == 2 || v == 4 || v == 8, "apl must be 0 (auto), 1, 2, 4 or 8");
            apl = static_cast<int>(v);
            return true;
        }
        if (k == "direction") {
            AMBER_REQUIRE(v >= 0 && v <= 2, "direction must be 0 (auto), 1 (pull) or 2 (push)");
            dir = static_cast<int>(v);
            return true;
        }
        return Model::set_option(key, v);
    }

    bool get_option(const char* key, int64_t* v) override
    {
        std::string k(key);
        if (k == "edges") { *v = g.arcs / 2; return true; }
        if (k == "direction") { *v = dir; return true; }
        if (k == "apl") { *v = lanes_apl(); return true; }
        return Model::get_option(key, v);
    }
};

Model* make_sir(int64_t n, const amber_sir_params& p, uint64_t seed, const amber_runtime* rt)
{
    return new SirModel(n, p, seed, rt);
}

}  // namespace amber
