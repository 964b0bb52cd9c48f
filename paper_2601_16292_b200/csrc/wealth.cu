// wealth.cu -- wealth-transfer model (Sec. 5.1.1; W1-W3).
//
// One fused kernel per step.  Launch t:
//   apply   step t  : w'_i = w_i - a*s_i + a*c_i,  c_i = counter i of step t (read + zeroed)
//   scatter step t+1: s'_i = [w'_i >= a], r_i = Philox receiver, counter[r_i] += 1
// so each step streams the int32 wealth column once in and once out (8 B per
// agent) while the per-receiver counters of steps t and t+1 (packed 4-bit by
// default: 2 x N/2 bytes) stay in L2 and take the scatter as L2 atomics.
// A counter overflow is detected exactly (sum of decoded counters != number of
// increments) and the affected step window is replayed with 32-bit counters
// from a pinned copy of the window's first state (3 rotating wealth buffers).
#include <algorithm>
#include <type_traits>

#include "internal.cuh"
#include "philox.cuh"
#include "wealth.cuh"

namespace amber {

namespace {

#ifndef AMBER_WEALTH_QPT
#define AMBER_WEALTH_QPT 8
#endif
// Sharded-step tunables (r02 ncu launch lists, tools/shard_phase_probe.py, fused
// step per rank at G = 8 / G = 2): ranks taken when staging 87.3 / 292.7 us vs
// in a flush pass 90.0 / 301.2; three blocks per SM (80 registers, spills)
// 85.7-86.2 / 301.6-302.3 -- kept at two (no spills).
#ifndef AMBER_WEALTH_STAGE_RANK
#define AMBER_WEALTH_STAGE_RANK 1  // destination ranks taken when staging (shared atomic per append)
#endif
#ifndef AMBER_WEALTH_MINB_REMOTE
#define AMBER_WEALTH_MINB_REMOTE 2
#endif
#ifndef AMBER_WEALTH_MINB
#define AMBER_WEALTH_MINB 1
#endif
#ifndef AMBER_WEALTH_HINT
#define AMBER_WEALTH_HINT 1
#endif
constexpr int kQPT = AMBER_WEALTH_QPT;   // quads (4 agents) per thread per chunk
constexpr int kChunkAgents = 4 * kQPT * 32;  // agents per warp chunk (512)
// Remote-bucket slices per destination and the cursor spacing (words).  One
// cursor per destination took one same-address atomic per warp call and
// destination: every warp of the grid serialised on world - 1 addresses (r02,
// tools/shard_phase_probe.py under the ncu launch list: the G = 8 fused step
// 389 us per rank for 1.25e7 agents, G = 2 1,418 us for 5e7 -- ~0.9 ns per
// atomic per address).  64 slices on separate 128-byte lines spread them.
constexpr int kRemoteSlices = 64;
constexpr int kCountStride = 32;

using Slot = WealthSlot;

struct WealthArgs {
    PhiloxKey key;
    const int32_t* w_in;
    int32_t* w_out;
    uint32_t* inc_cur;   // counters of the applied step (read + zeroed)
    uint32_t* inc_next;  // counters of the scattered step (atomics)
    int64_t nchunks;     // warp chunks (kChunkAgents agents each) of the padded shard
    int64_t n_loc;       // real agents in this shard
    unsigned long long lo;      // global id of local agent 0
    unsigned long long n_glob;  // N
    int32_t amount;
    int32_t exclude_self;
    uint32_t t_apply, t_scatter;
    Slot* slot_apply;    // record of the applied step
    Slot* slot_scatter;  // record receiving the scattered step's increment count
    Slot* slot_zero;     // slot zeroed at kernel start (two steps ahead), may be null
    // cross-shard receivers (REMOTE): per destination rank, kRemoteSlices
    // slices (warp chunk c appends to slice c % kRemoteSlices), each with its
    // own cursor on its own 128-byte line -- see remote_append
    int world;
    unsigned long long shard_size;
    uint32_t shard_magic;             // 0xFFFFFFFF / shard_size (dest_of: no 64-bit division)
    unsigned long long slo, slim;     // non-REMOTE scatter: counter index = receiver - slo, < slim (the
                                      // shard: lo / n_loc; the dense exchange: 0 / N, global counters)
    uint32_t* remote_ids;             // [world][kRemoteSlices][remote_cap] global receiver ids
    unsigned int* remote_count;       // [world][kRemoteSlices] cursors, kCountStride words apart
    unsigned long long remote_cap;    // ids per slice
};

// ---- packed counters: 4 agents (a quad) own 4*B contiguous bits ----
template <int B>
__device__ __forceinline__ void load_quad_counts(const uint32_t* inc, int64_t q, uint32_t c[4])
{
    if constexpr (B == 2) {
        const uint32_t v = reinterpret_cast<const uint8_t*>(inc)[q];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = (v >> (2 * k)) & 3u;
    } else if constexpr (B == 4) {
        const uint32_t v = reinterpret_cast<const uint16_t*>(inc)[q];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = (v >> (4 * k)) & 15u;
    } else if constexpr (B == 8) {
        const uint32_t v = inc[q];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = (v >> (8 * k)) & 255u;
    } else if constexpr (B == 16) {
        const uint2 v = reinterpret_cast<const uint2*>(inc)[q];
        c[0] = v.x & 0xFFFFu; c[1] = v.x >> 16; c[2] = v.y & 0xFFFFu; c[3] = v.y >> 16;
    } else {
        const uint4 v = reinterpret_cast<const uint4*>(inc)[q];
        c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w;
    }
}

template <int B>
__device__ __forceinline__ void zero_quad_counts(uint32_t* inc, int64_t q)
{
    if constexpr (B == 2) reinterpret_cast<uint8_t*>(inc)[q] = 0;
    else if constexpr (B == 4) reinterpret_cast<uint16_t*>(inc)[q] = 0;
    else if constexpr (B == 8) inc[q] = 0u;
    else if constexpr (B == 16) reinterpret_cast<uint2*>(inc)[q] = make_uint2(0u, 0u);
    else reinterpret_cast<uint4*>(inc)[q] = make_uint4(0u, 0u, 0u, 0u);
}

// L2 eviction-priority policies: keep the counters resident, stream the column.
__device__ __forceinline__ unsigned long long policy_evict_last()
{
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void red_add_hint(uint32_t* addr, uint32_t v, unsigned long long pol)
{
#if AMBER_WEALTH_HINT
    asm volatile("red.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(addr), "r"(v), "l"(pol) : "memory");
#else
    (void)pol;
    atomicAdd(addr, v);
#endif
}

template <int B, class Id>
__device__ __forceinline__ void add_count(uint32_t* inc, Id rl, unsigned long long pol, unsigned long long lim)
{
    AMBER_DCHECK(static_cast<unsigned long long>(rl) < lim, "wealth: receiver counter index out of the shard");
    if constexpr (B == 32) {
        red_add_hint(inc + rl, 1u, pol);
    } else {
        constexpr Id per = 32 / B;
        red_add_hint(inc + (rl / per), 1u << (static_cast<uint32_t>(rl % per) * B), pol);
    }
}

// R6/W2 receiver; `m` = N (or N-1 when excluding self), precomputed on the host.
template <bool FAST32>
__device__ __forceinline__ unsigned long long receiver(unsigned long long x, unsigned long long i,
                                                       unsigned long long m, int exclude_self)
{
    unsigned long long r;
    if constexpr (FAST32) r = mulhi64_n32(x, static_cast<uint32_t>(m));
    else r = mulhi64(x, m);
    if (exclude_self) r += (r >= i);
    return r;
}

// Owning rank of global id r (sharded runs have ids < 2^32): q = umulhi(r, m)
// with m = floor((2^32 - 1) / s) is floor(r / s) or one less, fixed by one
// compare -- the 64-bit division it replaces was 17% of the sharded fused
// step's instructions (r02 ncu, G = 8).
__device__ __forceinline__ unsigned dest_of(const WealthArgs& a, unsigned long long r)
{
    const uint32_t r32 = static_cast<uint32_t>(r), s32 = static_cast<uint32_t>(a.shard_size);
    uint32_t q = __umulhi(r32, a.shard_magic);
    if (r32 - q * s32 >= s32) ++q;
    return q < static_cast<uint32_t>(a.world) ? q : static_cast<uint32_t>(a.world - 1);
}

// Warp-aggregated append of a cross-shard receiver into its destination
// bucket's slice `sl` (the warp chunk's index mod kRemoteSlices; a slice's
// capacity covers every agent of its chunks, so it cannot overflow).  Must be
// reached by all 32 lanes (flag selects the participating ones).
__device__ __forceinline__ void remote_append(const WealthArgs& a, bool flag, unsigned long long r, unsigned sl)
{
    const unsigned mask = __ballot_sync(0xffffffffu, flag);
    if (!flag) return;
    AMBER_DCHECK(r < a.n_glob, "wealth: remote receiver id >= N");
    const unsigned dest = dest_of(a, r);
    const unsigned peers = __match_any_sync(mask, dest);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    const unsigned rank = __popc(peers & ((1u << lane) - 1u));
    unsigned base = 0;
    const unsigned long long bucket = static_cast<unsigned long long>(dest) * kRemoteSlices + sl;
    if (lane == leader) base = atomicAdd(a.remote_count + bucket * kCountStride, static_cast<unsigned>(__popc(peers)));
    base = __shfl_sync(peers, base, leader);
    const unsigned long long pos = base + rank;
    AMBER_DCHECK(pos < a.remote_cap, "wealth: remote bucket slice overflow");
    if (pos < a.remote_cap) a.remote_ids[bucket * a.remote_cap + pos] = static_cast<uint32_t>(r);
}

// Warp-staged remote appends (world <= 32): the receivers a warp sends off-shard
// are queued in shared memory (no global atomic per append) and flushed every
// kFlushQuads quad rows: per destination ONE cursor atomic for the whole batch
// (issued by all destination lanes together, so a flush exposes one L2 round
// trip), then the ids are stored behind it.  The direct warp-aggregated
// append (remote_append) waited on a returning cursor atomic in every call --
// ~32 round trips per warp chunk (r02 launch list, G = 8: the fused step 182
// us per rank with sliced cursors, vs ~49 us of the unsharded kernel's work).
constexpr int kFlushQuads = 4;                      // quad rows between flushes
constexpr int kStageCap = kFlushQuads * 4 * 32;     // receivers staged per warp (<= 1 per agent)
struct RemoteStage {
    uint32_t id[8][kStageCap];      // receiver ids, arrival order (8 warps per 256-thread block)
    uint16_t meta[8][kStageCap];    // destination << 10 | rank within the destination
    unsigned cnt[8][32];            // per-destination counts of the batch
    unsigned base[8][32];           // per-destination cursor bases
};
static_assert(kStageCap <= 1024, "meta packs the rank in 10 bits");

__device__ __forceinline__ void remote_stage(const WealthArgs& a, RemoteStage& st, int wq, unsigned& qn, bool flag,
                                             unsigned long long r)
{
    const unsigned mask = __ballot_sync(0xffffffffu, flag);
    const int lane = threadIdx.x & 31;
    if (flag) {
        AMBER_DCHECK(r < a.n_glob, "wealth: remote receiver id >= N");
        const unsigned dest = dest_of(a, r);
        const unsigned pos = qn + __popc(mask & ((1u << lane) - 1u));
        st.id[wq][pos] = static_cast<uint32_t>(r);
#if AMBER_WEALTH_STAGE_RANK
        const unsigned rank = atomicAdd(&st.cnt[wq][dest], 1u);  // shared-memory atomic: rank within the destination
        st.meta[wq][pos] = static_cast<uint16_t>((dest << 10) | rank);
#else
        st.meta[wq][pos] = static_cast<uint16_t>(dest << 10);
#endif
    }
    qn += __popc(mask);
}

__device__ __forceinline__ void remote_flush(const WealthArgs& a, RemoteStage& st, int wq, unsigned& qn, unsigned sl)
{
    const int lane = threadIdx.x & 31;
    if (qn == 0) return;  // warp-uniform
#if !AMBER_WEALTH_STAGE_RANK
    st.cnt[wq][lane] = 0u;
    __syncwarp();
    for (unsigned e = lane; e < qn; e += 32) {
        const unsigned d = st.meta[wq][e] >> 10;
        const unsigned rank = atomicAdd(&st.cnt[wq][d], 1u);  // shared-memory atomic
        st.meta[wq][e] = static_cast<uint16_t>((d << 10) | rank);
    }
#endif
    __syncwarp();
    const unsigned c = st.cnt[wq][lane];
#if AMBER_WEALTH_STAGE_RANK
    st.cnt[wq][lane] = 0u;  // the next batch ranks from zero (read above, before the stores below)
#endif
    if (c) {
        // the batch's first element index in remote_ids (< world * kRemoteSlices *
        // remote_cap, which is < 2^32 for the sharded id range)
        const unsigned long long bucket = static_cast<unsigned long long>(lane) * kRemoteSlices + sl;
        const unsigned b0 = atomicAdd(a.remote_count + bucket * kCountStride, c);
        AMBER_DCHECK(static_cast<unsigned long long>(b0) + c <= a.remote_cap, "wealth: remote bucket slice overflow");
        st.base[wq][lane] = static_cast<unsigned long long>(b0) + c <= a.remote_cap
                                ? static_cast<unsigned>(bucket * a.remote_cap + b0)
                                : 0xffffffffu;  // impossible by the slice capacity; drop rather than overrun
    }
    __syncwarp();
    for (unsigned e = lane; e < qn; e += 32) {
        const unsigned mt = st.meta[wq][e], b = st.base[wq][mt >> 10];
        if (b != 0xffffffffu) a.remote_ids[b + (mt & 1023u)] = st.id[wq][e];
    }
    __syncwarp();  // the stage is rewritten by the next batch
    qn = 0;
}

// One launch of the step pipeline.  Thread layout: a warp owns a chunk of
// kQPT*32 quads (4 agents each); lane l takes quads chunk*kQPT*32 + j*32 + l,
// so every global load/store instruction of the warp is a contiguous 512-byte
// (w) or 64-byte (4-bit counters) segment.  FAST32: all ids < 2^32 (32-bit
// index arithmetic); REMOTE: receivers outside this shard are bucketed for
// the exchange instead of counted locally.
template <int B, bool APPLY, bool SCATTER, bool DIGEST, bool REMOTE, bool FAST32>
__global__ void __launch_bounds__(256, REMOTE ? AMBER_WEALTH_MINB_REMOTE : AMBER_WEALTH_MINB) wealth_step_kernel(const WealthArgs a)
{
    using Id = typename std::conditional<FAST32, uint32_t, unsigned long long>::type;
    if (a.slot_zero && blockIdx.x == 0 && threadIdx.x == 0) *a.slot_zero = Slot{0, 0, 0, 0, 0};

    const int lane = threadIdx.x & 31;
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const unsigned long long pol = policy_evict_last();
    const Id lo = static_cast<Id>(a.lo), n_loc = static_cast<Id>(a.n_loc);
    const Id slo = REMOTE ? lo : static_cast<Id>(a.slo);
    const unsigned long long slim = REMOTE ? a.n_loc : a.slim;
    const unsigned long long m = a.n_glob - (a.exclude_self ? 1 : 0);
    unsigned long long tot = 0, dig = 0;
    uint32_t act = 0, sent = 0, got = 0;
    RemoteStage* stg = nullptr;
    if constexpr (REMOTE) {
        __shared__ RemoteStage st_;
        stg = &st_;
    }
    const int wq = threadIdx.x >> 5;
    const bool staged = REMOTE && a.world <= 32 && blockDim.x <= 256;
    unsigned qn = 0;  // staged remote receivers of this warp (warp-uniform)
    if constexpr (REMOTE) {
        if (staged) stg->cnt[wq][lane] = 0u;
        __syncwarp();
    }

    for (int64_t chunk = warp; chunk < a.nchunks; chunk += nwarps) {
        const unsigned sl = REMOTE ? static_cast<unsigned>(chunk % kRemoteSlices) : 0u;
        int4 w[kQPT];
        uint32_t c[kQPT][4];
#pragma unroll
        for (int j = 0; j < kQPT; ++j) {
            const Id q = static_cast<Id>((chunk * kQPT + j) * 32 + lane);
            w[j] = __ldcs(reinterpret_cast<const int4*>(a.w_in) + q);  // streaming: evict-first
            if constexpr (APPLY) load_quad_counts<B>(a.inc_cur, q, c[j]);
        }
        int32_t tsum = 0;
#pragma unroll
        for (int j = 0; j < kQPT; ++j) {
            const Id q = static_cast<Id>((chunk * kQPT + j) * 32 + lane);
            int32_t v[4] = {w[j].x, w[j].y, w[j].z, w[j].w};
            if constexpr (APPLY) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int32_t s = v[k] >= a.amount ? a.amount : 0;
                    v[k] = v[k] - s + a.amount * static_cast<int32_t>(c[j][k]);
                    got += c[j][k];
                }
                __stcs(reinterpret_cast<int4*>(a.w_out) + q, make_int4(v[0], v[1], v[2], v[3]));
                zero_quad_counts<B>(a.inc_cur, q);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    tsum += v[k];
                    act += v[k] > 0;
                    if constexpr (DIGEST) {
                        const Id loc = 4 * q + k;
                        if (loc < n_loc)
                            dig += digest_term(a.lo + static_cast<unsigned long long>(loc),
                                               static_cast<uint32_t>(v[k]));
                    }
                }
            }
            if constexpr (SCATTER) {
                const Id i0 = lo + 4 * q;  // even: shards start at multiples of 8
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const uint4 x = stream_block(a.key, TAG_WEALTH_RECV, (i0 >> 1) + p, a.t_scatter);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const bool s = v[2 * p + h] >= a.amount;
                        const Id i = i0 + 2 * p + h;
                        const Id r = static_cast<Id>(receiver<FAST32>(lane64_of(x, h), i, m, a.exclude_self));
                        const Id rl = r - slo;
                        bool local = s;
                        if constexpr (REMOTE) local = s && rl < n_loc;
#ifndef AMBER_EXPERIMENT_NO_RED
                        if (local) add_count<B>(a.inc_next, rl, pol, slim);
#else
                        if (local && rl == ~Id(0)) add_count<B>(a.inc_next, rl, pol, slim);  // never: cost without REDs
#endif
                        sent += local;
                        if constexpr (REMOTE) {
                            if (staged) remote_stage(a, *stg, wq, qn, s && !local, r);
                            else remote_append(a, s && !local, r, sl);
                        }
                    }
                }
                if constexpr (REMOTE)
                    if (staged && ((j % kFlushQuads) == kFlushQuads - 1 || j == kQPT - 1)) remote_flush(a, *stg, wq, qn, sl);
            }
        }
        // per-chunk partial in 32 bits (at most 16 agents' wealth), then widen
        tot += static_cast<unsigned long long>(static_cast<long long>(tsum));
    }

    unsigned long long vals[5] = {tot, act, dig, sent, got};
    unsigned long long* const outs[5] = {
        APPLY ? &a.slot_apply->total : nullptr, APPLY ? &a.slot_apply->active : nullptr,
        (APPLY && DIGEST) ? &a.slot_apply->digest : nullptr, SCATTER ? &a.slot_scatter->sent : nullptr,
        APPLY ? &a.slot_apply->got : nullptr};
    block_sum_atomic<5>(vals, outs);
}


// Small populations (C1): every step of a call in ONE single-CTA launch.  The
// wealth column and exact 32-bit receiver counters live in shared memory, so
// a step costs two __syncthreads instead of a kernel launch, and no counter
// can overflow (sent == got by construction).
constexpr int kSmallMax = 16384;  // agents (64 KB column + 2 x 64 KB counters)

struct SmallArgs {
    PhiloxKey key;
    const int32_t* w_in;
    int32_t* w_out;
    int64_t n;                 // agents (single GPU)
    int32_t amount, exclude_self;
    uint32_t t0;
    int64_t steps;
    Slot* ring;
    int64_t ring_cap;
    int digest;
};

// One __syncthreads per step: a thread applies step t to its own agent pairs
// (the counts of step t were completed before the barrier), then immediately
// scatters step t+1 from the new wealth of the same pair into the other
// counter buffer and re-zeroes its entries of this one; per-step observables
// are warp-reduced into shared accumulators (three rotating sets: step t's
// values are complete after the barrier while steps t+1, t+2 accumulate) and
// written to the ring by thread 0.
__global__ void __launch_bounds__(1024, 1) wealth_small_kernel(const SmallArgs a)
{
    extern __shared__ __align__(16) int32_t sw[];
    uint32_t* cnt0 = reinterpret_cast<uint32_t*>(sw + kSmallMax);
    uint32_t* cnt1 = cnt0 + kSmallMax;
    // per-warp partial sums of the step records {total, active, digest, sent, got},
    // three rotating sets (step t's set is next written by step t + 3); plain
    // stores by each warp's lane 0 and one 32-way sum per field after the
    // step's barrier (shared 64-bit atomics are CAS loops: 16 contending warps
    // cost ~1 us per step)
    __shared__ unsigned long long part[3][32][5];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = (nt + 31) >> 5;
    const uint32_t n = static_cast<uint32_t>(a.n);
    const unsigned long long m = a.n - (a.exclude_self ? 1 : 0);
    for (uint32_t i = tid; i < n; i += nt) {
        sw[i] = a.w_in[i];
        cnt0[i] = 0u;
        cnt1[i] = 0u;
    }
    for (int k = tid; k < 3 * 32 * 5; k += nt) (&part[0][0][0])[k] = 0ull;
    __syncthreads();
    // scatter of step t from the pair (i0, i0 + 1) with wealth (v0, v1)
    auto scatter = [&](uint32_t p, int32_t v0, int32_t v1, uint32_t t, uint32_t* cnt) -> unsigned long long {
        const uint32_t i0 = 2 * p;
        const bool s0 = v0 >= a.amount, s1 = (i0 + 1 < n) && v1 >= a.amount;
        unsigned long long sent = 0;
        if (s0 || s1) {
            const uint4 x = stream_block(a.key, TAG_WEALTH_RECV, p, t);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h ? s1 : s0) {
                    unsigned long long r = mulhi64(lane64_of(x, h), m);
                    if (a.exclude_self) r += (r >= i0 + h);
                    AMBER_DCHECK(r < n, "wealth (small): receiver >= n");
                    atomicAdd(cnt + r, 1u);
                    ++sent;
                }
            }
        }
        return sent;
    };
    const uint32_t npairs = (n + 1) / 2;
    const uint32_t ring_cap = static_cast<uint32_t>(a.ring_cap);
    uint32_t slot_idx = static_cast<uint32_t>(a.t0 % a.ring_cap);
    {   // prime: scatter of step t0
        unsigned long long sent = 0;
        for (uint32_t p = tid; p < npairs; p += nt)
            sent += scatter(p, sw[2 * p], 2 * p + 1 < n ? sw[2 * p + 1] : 0, a.t0, (a.t0 & 1) ? cnt1 : cnt0);
        const unsigned sw0 = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(sent));
        if (lane == 0) part[a.t0 % 3][warp][3] = sw0;
    }
    __syncthreads();
    for (int64_t k = 0; k < a.steps; ++k) {
        const uint32_t t = a.t0 + static_cast<uint32_t>(k);
        uint32_t* cur = (t & 1) ? cnt1 : cnt0;
        uint32_t* nxt = (t & 1) ? cnt0 : cnt1;
        const bool more = k + 1 < a.steps;
        unsigned long long tot = 0, act = 0, got = 0, dig = 0, sent = 0;
        for (uint32_t p = tid; p < npairs; p += nt) {
            int32_t v[2] = {0, 0};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t i = 2 * p + h;
                if (i >= n) continue;
                const uint32_t c = cur[i];
                cur[i] = 0u;
                int32_t x = sw[i];
                x = x - (x >= a.amount ? a.amount : 0) + a.amount * static_cast<int32_t>(c);
                sw[i] = x;
                v[h] = x;
                tot += static_cast<unsigned long long>(static_cast<long long>(x));
                act += x > 0;
                got += c;
                if (a.digest) dig += digest_term(i, static_cast<uint32_t>(x));
            }
            if (more) sent += scatter(p, v[0], v[1], t + 1, nxt);
        }
        // per-warp sums fit 32 bits (total wealth < 2^31 is checked at creation):
        // one REDUX each; only the digest needs a 64-bit shuffle reduction
        const int tw = __reduce_add_sync(0xffffffffu, static_cast<int>(static_cast<long long>(tot)));
        const unsigned aw = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(act));
        const unsigned gw = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(got));
        const unsigned sw_ = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(sent));
        if (a.digest) dig = warp_sum_u64(dig);
        if (lane == 0) {
            unsigned long long* x = part[t % 3][warp];
            x[0] = static_cast<unsigned long long>(static_cast<long long>(tw));
            x[1] = aw;
            x[2] = dig;
            x[4] = gw;
            part[(t + 1) % 3][warp][3] = sw_;
        }
        __syncthreads();
        if (tid < 5) {  // step t's record is complete
            unsigned long long v = 0;
            for (int w = 0; w < nwarps; ++w) v += part[t % 3][w][tid];
            (&a.ring[slot_idx].total)[tid] = v;
        }
        if (++slot_idx == ring_cap) slot_idx = 0;
    }
    for (uint32_t i = tid; i < n; i += nt) a.w_out[i] = sw[i];
}

// Received cross-shard receivers -> local counters of the scattered step.
template <int B>
__global__ void wealth_recv_kernel(const uint32_t* __restrict__ ids, const unsigned long long* __restrict__ n_ids,
                                   unsigned long long lo, unsigned long long n_loc, uint32_t* inc, Slot* slot)
{
    const unsigned long long n = *n_ids;
    unsigned long long cnt = 0;
    for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n;
         k += (unsigned long long)gridDim.x * blockDim.x) {
        add_count<B>(inc, static_cast<unsigned long long>(ids[k]) - lo, policy_evict_last(), n_loc);
        cnt += 1;
    }
    unsigned long long vals[1] = {cnt};
    unsigned long long* const outs[1] = {&slot->sent};
    block_sum_atomic<1>(vals, outs);
}

// P2P receive (fused transfer + apply): block row y = peer p; the bucket rank p
// filled for this rank in the scattered step's parity is read straight from
// p's memory (mapped over NVLink; __ldcv/__ldcs: never a stale cached copy)
// and applied to the local counters.
// gridDim.x is a multiple of kRemoteSlices: block x reads slice x %
// kRemoteSlices of the bucket, striding with the other x / kRemoteSlices blocks.
template <int B>
__global__ void wealth_recv_p2p_kernel(const unsigned long long* __restrict__ peer_base, int world, int me,
                                       size_t cnt_off, size_t ids_off, unsigned long long cap, unsigned long long lo,
                                       unsigned long long n_loc, uint32_t* inc, Slot* slot)
{
    const int p = blockIdx.y;
    unsigned long long got = 0;
    if (p != me) {
        const unsigned char* base = reinterpret_cast<const unsigned char*>(peer_base[p]);
        const unsigned sl = blockIdx.x % kRemoteSlices;
        const unsigned long long sub = blockIdx.x / kRemoteSlices, nsub = gridDim.x / kRemoteSlices;
        const unsigned long long bucket = static_cast<unsigned long long>(me) * kRemoteSlices + sl;
        const unsigned int n = __ldcv(reinterpret_cast<const unsigned int*>(base + cnt_off) + bucket * kCountStride);
        const unsigned long long m = n < cap ? n : cap;
        const uint32_t* ids = reinterpret_cast<const uint32_t*>(base + ids_off) + bucket * cap;
        for (unsigned long long k = sub * blockDim.x + threadIdx.x; k < m; k += nsub * blockDim.x) {
            add_count<B>(inc, static_cast<unsigned long long>(__ldcs(ids + k)) - lo, policy_evict_last(), n_loc);
            got += 1;
        }
    }
    unsigned long long vals[1] = {got};
    unsigned long long* const outs[1] = {&slot->sent};
    block_sum_atomic<1>(vals, outs);
}

// Dense exchange (AMBER_WEALTH_EXCHANGE=dense): every rank's fused step adds
// ALL its transfers into its own packed counters over the whole population
// (global index, no remote staging); after the barrier the owner sums the
// peers' packed words of its shard (plain 32-bit adds of the packed words: a
// carry shows up as a lower decoded total, caught by the global sent/got
// check) into its own counters, and zeroes its own other-parity global
// counters (last read by the owners before this barrier, next written by the
// next step).  peer_base[p] + dense_off = rank p's global counters of this parity.
__global__ void wealth_recv_dense_kernel(const unsigned long long* __restrict__ peer_base, int world,
                                         size_t dense_off, size_t word0, size_t words, uint32_t* __restrict__ inc_own,
                                         uint4* __restrict__ zero_own, size_t zero_n)
{
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
    // four words per thread per round: 4 x world independent loads in flight
    size_t w = tid;
    for (; w + 3 * nt < words; w += 4 * nt) {
        uint32_t v[4] = {0u, 0u, 0u, 0u};
        for (int p = 0; p < world; ++p) {
            const uint32_t* src =
                reinterpret_cast<const uint32_t*>(reinterpret_cast<const unsigned char*>(peer_base[p]) + dense_off) + word0;
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] += __ldcg(src + w + u * nt);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) inc_own[w + u * nt] = v[u];
    }
    for (; w < words; w += nt) {
        uint32_t v = 0;
        for (int p = 0; p < world; ++p)
            v += __ldcg(reinterpret_cast<const uint32_t*>(reinterpret_cast<const unsigned char*>(peer_base[p]) + dense_off) +
                        word0 + w);
        inc_own[w] = v;
    }
    for (size_t z = tid; z < zero_n; z += nt) zero_own[z] = make_uint4(0u, 0u, 0u, 0u);
}

// Sliced buckets -> contiguous per-destination blocks for the transports that
// ship one block per destination (NCCL send/recv, loopback and host-collective
// copies): block (x, p) copies slice x of destination p behind the slices
// before it; block 0 of each destination writes its total.
__global__ void wealth_compact_kernel(const uint32_t* __restrict__ ids, const unsigned int* __restrict__ cnt,
                                      unsigned long long cap, uint32_t* __restrict__ out,
                                      unsigned int* __restrict__ out_cnt, unsigned long long out_cap)
{
    const unsigned long long p = blockIdx.y;
    const int sl = blockIdx.x;
    __shared__ unsigned long long off_s, tot_s;
    if (threadIdx.x == 0) {
        unsigned long long off = 0, tot = 0;
        for (int k = 0; k < kRemoteSlices; ++k) {
            const unsigned long long c = cnt[(p * kRemoteSlices + k) * kCountStride];
            if (k < sl) off += c;
            tot += c;
        }
        off_s = off;
        tot_s = tot;
    }
    __syncthreads();
    const unsigned long long n = cnt[(p * kRemoteSlices + sl) * kCountStride];
    const uint32_t* src = ids + (p * kRemoteSlices + sl) * cap;
    uint32_t* dst = out + p * out_cap + off_s;
    for (unsigned long long k = threadIdx.x; k < n; k += blockDim.x) dst[k] = src[k];
    if (sl == 0 && threadIdx.x == 0) out_cnt[p] = static_cast<unsigned int>(tot_s);
}

// Fault injection (test hook, option "inject_counter_fault"): one extra count
// in the pending counters of local agent k -- a corrupted counter the exact
// overflow check (sent != got) must catch and the replay must repair.
__global__ void wealth_inject_kernel(uint32_t* inc, int64_t k, int B)
{
    const int per = 32 / B;
    atomicAdd(inc + k / per, 1u << (static_cast<uint32_t>(k % per) * B));
}

__global__ void wealth_fill_kernel(int32_t* w, int64_t n_loc, int64_t n_pad, int32_t w0)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pad; i += (int64_t)gridDim.x * blockDim.x)
        w[i] = i < n_loc ? w0 : 0;
}

__global__ void zero_slots_kernel(Slot* ring, int64_t cap, int64_t s0, int64_t count)
{
    for (int64_t k = threadIdx.x; k < count; k += blockDim.x) ring[(s0 + k) % cap] = Slot{0, 0, 0, 0, 0};
}

}  // namespace

// Host side of the cross-shard exchange (defined in dist.cu).
struct WealthExchange;
WealthExchange* make_wealth_exchange_rt(Runtime& rt, const amber_runtime* r);
void wealth_exchange_run(WealthExchange* x, Runtime& rt, const unsigned int* d_send_counts,
                         const uint32_t* d_send_ids, uint64_t send_cap, uint32_t* d_recv_ids,
                         unsigned long long* d_recv_total);
bool wealth_exchange_any(WealthExchange* x, Runtime& rt, bool local_flag);
void wealth_exchange_allreduce_u64(WealthExchange* x, Runtime& rt, unsigned long long* d_vals, int n);
void destroy_wealth_exchange(WealthExchange* x);
bool wealth_p2p_open(WealthExchange* x, Runtime& rt, void* my_base, std::vector<void*>& peers);
void wealth_p2p_barrier(WealthExchange* x, Runtime& rt);

class WealthModel final : public Model {
public:
    int64_t n = 0, lo = 0, hi = 0, n_loc = 0, n_pad = 0, shard = 0;
    amber_wealth_params p{};
    uint64_t seed = 0;
    PhiloxKey key{};
    int B = 4;
    bool fast32 = true;  // every id and padded index < 2^32 (32-bit index arithmetic)
    DevBuf<int32_t> wb[3];
    int cur = 0, pinned = -1;
    DevBuf<uint32_t> inc[2], inc32[2];
    bool pending = false;
    int64_t win_start = -1;
    DevBuf<Slot> ring;
    Slot* h_ring = nullptr;  // pinned host mirror of the ring (only the needed slots are copied)
    int64_t h_ring_cap = 0;
    int64_t h_lo = 0, h_hi = 0;  // slots [h_lo, h_hi) of the mirror are current
    int64_t m_first = 0, replays = 0;
    // cross-shard exchange (world > 1)
    WealthExchange* xch = nullptr;
    DevBuf<uint32_t> send_ids, recv_ids;
    DevBuf<unsigned int> send_counts;
    // P2P exchange (default when every rank can map its peers' buckets): both
    // parities' buckets in one cudaMalloc block (IPC-exportable)
    bool p2p = false, p2p_wanted = false;
    void* p2p_block = nullptr;
    size_t p2p_cnt_off[2] = {0, 0}, p2p_ids_off[2] = {0, 0};
    DevBuf<unsigned long long> p2p_peers;
    DevBuf<unsigned long long> recv_total;
    uint64_t send_cap = 0;    // ids per destination region (kRemoteSlices slices) and per compacted block
    uint64_t slice_cap = 0;   // ids per slice: every agent of the slice's warp chunks
    // dense exchange (AMBER_WEALTH_EXCHANGE=dense, P2P only): global packed counters
    // per parity inside the peer-mapped block
    bool dense_mode = false;
    size_t dense_off[2] = {0, 0}, dense_words = 0;
    DevBuf<unsigned long long> dsum;   // verify(): global sent / got sums
    DevBuf<uint32_t> cmp_ids;          // compacted per-destination blocks (non-P2P transports)
    DevBuf<unsigned int> cmp_counts;

    WealthModel(int64_t n_, const amber_wealth_params& p_, uint64_t seed_, const amber_runtime* r)
    {
        rt.init(r);
        n = n_;
        p = p_;
        seed = seed_;
        key = philox_key(seed);
        // 0: default = 4-bit packed counters with L2 atomics (the three atomic-free
        // scatters measured slower live in tools/experiments/)
        if (p.counter_bits == 0) p.counter_bits = 4;
        B = p.counter_bits;
        AMBER_REQUIRE(B == 2 || B == 4 || B == 8 || B == 16 || B == 32, "counter_bits must be 0, 2, 4, 8, 16 or 32");
        AMBER_REQUIRE(p.amount >= 1, "amount must be >= 1");
        AMBER_REQUIRE(p.w0 >= 0, "w0 must be >= 0");
        AMBER_REQUIRE(!p.exclude_self || n >= 2, "exclude_self needs n_agents >= 2");
        AMBER_REQUIRE(static_cast<double>(n) * p.w0 < 2147483647.0 || n == 1,
                      "n_agents * w0 must fit int32 wealth of a single agent");
        AMBER_REQUIRE(rt.world == 1 || n < (1ll << 32), "sharded wealth needs n_agents < 2^32");
        shard = ((ceil_div(n, rt.world) + 7) / 8) * 8;
        shard_range(n, rt.world, rt.rank, &lo, &hi);
        n_loc = hi - lo;
        n_pad = std::max<int64_t>(ceil_div(std::max<int64_t>(n_loc, 1), kChunkAgents) * kChunkAgents, kChunkAgents);
        fast32 = n < (1ll << 32) - 1 && lo + n_pad < (1ll << 32);
        AMBER_REQUIRE(fast32 || rt.world == 1, "sharded wealth needs ids < 2^32");
        for (auto& b : wb) b.allocate(&rt, n_pad);
        {
            const int64_t inc_words = ceil_div(n_pad * B, 32) + 4;
            for (auto& b : inc) {
                b.allocate(&rt, inc_words);
                b.zero_async(rt.stream);
            }
        }
        ring.allocate(&rt, metrics_cap);
        ring.zero_async(rt.stream);
        for (auto& b : wb) b.zero_async(rt.stream);
        wealth_fill_kernel<<<rt.num_sms * 4, 256, 0, rt.stream>>>(wb[0].p, n_loc, n_pad, p.w0);
        check_launch("wealth_fill_kernel");
        // AMBER_TEST_FORCE_EXCHANGE=1 with a unique id builds the exchange even for
        // world == 1 (a one-rank NCCL communicator): exercises the NCCL plumbing on one GPU
        const char* force = getenv("AMBER_TEST_FORCE_EXCHANGE");
        const bool force_x = force && force[0] == '1' && r && r->nccl_unique_id && rt.world == 1;
        if (rt.world > 1 || force_x) {
            xch = make_wealth_exchange_rt(rt, r);
            // same on every rank (from the common shard size): peers index each other's buckets
            const int64_t nch_max = ceil_div(std::max<int64_t>(shard, 1), kChunkAgents);
            slice_cap = static_cast<uint64_t>(ceil_div(nch_max, kRemoteSlices) * kChunkAgents);
            send_cap = slice_cap * kRemoteSlices;
            send_ids.allocate(&rt, send_cap * rt.world);
            recv_ids.allocate(&rt, static_cast<size_t>(shard) * rt.world + 1);
            send_counts.allocate(&rt, static_cast<int64_t>(rt.world) * kRemoteSlices * kCountStride);
            send_counts.zero_async(rt.stream);
            // AMBER_WEALTH_EXCHANGE: "dense" / "sparse" (P2P), "nccl"; default: P2P, dense
            // up to 8 ranks (one box; per-rank phases measured on one B200, DESIGN 7),
            // sparse buckets above (the dense payload does not shrink with the ranks)
            const char* mode = getenv("AMBER_WEALTH_EXCHANGE");
            const std::string ms = mode ? mode : "";
            p2p_wanted = ms != "nccl";  // mapped at the first exchange (collective)
            // (each shard's block of the global packed counters must start on a word:
            // shard * B a multiple of 32 -- always for B >= 4, shards being multiples of 8)
            dense_mode = rt.world > 1 && (ms == "dense" || (ms.empty() && rt.world <= 8)) && (shard * B) % 32 == 0;
            recv_total.allocate(&rt, 1);
        }
        rt.sync();
    }

    // Bucket block [counts par 0 | counts par 1 | ids par 0 | ids par 1] mapped into
    // every peer (dist.cu wealth_p2p_open); falls back to the NCCL send/recv
    // exchange if any rank cannot map its peers.
    void setup_p2p()
    {
        const size_t cbytes = ((static_cast<size_t>(rt.world) * kRemoteSlices * kCountStride * 4 + 255) / 256) * 256;
        const size_t ibytes = static_cast<size_t>(rt.world) * send_cap * 4;
        p2p_cnt_off[0] = 0;
        p2p_cnt_off[1] = cbytes;
        p2p_ids_off[0] = 2 * cbytes;
        p2p_ids_off[1] = 2 * cbytes + ibytes;
        // dense exchange: global packed counters (all N agents, B bits) per parity
        dense_words = dense_mode ? static_cast<size_t>(ceil_div(static_cast<int64_t>(rt.world) * shard * B, 32) + 8) : 0;
        dense_words = (dense_words + 3) / 4 * 4;  // whole uint4s (zeroing)
        dense_off[0] = 2 * cbytes + 2 * ibytes;
        dense_off[1] = dense_off[0] + dense_words * 4;
        const size_t total = 2 * cbytes + 2 * ibytes + 2 * dense_words * 4;
        if (cudaMalloc(&p2p_block, total) != cudaSuccess) {
            cudaGetLastError();
            p2p_block = nullptr;
        }
        if (p2p_block) AMBER_CUDA(cudaMemsetAsync(p2p_block, 0, 2 * cbytes, rt.stream));
        if (p2p_block && dense_words)
            AMBER_CUDA(cudaMemsetAsync(static_cast<char*>(p2p_block) + dense_off[0], 0, 2 * dense_words * 4, rt.stream));
        rt.sync();
        std::vector<void*> peers;
        if (p2p_block && wealth_p2p_open(xch, rt, p2p_block, peers)) {
            std::vector<unsigned long long> h(peers.size());
            for (size_t k = 0; k < peers.size(); ++k) h[k] = reinterpret_cast<unsigned long long>(peers[k]);
            p2p_peers.allocate(&rt, h.size());
            AMBER_CUDA(cudaMemcpyAsync(p2p_peers.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, rt.stream));
            rt.sync();
            p2p = true;
        } else if (p2p_block) {
            cudaFree(p2p_block);
            p2p_block = nullptr;
        }
    }

    uint32_t* dense_ctr(int par) { return reinterpret_cast<uint32_t*>(static_cast<char*>(p2p_block) + dense_off[par]); }
    unsigned int* p2p_counts(int par) { return reinterpret_cast<unsigned int*>(static_cast<char*>(p2p_block) + p2p_cnt_off[par]); }
    uint32_t* p2p_ids(int par) { return reinterpret_cast<uint32_t*>(static_cast<char*>(p2p_block) + p2p_ids_off[par]); }

    ~WealthModel() override
    {
        if (rt.stream) cudaStreamSynchronize(rt.stream);
        if (xch) destroy_wealth_exchange(xch);
        if (p2p_block) cudaFree(p2p_block);
        p2p_peers.reset();
        for (auto& b : wb) b.reset();
        for (auto& b : inc) b.reset();
        for (auto& b : inc32) b.reset();
        ring.reset();
        if (h_ring) cudaFreeHost(h_ring);
        send_ids.reset();
        recv_ids.reset();
        send_counts.reset();
        recv_total.reset();
        cmp_ids.reset();
        cmp_counts.reset();
        dsum.reset();
        rt.destroy();
    }

    int other(int a, int b) const
    {
        for (int k = 0; k < 3; ++k)
            if (k != a && k != b) return k;
        return -1;
    }

    Slot* slot(int64_t s) { return ring.p + (s % metrics_cap); }

    template <int BB, bool APPLY, bool SCATTER, bool DIGEST, bool REMOTE>
    void launch_inst(const WealthArgs& a)
    {
        constexpr bool kFast = true;
        auto kern = fast32 ? wealth_step_kernel<BB, APPLY, SCATTER, DIGEST, REMOTE, kFast>
                           : wealth_step_kernel<BB, APPLY, SCATTER, DIGEST, REMOTE, REMOTE>;
        int threads = block ? static_cast<int>(block) : 256;
        int g = static_cast<int>(grid);
        if (!g) {
            int per_sm = 0;
            AMBER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0));
            g = static_cast<int>(std::min<int64_t>(a.nchunks * 32 / threads + 1,
                                                   static_cast<int64_t>(std::max(per_sm, 1)) * rt.num_sms));
        }
        const char* name = APPLY ? (SCATTER ? "wealth_step_fused" : "wealth_apply") : "wealth_scatter";
        prof.launch(rt.stream, name, [&] { kern<<<g, threads, 0, rt.stream>>>(a); });
        check_launch(name);
    }

    template <int BB>
    void launch_b(const WealthArgs& a, bool apply, bool scatter, bool dig, bool remote)
    {
#define AMBER_W_DISPATCH(AP, SC)                                                         \
    if (apply == AP && scatter == SC) {                                                  \
        if (dig) {                                                                       \
            if (remote) launch_inst<BB, AP, SC, true, true>(a);                          \
            else launch_inst<BB, AP, SC, true, false>(a);                                \
        } else {                                                                         \
            if (remote) launch_inst<BB, AP, SC, false, true>(a);                         \
            else launch_inst<BB, AP, SC, false, false>(a);                               \
        }                                                                                \
        return;                                                                          \
    }
        AMBER_W_DISPATCH(true, true)
        AMBER_W_DISPATCH(false, true)
        AMBER_W_DISPATCH(true, false)
#undef AMBER_W_DISPATCH
    }

    // One launch: apply step ta (if apply) from wb[src] into wb[dst], scatter step ts (if scatter).
    void launch(int bits, bool exact, bool apply, bool scatter, int64_t ta, int64_t ts, int src, int dst)
    {
        DevBuf<uint32_t>* ib = exact ? inc32 : inc;
        WealthArgs a{};
        a.key = key;
        a.w_in = wb[src].p;
        a.w_out = apply ? wb[dst].p : nullptr;
        a.inc_cur = apply ? ib[ta & 1].p : nullptr;
        a.inc_next = scatter ? ib[ts & 1].p : nullptr;
        a.nchunks = n_pad / kChunkAgents;
        a.n_loc = n_loc;
        a.lo = static_cast<unsigned long long>(lo);
        a.n_glob = static_cast<unsigned long long>(n);
        a.amount = p.amount;
        a.exclude_self = p.exclude_self;
        a.t_apply = static_cast<uint32_t>(ta);
        a.t_scatter = static_cast<uint32_t>(ts);
        a.slot_apply = apply ? slot(ta) : nullptr;
        a.slot_scatter = scatter ? slot(ts) : nullptr;
        a.slot_zero = (apply && scatter) ? slot(ta + 2) : nullptr;
        a.slo = static_cast<unsigned long long>(lo);
        a.slim = static_cast<unsigned long long>(n_loc);
        bool remote = xch != nullptr && scatter;
        if (remote && p2p_wanted) {  // collective: every rank reaches its first exchange here
            p2p_wanted = false;
            setup_p2p();
        }
        const bool dense = remote && p2p && dense_mode && !exact;
        if (dense) {
            // all transfers into this rank's global counters of the scattered step's
            // parity (zeroed by the owner pass of the step before); no remote staging
            remote = false;
            a.inc_next = dense_ctr(ts & 1);
            a.slo = 0;
            a.slim = static_cast<unsigned long long>(rt.world) * static_cast<unsigned long long>(shard);
        }
        if (remote) {
            a.world = rt.world;
            a.shard_size = static_cast<unsigned long long>(shard);
            a.shard_magic = static_cast<uint32_t>(0xFFFFFFFFull / static_cast<unsigned long long>(shard));
            a.remote_ids = send_ids.p;
            a.remote_count = send_counts.p;
            a.remote_cap = slice_cap;
            if (p2p) {  // the scattered step's parity; its previous readers finished (barrier of ts - 1)
                a.remote_ids = p2p_ids(ts & 1);
                a.remote_count = p2p_counts(ts & 1);
                AMBER_CUDA(cudaMemsetAsync(a.remote_count, 0,
                                           static_cast<size_t>(rt.world) * kRemoteSlices * kCountStride * sizeof(unsigned int),
                                           rt.stream));
            } else {
                send_counts.zero_async(rt.stream);
            }
        }
        const bool dig = digest_on != 0;
        switch (bits) {
            case 2: launch_b<2>(a, apply, scatter, dig, remote); break;
            case 4: launch_b<4>(a, apply, scatter, dig, remote); break;
            case 8: launch_b<8>(a, apply, scatter, dig, remote); break;
            case 16: launch_b<16>(a, apply, scatter, dig, remote); break;
            default: launch_b<32>(a, apply, scatter, dig, remote); break;
        }
        if (remote) exchange(bits, exact, ts);
        if (dense) exchange_dense(bits, ts);
    }

    // Dense exchange of step ts: after the barrier, this rank's counters of ts =
    // the sum of every rank's global counters over its shard (read in place over
    // the peer mappings); its own other-parity global counters are zeroed.
    void exchange_dense(int bits, int64_t ts)
    {
        wealth_p2p_barrier(xch, rt);
        const size_t word0 = static_cast<size_t>(lo) * bits / 32;
        const size_t words = static_cast<size_t>(ceil_div(n_loc * bits, 32));
        const int g = rt.num_sms * 4;
        prof.launch(rt.stream, "wealth_recv_dense", [&] {
            wealth_recv_dense_kernel<<<g, 256, 0, rt.stream>>>(p2p_peers.p, rt.world, dense_off[ts & 1], word0, words,
                                                               inc[ts & 1].p, reinterpret_cast<uint4*>(dense_ctr((ts + 1) & 1)),
                                                               dense_words / 4);
        });
        check_launch("wealth_recv_dense_kernel");
    }

    // Cross-shard step: ship remote receivers to their owners, add them to the
    // owners' counters of step ts.
    void exchange(int bits, bool exact, int64_t ts)
    {
        DevBuf<uint32_t>* ib = exact ? inc32 : inc;
        if (p2p) {
            wealth_p2p_barrier(xch, rt);
            auto launch_p2p = [&](auto kern) {
                // a multiple of kRemoteSlices blocks per peer (the kernel's slice mapping)
                const int per = std::max(1, rt.num_sms * 8 / std::max(rt.world - 1, 1) / kRemoteSlices);
                const dim3 g(static_cast<unsigned>(per * kRemoteSlices), static_cast<unsigned>(rt.world));
                prof.launch(rt.stream, "wealth_recv_p2p", [&] {
                    kern<<<g, 256, 0, rt.stream>>>(p2p_peers.p, rt.world, rt.rank, p2p_cnt_off[ts & 1],
                                                   p2p_ids_off[ts & 1], static_cast<unsigned long long>(slice_cap),
                                                   static_cast<unsigned long long>(lo),
                                                   static_cast<unsigned long long>(n_loc), ib[ts & 1].p, slot(ts));
                });
                check_launch("wealth_recv_p2p_kernel");
            };
            switch (bits) {
                case 2: launch_p2p(wealth_recv_p2p_kernel<2>); break;
                case 4: launch_p2p(wealth_recv_p2p_kernel<4>); break;
                case 8: launch_p2p(wealth_recv_p2p_kernel<8>); break;
                case 16: launch_p2p(wealth_recv_p2p_kernel<16>); break;
                default: launch_p2p(wealth_recv_p2p_kernel<32>); break;
            }
            return;
        }
        if (!cmp_ids.p) {
            cmp_ids.allocate(&rt, send_cap * rt.world);
            cmp_counts.allocate(&rt, rt.world);
        }
        prof.launch(rt.stream, "wealth_compact", [&] {
            wealth_compact_kernel<<<dim3(kRemoteSlices, rt.world), 256, 0, rt.stream>>>(
                send_ids.p, send_counts.p, static_cast<unsigned long long>(slice_cap), cmp_ids.p, cmp_counts.p,
                static_cast<unsigned long long>(send_cap));
        });
        check_launch("wealth_compact_kernel");
        wealth_exchange_run(xch, rt, cmp_counts.p, cmp_ids.p, send_cap, recv_ids.p, recv_total.p);
        auto launch_recv = [&](auto kern) {
            prof.launch(rt.stream, "wealth_recv_apply", [&] {
                kern<<<rt.num_sms * 4, 256, 0, rt.stream>>>(recv_ids.p, recv_total.p,
                                                          static_cast<unsigned long long>(lo),
                                                          static_cast<unsigned long long>(n_loc), ib[ts & 1].p,
                                                          slot(ts));
            });
            check_launch("wealth_recv_kernel");
        };
        switch (bits) {
            case 2: launch_recv(wealth_recv_kernel<2>); break;
            case 4: launch_recv(wealth_recv_kernel<4>); break;
            case 8: launch_recv(wealth_recv_kernel<8>); break;
            case 16: launch_recv(wealth_recv_kernel<16>); break;
            default: launch_recv(wealth_recv_kernel<32>); break;
        }
    }

    void zero_slots(int64_t s0, int64_t count)
    {
        zero_slots_kernel<<<1, 64, 0, rt.stream>>>(ring.p, metrics_cap, s0, count);
        check_launch("zero_slots_kernel");
    }

    bool small_path() const { return rt.world == 1 && !xch && n <= kSmallMax && persistent; }

    void step(int64_t nsteps) override
    {
        AMBER_REQUIRE(nsteps >= 0, "n_steps must be >= 0");
        h_hi = h_lo;  // the ring changes: the host mirror is stale
        AMBER_REQUIRE(t + nsteps < (1ll << 32) - 2, "step index would exceed 2^32");
        if (small_path() && nsteps > 0) {
            // no pending scatter across calls on this path; flush any from the large path
            verify();
            invalidate_pending();
            int64_t done = 0;
            while (done < nsteps) {
                const int64_t chunk = std::min<int64_t>(nsteps - done, metrics_cap - 4);
                SmallArgs a{key, wb[cur].p, wb[other(cur, -1)].p, n, p.amount, p.exclude_self,
                            static_cast<uint32_t>(t), chunk, ring.p, metrics_cap, digest_on ? 1 : 0};
                const size_t smem = static_cast<size_t>(kSmallMax) * 12;  // column + two counter buffers
                AMBER_CUDA(cudaFuncSetAttribute(wealth_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                static_cast<int>(smem)));
                // one thread per agent pair (R4: one Philox block feeds a pair)
                int threads = static_cast<int>(std::min<int64_t>(1024, std::max<int64_t>(32, ceil_div((n + 1) / 2, 32) * 32)));
                if (block) threads = static_cast<int>(block);
                prof.launch(rt.stream, "wealth_small_persistent", [&] {
                    wealth_small_kernel<<<1, threads, smem, rt.stream>>>(a);
                });
                check_launch("wealth_small_kernel");
                cur = other(cur, -1);
                t += chunk;
                done += chunk;
            }
            return;
        }
        for (int64_t k = 0; k < nsteps; ++k) {
            if (win_start >= 0 && t - win_start >= metrics_cap - 4) verify();
            if (win_start < 0) {
                win_start = t;
                pinned = cur;
            }
            if (!pending) {
                zero_slots(t, 2);
                launch(B, false, false, true, t, t, cur, cur);
            }
            const int dst = other(cur, pinned == cur ? -1 : pinned);
            launch(B, false, true, true, t, t + 1, cur, dst);
            cur = dst;
            ++t;
            pending = true;
        }
    }

    // Copy ring slots [s0, s1) into the pinned mirror (same slot positions; at most
    // two contiguous pieces) and wait: per-step reads move only the slots they use.
    const Slot* fetch_slots(int64_t s0, int64_t s1)
    {
        if (h_ring_cap == metrics_cap && s0 >= h_lo && s1 <= h_hi) return h_ring;  // fetched since the last step
        if (h_ring_cap != metrics_cap) {
            if (h_ring) cudaFreeHost(h_ring);
            AMBER_CUDA(cudaMallocHost(&h_ring, metrics_cap * sizeof(Slot)));
            h_ring_cap = metrics_cap;
        }
        if (s1 > s0) {
            if (s1 - s0 >= metrics_cap) {
                AMBER_CUDA(cudaMemcpyAsync(h_ring, ring.p, metrics_cap * sizeof(Slot), cudaMemcpyDeviceToHost, rt.stream));
            } else {
                const int64_t a = s0 % metrics_cap, b = (s1 - 1) % metrics_cap;
                if (a <= b) {
                    AMBER_CUDA(cudaMemcpyAsync(h_ring + a, ring.p + a, (b - a + 1) * sizeof(Slot), cudaMemcpyDeviceToHost,
                                               rt.stream));
                } else {
                    AMBER_CUDA(cudaMemcpyAsync(h_ring + a, ring.p + a, (metrics_cap - a) * sizeof(Slot),
                                               cudaMemcpyDeviceToHost, rt.stream));
                    AMBER_CUDA(cudaMemcpyAsync(h_ring, ring.p, (b + 1) * sizeof(Slot), cudaMemcpyDeviceToHost, rt.stream));
                }
            }
        }
        rt.sync();
        h_lo = s0;
        h_hi = s1;
        return h_ring;
    }

    // Exact overflow check of the open window; replays it with 32-bit counters if needed.
    void verify()
    {
        if (win_start < 0) {
            rt.sync();
            return;
        }
        const Slot* h = fetch_slots(win_start, t);
        bool bad = false;
        if (dense_mode && p2p) {
            // dense exchange: a rank's increments land on other ranks' agents, so
            // only the global totals match (a carry lowers the decoded total)
            unsigned long long v[2] = {0, 0};
            for (int64_t s = win_start; s < t; ++s) {
                v[0] += h[s % metrics_cap].sent;
                v[1] += h[s % metrics_cap].got;
            }
            if (!dsum.p) dsum.allocate(&rt, 2);
            AMBER_CUDA(cudaMemcpyAsync(dsum.p, v, sizeof(v), cudaMemcpyHostToDevice, rt.stream));
            wealth_exchange_allreduce_u64(xch, rt, dsum.p, 2);
            AMBER_CUDA(cudaMemcpyAsync(v, dsum.p, sizeof(v), cudaMemcpyDeviceToHost, rt.stream));
            rt.sync();
            bad = v[0] != v[1];
        } else {
            for (int64_t s = win_start; s < t; ++s) {
                const Slot& x = h[s % metrics_cap];
                if (x.sent != x.got) bad = true;
            }
            if (xch) bad = wealth_exchange_any(xch, rt, bad);
        }
        if (bad) replay(win_start, t);
        win_start = -1;
        pinned = -1;
    }

    void replay(int64_t s0, int64_t s1)
    {
        ++replays;
        h_hi = h_lo;
        cur = pinned;
        for (auto& b : inc) b.zero_async(rt.stream);
        for (auto& b : inc32) {
            if (!b.p) b.allocate(&rt, n_pad + 4);
            b.zero_async(rt.stream);
        }
        ring.zero_async(rt.stream);
        if (xch) send_counts.zero_async(rt.stream);
        if (p2p) AMBER_CUDA(cudaMemsetAsync(p2p_block, 0, p2p_ids_off[0], rt.stream));
        if (p2p && dense_words)
            AMBER_CUDA(cudaMemsetAsync(dense_ctr(0), 0, 2 * dense_words * 4, rt.stream));
        for (int64_t s = s0; s < s1; ++s) {
            if (s == s0) launch(32, true, false, true, s, s, cur, cur);
            const int dst = other(cur, -1);
            launch(32, true, true, s + 1 < s1, s, s + 1, cur, dst);
            cur = dst;
        }
        t = s1;
        pending = false;
        std::vector<Slot> h(metrics_cap);
        AMBER_CUDA(cudaMemcpyAsync(h.data(), ring.p, metrics_cap * sizeof(Slot), cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        for (int64_t s = s0; s < s1; ++s)
            if (h[s % metrics_cap].sent != h[s % metrics_cap].got)
                fail(AMBER_E_CUDA, "wealth replay: increment count mismatch with 32-bit counters");
        if (m_first < s0) m_first = s0;  // earlier records were cleared with the ring
    }

    void invalidate_pending()
    {
        if (pending) {
            if (inc[t & 1].p) inc[t & 1].zero_async(rt.stream);
            pending = false;
        }
    }

    void synchronize() override { verify(); }

    bool column_info(const char* name, amber_dtype* dt, int64_t* glen, int64_t* off, int64_t* len) override
    {
        if (std::string(name) != "wealth") return false;
        if (dt) *dt = AMBER_I32;
        if (glen) *glen = n;
        if (off) *off = lo;
        if (len) *len = n_loc;
        return true;
    }

    void read_column(const char* name, void* dst, size_t bytes, bool on_dev) override
    {
        if (std::string(name) != "wealth") fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        if (bytes < static_cast<size_t>(n_loc) * 4) fail(AMBER_E_BUFFER_TOO_SMALL, "dst too small for wealth slice");
        verify();
        copy_out(rt, dst, wb[cur].p, n_loc * 4, on_dev);
    }

    void write_column(const char* name, const void* src, size_t bytes, bool on_dev) override
    {
        if (std::string(name) != "wealth") fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        if (bytes < static_cast<size_t>(n_loc) * 4) fail(AMBER_E_BUFFER_TOO_SMALL, "src smaller than wealth slice");
        verify();
        invalidate_pending();
        copy_in(rt, wb[cur].p, src, n_loc * 4, on_dev);
    }

    void read_metrics(const char* name, void* dst, size_t bytes, int64_t* n_out) override
    {
        verify();
        std::string k(name);
        size_t off;
        if (k == "total_wealth") off = offsetof(Slot, total);
        else if (k == "active") off = offsetof(Slot, active);
        else if (k == "digest" && digest_on) off = offsetof(Slot, digest);
        else fail(AMBER_E_UNKNOWN_NAME, "no metric " + k + (k == "digest" ? " (set option digest=1)" : ""));
        const int64_t first = std::max(m_first, t - metrics_cap + 3);
        const int64_t cnt = std::max<int64_t>(t - first, 0);
        const Slot* h = fetch_slots(first, t);
        if (bytes < static_cast<size_t>(cnt) * 8) fail(AMBER_E_BUFFER_TOO_SMALL, "metrics dst too small");
        std::vector<unsigned long long> vals(cnt);
        for (int64_t s = first; s < t; ++s)
            std::memcpy(&vals[s - first], reinterpret_cast<const char*>(&h[s % metrics_cap]) + off, 8);
        if (xch && cnt) {  // global values: sum over ranks
            DevBuf<unsigned long long> d;
            d.allocate(&rt, cnt);
            AMBER_CUDA(cudaMemcpyAsync(d.p, vals.data(), cnt * 8, cudaMemcpyHostToDevice, rt.stream));
            wealth_exchange_allreduce_u64(xch, rt, d.p, static_cast<int>(cnt));
            AMBER_CUDA(cudaMemcpyAsync(vals.data(), d.p, cnt * 8, cudaMemcpyDeviceToHost, rt.stream));
            rt.sync();
        }
        std::memcpy(dst, vals.data(), cnt * 8);
        if (n_out) *n_out = cnt;
    }

    void reset_metrics() override
    {
        verify();
        m_first = t;
    }

    uint64_t digest(const char* name) override
    {
        if (std::string(name) != "wealth") fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        verify();
        uint64_t d = device_digest_u32(rt, reinterpret_cast<const uint32_t*>(wb[cur].p), n_loc, lo);
        if (xch) {
            DevBuf<unsigned long long> b;
            b.allocate(&rt, 1);
            AMBER_CUDA(cudaMemcpyAsync(b.p, &d, 8, cudaMemcpyHostToDevice, rt.stream));
            wealth_exchange_allreduce_u64(xch, rt, b.p, 1);
            AMBER_CUDA(cudaMemcpyAsync(&d, b.p, 8, cudaMemcpyDeviceToHost, rt.stream));
            rt.sync();
        }
        return d;
    }

    void set_step(int64_t s) override
    {
        AMBER_REQUIRE(s >= 0 && s < (1ll << 32) - 2, "step out of range");
        verify();
        invalidate_pending();
        t = s;
        m_first = s;
    }

    bool set_option(const char* key, int64_t v) override
    {
        std::string k(key);
        if (k == "inject_counter_fault") {  // test hook: corrupt one pending counter (fault injection)
            AMBER_REQUIRE(pending && v >= 0 && v < n_loc, "inject_counter_fault needs a pending scatter and 0 <= v < n_loc");
            wealth_inject_kernel<<<1, 1, 0, rt.stream>>>(inc[t & 1].p, v, B);
            check_launch("wealth_inject_kernel");
            return true;
        }
        if (k == "metrics_capacity") {
            AMBER_REQUIRE(v >= 16, "metrics_capacity must be >= 16");
            verify();
            invalidate_pending();
            metrics_cap = v;
            ring.allocate(&rt, metrics_cap);
            ring.zero_async(rt.stream);
            m_first = t;
            return true;
        }
        if (k == "block") AMBER_REQUIRE(v <= 256, "wealth kernels are built for <= 256 threads per block");
        if (k == "digest" || k == "block" || k == "grid") verify();
        return Model::set_option(key, v);
    }

    bool get_option(const char* key, int64_t* v) override
    {
        std::string k(key);
        if (k == "replays") {
            verify();
            *v = replays;
            return true;
        }
        if (k == "counter_bits") {
            *v = B;
            return true;
        }
        if (k == "exchange") {  // 0: none (one rank), 1: NCCL send/recv, 2: P2P (peer-mapped buckets), 3: dense
            *v = xch ? (p2p ? (dense_mode ? 3 : 2) : 1) : 0;
            return true;
        }
        if (k == "scatter") {  // 1: packed-counter L2 atomics (the one shipped scatter)
            *v = 1;
            return true;
        }
        return Model::get_option(key, v);
    }
};

Model* make_wealth(int64_t n, const amber_wealth_params& p, uint64_t seed, const amber_runtime* rt)
{
    return new WealthModel(n, p, seed, rt);
}

}  // namespace amber
