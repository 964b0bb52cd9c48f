// wealth_bins.cu -- range-partitioned scatter for the wealth step (default on
// one GPU).
//
// The packed-counter kernel (wealth.cu) issues one random L2 atomic per
// sender; at N = 1e8 those 6e7 REDs per step (half of them forwarded across
// the die fabric) saturate the L2 tag pipeline long before HBM.  Here the
// scatter is a counting sort instead:
//
//  produce (wealth_bin_kernel, 1 CTA/SM, ~210 KB shared memory): a CTA takes a
//    tile of 32768 agents, computes the Philox receivers of its senders,
//    stages them in shared memory, counting-sorts them by 2^16-agent range,
//    reserves one contiguous run per range with a single global atomic, and
//    writes each run as a contiguous burst of 16-bit offsets.
//  apply (wealth_binapply_kernel, several CTAs/SM, 64 KB shared memory): a
//    CTA takes one range, builds the per-agent counts of that range in a
//    shared-memory histogram (8-bit counters, 4 per word) from the range's
//    bin, then streams the range's wealth: w' = w - a*s + a*c.
//
// Exactness: entries beyond a bin's capacity are dropped and an 8-bit count
// >= 256 carries; both make the decoded total of the step (`got`) smaller
// than the number of entries produced (`sent`), which the model checks and
// answers with an exact replay (wealth.cu).
#include <algorithm>
#include <cub/block/block_scan.cuh>

#include "wealth_experiments.cuh"

namespace amber {

namespace {

constexpr int kProdThreads = 1024;
constexpr int kMaxBins = 4096;

struct ProdArgs {
    PhiloxKey key;
    const int32_t* w;
    int64_t n_loc;           // agents of this shard (w padded with zeros beyond)
    unsigned long long lo, m;  // global id of local agent 0; receiver modulus (N or N-1)
    int32_t amount, exclude_self;
    uint32_t t;
    uint16_t* data;
    uint32_t* cnt;
    uint32_t cap;
    int K, tile;
    int64_t n_tiles;
    int* queue;              // queue[0]: tile counter (this launch), queue[1]: apply counter (reset here)
    WealthSlot* slot;
};

__global__ void __launch_bounds__(kProdThreads, 1) wealth_bin_kernel(const ProdArgs a)
{
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* stage = smem;                                             // tile entries (global receiver ids)
    uint16_t* sorted = reinterpret_cast<uint16_t*>(stage + a.tile);     // tile offsets, grouped by range
    uint32_t* bcnt = reinterpret_cast<uint32_t*>(sorted + a.tile);      // K
    uint32_t* bstart = bcnt + a.K;                                      // K
    uint32_t* bcur = bstart + a.K;                                      // K
    uint32_t* gbase = bcur + a.K;                                       // K
    __shared__ int tile_s;
    __shared__ uint32_t nstage;
    using Scan = cub::BlockScan<uint32_t, kProdThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    const int tid = threadIdx.x, lane = tid & 31;
    const int per_thread = (a.K + kProdThreads - 1) / kProdThreads;
    if (blockIdx.x == 0 && tid == 0) a.queue[1] = 0;  // apply queue of this step (runs after us)
    unsigned long long sent = 0;

    for (;;) {
        if (tid == 0) {
            tile_s = atomicAdd(a.queue, 1);
            nstage = 0;
        }
        for (int b = tid; b < a.K; b += kProdThreads) bcnt[b] = 0;
        __syncthreads();
        const int64_t tile = tile_s;
        if (tile >= a.n_tiles) break;
        // 1) receivers of this tile's senders -> stage (warp-aggregated append)
        const int64_t q0 = tile * (a.tile / 4);
        for (int qi = tid; qi < a.tile / 4; qi += kProdThreads) {
            const int64_t q = q0 + qi;
            const int4 w4 = __ldcs(reinterpret_cast<const int4*>(a.w) + q);
            const int32_t v[4] = {w4.x, w4.y, w4.z, w4.w};
            const unsigned long long i0 = a.lo + 4ull * static_cast<unsigned long long>(q);
            const uint4 x0 = stream_block(a.key, TAG_WEALTH_RECV, (i0 >> 1), a.t);
            const uint4 x1 = stream_block(a.key, TAG_WEALTH_RECV, (i0 >> 1) + 1, a.t);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const bool s = v[h] >= a.amount;
                const unsigned long long x = lane64_of(h < 2 ? x0 : x1, h & 1);
                unsigned long long r = (a.m >> 32) ? mulhi64(x, a.m) : mulhi64_n32(x, static_cast<uint32_t>(a.m));
                if (a.exclude_self) r += (r >= i0 + h);
                const unsigned mask = __ballot_sync(0xffffffffu, s);
                uint32_t base = 0;
                if (lane == 0 && mask) base = atomicAdd(&nstage, static_cast<uint32_t>(__popc(mask)));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (s) {
                    stage[base + __popc(mask & ((1u << lane) - 1u))] = static_cast<uint32_t>(r);
                    atomicAdd(&bcnt[r >> kBinShift], 1u);
                }
            }
        }
        __syncthreads();
        // 2) exclusive scan of the per-range counts; reserve one run per range
        {
            uint32_t loc[kMaxBins / kProdThreads];
            uint32_t sum = 0;
#pragma unroll
            for (int j = 0; j < kMaxBins / kProdThreads; ++j) {
                const int b = tid * per_thread + j;
                loc[j] = (j < per_thread && b < a.K) ? bcnt[b] : 0u;
                sum += loc[j];
            }
            uint32_t ex;
            Scan(scan_tmp).ExclusiveSum(sum, ex);
#pragma unroll
            for (int j = 0; j < kMaxBins / kProdThreads; ++j) {
                const int b = tid * per_thread + j;
                if (j < per_thread && b < a.K) {
                    bstart[b] = ex;
                    bcur[b] = ex;
                    gbase[b] = loc[j] ? atomicAdd(a.cnt + b, loc[j]) : 0u;
                    ex += loc[j];
                }
            }
        }
        __syncthreads();
        // 3) counting-sort placement (offsets within the range)
        const uint32_t ns = nstage;
        for (uint32_t e = tid; e < ns; e += kProdThreads) {
            const uint32_t r = stage[e];
            const uint32_t pos = atomicAdd(&bcur[r >> kBinShift], 1u);
            sorted[pos] = static_cast<uint16_t>(r & (kBinRange - 1));
        }
        __syncthreads();
        // 4) flush: one contiguous run per range (a warp per range)
        for (int b = tid >> 5; b < a.K; b += kProdThreads >> 5) {
            const uint32_t c = bcnt[b];
            if (!c) continue;
            const uint32_t g0 = gbase[b], s0 = bstart[b];
            uint16_t* dst = a.data + static_cast<size_t>(b) * a.cap;
            for (uint32_t k = lane; k < c; k += 32)
                if (g0 + k < a.cap) dst[g0 + k] = sorted[s0 + k];
        }
        if (tid == 0) sent += ns;
        __syncthreads();
    }
    if (tid == 0 && sent) atomicAdd(&a.slot->sent, sent);
}

struct ApplyArgs {
    const int32_t* w_in;
    int32_t* w_out;
    const uint16_t* data;
    uint32_t* cnt;
    uint32_t cap;
    int k0, k_loc;
    int64_t n_loc;
    unsigned long long lo;
    int32_t amount;
    int digest;
    int* queue;               // queue[1]: range counter (this launch), queue[0]: tile counter (reset here)
    WealthSlot* slot;         // record of this step
    WealthSlot* slot_next;    // zeroed here (next step's record)
};

template <bool DIGEST>
__global__ void __launch_bounds__(512, 3) wealth_binapply_kernel(const ApplyArgs a)
{
    extern __shared__ __align__(16) uint32_t hist[];  // 2^16 8-bit counters, 4 per word
    __shared__ int range_s;
    const int tid = threadIdx.x, nt = blockDim.x;
    if (blockIdx.x == 0 && tid == 0) {
        a.queue[0] = 0;  // next step's production queue
        if (a.slot_next) *a.slot_next = WealthSlot{0, 0, 0, 0, 0};
    }
    unsigned long long tot = 0, act = 0, got = 0, dig = 0;
    constexpr int kWords = static_cast<int>(kBinRange / 4);
    for (;;) {
        if (tid == 0) range_s = atomicAdd(a.queue + 1, 1);
        for (int j = tid; j < kWords; j += nt) hist[j] = 0u;
        __syncthreads();
        const int k = range_s;
        if (k >= a.k_loc) break;
        const int kg = a.k0 + k;
        // 1) histogram of this range's entries
        const uint32_t c = min(a.cnt[kg], a.cap);
        const uint16_t* src = a.data + static_cast<size_t>(kg) * a.cap;
        for (uint32_t e = tid; e < c; e += nt) {
            const uint32_t off = src[e];
            atomicAdd(&hist[off >> 2], 1u << ((off & 3u) * 8u));
        }
        __syncthreads();
        if (tid == 0) a.cnt[kg] = 0;  // this parity's bin is empty again
        // 2) stream the range: quad j of the range <-> hist word j
        const int64_t q0 = static_cast<int64_t>(k) * kWords;
        int32_t tsum = 0;
#pragma unroll 4
        for (int j = tid; j < kWords; j += nt) {
            const int4 w4 = __ldcs(reinterpret_cast<const int4*>(a.w_in) + q0 + j);
            const uint32_t h = hist[j];
            int32_t v[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int32_t ci = static_cast<int32_t>((h >> (8 * i)) & 255u);
                v[i] = v[i] - (v[i] >= a.amount ? a.amount : 0) + a.amount * ci;
                tsum += v[i];
                act += v[i] > 0;
                got += static_cast<unsigned>(ci);
                if constexpr (DIGEST) {
                    const int64_t loc = 4 * (q0 + j) + i;
                    if (loc < a.n_loc)
                        dig += digest_term(a.lo + static_cast<unsigned long long>(loc), static_cast<uint32_t>(v[i]));
                }
            }
            __stcs(reinterpret_cast<int4*>(a.w_out) + q0 + j, make_int4(v[0], v[1], v[2], v[3]));
        }
        tot += static_cast<unsigned long long>(static_cast<long long>(tsum));
        __syncthreads();
    }
    unsigned long long vals[4] = {tot, act, dig, got};
    unsigned long long* const outs[4] = {&a.slot->total, &a.slot->active, DIGEST ? &a.slot->digest : nullptr,
                                         &a.slot->got};
    block_sum_atomic<4>(vals, outs);
}

}  // namespace

bool bins_plan(Runtime& rt, int64_t n, int64_t lo, int64_t n_pad, BinPlan& plan)
{
    const int64_t K = ceil_div(n, kBinRange);
    if (K > kMaxBins || lo % kBinRange != 0 || n_pad % kBinRange != 0) return false;
    int smem_max = 0;
    AMBER_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, rt.device));
    plan.K = static_cast<int>(K);
    plan.k0 = static_cast<int>(lo / kBinRange);
    plan.k_loc = static_cast<int>(n_pad / kBinRange);
    // per-bin capacity: expected <= 2^16 entries (f <= 1), + 16 sigma + slack
    plan.cap = static_cast<uint32_t>(((kBinRange + 16 * 256 + 1024) + 7) & ~7ll);
    const size_t fixed = static_cast<size_t>(4) * 4 * K + 2048 + 64;  // bin arrays + static (scan temp, scalars)
    int64_t tile = 32768;
    while (tile > 4096 && static_cast<size_t>(tile) * 6 + fixed > static_cast<size_t>(smem_max)) tile /= 2;
    if (static_cast<size_t>(tile) * 6 + fixed > static_cast<size_t>(smem_max)) return false;
    plan.tile = static_cast<int>(tile);
    plan.prod_smem = static_cast<size_t>(tile) * 6 + static_cast<size_t>(4) * 4 * K;
    plan.apply_smem = static_cast<size_t>(kBinRange);  // 2^16 one-byte counters
    AMBER_CUDA(cudaFuncSetAttribute(wealth_bin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(plan.prod_smem)));
    AMBER_CUDA(cudaFuncSetAttribute(wealth_binapply_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(plan.apply_smem)));
    AMBER_CUDA(cudaFuncSetAttribute(wealth_binapply_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(plan.apply_smem)));
    int per_sm = 0;
    AMBER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wealth_bin_kernel, kProdThreads, plan.prod_smem));
    plan.prod_grid = std::max(per_sm, 1) * rt.num_sms;
    AMBER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wealth_binapply_kernel<false>, plan.apply_threads,
                                                             plan.apply_smem));
    plan.apply_grid = std::max(per_sm, 1) * rt.num_sms;
    return true;
}

void bins_allocate(Runtime& rt, const BinPlan& plan, BinBuffers& b)
{
    for (int par = 0; par < 2; ++par) {
        b.data[par].allocate(&rt, static_cast<size_t>(plan.K) * plan.cap);
        b.cnt[par].allocate(&rt, plan.K);
        b.cnt[par].zero_async(rt.stream);
    }
    b.queue.allocate(&rt, 2);
    b.queue.zero_async(rt.stream);
}

void bins_step(Runtime& rt, Profiler& prof, const BinPlan& plan, BinBuffers& b, const WealthStepCfg& c, uint32_t t,
               const int32_t* w, int32_t* w_out, WealthSlot* slot_t, WealthSlot* slot_next)
{
    const int par = t & 1;
    ProdArgs pa{};
    pa.key = c.key;
    pa.w = w;
    pa.n_loc = c.n_loc;
    pa.lo = c.lo;
    pa.m = c.n_glob - (c.exclude_self ? 1 : 0);
    pa.amount = c.amount;
    pa.exclude_self = c.exclude_self;
    pa.t = t;
    pa.data = b.data[par].p;
    pa.cnt = b.cnt[par].p;
    pa.cap = plan.cap;
    pa.K = plan.K;
    pa.tile = plan.tile;
    pa.n_tiles = c.n_pad / plan.tile;
    pa.queue = b.queue.p;
    pa.slot = slot_t;
    prof.launch(rt.stream, "wealth_bin_produce", [&] {
        wealth_bin_kernel<<<plan.prod_grid, kProdThreads, plan.prod_smem, rt.stream>>>(pa);
    });
    check_launch("wealth_bin_kernel");
    ApplyArgs aa{};
    aa.w_in = w;
    aa.w_out = w_out;
    aa.data = b.data[par].p;
    aa.cnt = b.cnt[par].p;
    aa.cap = plan.cap;
    aa.k0 = plan.k0;
    aa.k_loc = plan.k_loc;
    aa.n_loc = c.n_loc;
    aa.lo = c.lo;
    aa.amount = c.amount;
    aa.digest = c.digest;
    aa.queue = b.queue.p;
    aa.slot = slot_t;
    aa.slot_next = slot_next;
    prof.launch(rt.stream, "wealth_bin_apply", [&] {
        if (c.digest)
            wealth_binapply_kernel<true><<<plan.apply_grid, plan.apply_threads, plan.apply_smem, rt.stream>>>(aa);
        else
            wealth_binapply_kernel<false><<<plan.apply_grid, plan.apply_threads, plan.apply_smem, rt.stream>>>(aa);
    });
    check_launch("wealth_binapply_kernel");
}

}  // namespace amber
