// wealth_fb.cu -- fused, range-binned wealth step ("fb").
//
// One launch per step, like the packed-counter kernel, but with no global
// atomic per transfer.  Agents are grouped in ranges of 2^16; a CTA takes a
// range from a work queue and
//   1. builds the step-t transfer counts of the range in a shared-memory
//      histogram (8-bit counters, 4 per word) from the range's bin, written by
//      the previous launch;
//   2. streams the range's wealth (8 agents per thread per phase, 128-bit
//      loads/stores): w' = w - a*s + a*c;
//   3. for every sender of step t+1 (w' >= a, still in registers) draws the
//      receiver r and appends its 16-bit offset to a shared-memory
//      write-combining buffer of r's range (S slots per range, per CTA);
//      after each phase, full 8-entry chunks are flushed with ONE 16-byte store
//      at a chunk slot reserved by one global atomic (1 atomic per 8 transfers
//      instead of 1 RED per transfer).  Partial buffers are flushed at the end
//      of the launch into a separate per-range "tail" region.
// Status (r01): exact (tests/test_gpu_wealth.py), but 0.57 ms/step at N=1e8 vs
// 0.40 ms for the packed-counter kernel -- the per-phase buffer flushes (two
// barriers, ~300 chunk reservations per CTA per phase) cost more than the L2
// atomics they remove.  Opt-in via counter_bits = -2.
// Exactness: bin overflow (dropped entries) and 8-bit counter carries both
// make the decoded total (`got`) smaller than the entries produced (`sent`);
// the model then replays the window with exact 32-bit counters (wealth.cu).
#include <algorithm>

#include "wealth_experiments.cuh"

namespace amber {

namespace {

constexpr int kFbThreads = 512;
constexpr int kFbApt = 8;                          // agents per thread per phase
constexpr int kFbPhase = kFbThreads * kFbApt;      // 4096
constexpr int kFbPhases = static_cast<int>(kBinRange / kFbPhase);  // 16
constexpr int kHistWords = static_cast<int>(kBinRange / 4);        // 8-bit counters
constexpr int kChunk = 8;                          // entries per flushed chunk (16 B)

struct FbArgs {
    PhiloxKey key;
    const int32_t* w_in;
    int32_t* w_out;
    const uint16_t* in_data;   // bins of the applied step: [K][cap_lo + cap_hi]
    uint32_t* in_lo;           // full-chunk entries per range
    uint32_t* in_hi;           // tail entries per range
    uint16_t* out_data;        // bins of the produced step
    uint32_t* out_lo;
    uint32_t* out_hi;
    uint32_t cap_lo, cap_hi;
    int K, k0, k_loc, S;
    int64_t n_loc;
    unsigned long long lo, m;  // global id of local agent 0; receiver modulus (N or N-1)
    int32_t amount, exclude_self;
    uint32_t t_apply, t_prod;
    int* queue;                // [2]: work-queue counters, alternated by launch
    int q_use, q_reset;
    WealthSlot* slot_apply;
    WealthSlot* slot_prod;
    WealthSlot* slot_zero;
    int digest;
};

template <bool APPLY>
__global__ void __launch_bounds__(kFbThreads, 2) wealth_fb_kernel(const FbArgs a)
{
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* hist = sm;                                              // kHistWords (APPLY)
    uint32_t* wcn = sm + (APPLY ? kHistWords : 0);                    // K counters
    uint16_t* wc = reinterpret_cast<uint16_t*>(wcn + a.K);            // K * S entries
    __shared__ int range_s;
    const int tid = threadIdx.x;
    const size_t stride = static_cast<size_t>(a.cap_lo) + a.cap_hi;
    if (blockIdx.x == 0 && tid == 0) {
        a.queue[a.q_reset] = 0;
        if (a.slot_zero) *a.slot_zero = WealthSlot{0, 0, 0, 0, 0};
    }
    for (int d = tid; d < a.K; d += kFbThreads) wcn[d] = 0u;
    unsigned long long tot = 0, act = 0, got = 0, sent = 0, dig = 0;

    for (;;) {
        if (tid == 0) range_s = atomicAdd(a.queue + a.q_use, 1);
        if constexpr (APPLY)
            for (int j = tid; j < kHistWords; j += kFbThreads) hist[j] = 0u;
        __syncthreads();
        const int k = range_s;
        if (k >= a.k_loc) break;
        const int kg = a.k0 + k;
        if constexpr (APPLY) {
            // 1) step-t counts of this range
            const uint16_t* src = a.in_data + static_cast<size_t>(kg) * stride;
            const uint32_t nlo = min(a.in_lo[kg], a.cap_lo) & ~7u;
            const uint32_t nhi = min(a.in_hi[kg], a.cap_hi);
            for (uint32_t c = tid; c < nlo / kChunk; c += kFbThreads) {
                const uint4 v = __ldcs(reinterpret_cast<const uint4*>(src) + c);
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const uint32_t o0 = w4[h] & 0xFFFFu, o1 = w4[h] >> 16;
                    atomicAdd(&hist[o0 >> 2], 1u << ((o0 & 3u) * 8u));
                    atomicAdd(&hist[o1 >> 2], 1u << ((o1 & 3u) * 8u));
                }
            }
            for (uint32_t e = tid; e < nhi; e += kFbThreads) {
                const uint32_t o = src[a.cap_lo + e];
                atomicAdd(&hist[o >> 2], 1u << ((o & 3u) * 8u));
            }
            __syncthreads();
            if (tid == 0) {
                a.in_lo[kg] = 0u;  // consumed: this parity's bin is empty again
                a.in_hi[kg] = 0u;
            }
        }
        // 2)+3) stream the range in phases of 4096 agents
        const int64_t base = static_cast<int64_t>(k) * kBinRange;
        for (int ph = 0; ph < kFbPhases; ++ph) {
            const int64_t a0 = base + static_cast<int64_t>(ph) * kFbPhase + static_cast<int64_t>(tid) * kFbApt;
            int32_t v[kFbApt];
#pragma unroll
            for (int q = 0; q < kFbApt / 4; ++q) {
                const int4 x = __ldcs(reinterpret_cast<const int4*>(a.w_in + a0) + q);
                v[4 * q] = x.x;
                v[4 * q + 1] = x.y;
                v[4 * q + 2] = x.z;
                v[4 * q + 3] = x.w;
            }
            if constexpr (APPLY) {
                const int hw = static_cast<int>((a0 - base) >> 2);
                int32_t tsum = 0;
#pragma unroll
                for (int i = 0; i < kFbApt; ++i) {
                    const uint32_t hword = hist[hw + (i >> 2)];
                    const int32_t ci = static_cast<int32_t>((hword >> (8 * (i & 3))) & 255u);
                    v[i] = v[i] - (v[i] >= a.amount ? a.amount : 0) + a.amount * ci;
                    got += static_cast<unsigned>(ci);
                    tsum += v[i];
                    act += v[i] > 0;
                    if (a.digest) {
                        const int64_t loc = a0 + i;
                        if (loc < a.n_loc)
                            dig += digest_term(a.lo + static_cast<unsigned long long>(loc), static_cast<uint32_t>(v[i]));
                    }
                }
                tot += static_cast<unsigned long long>(static_cast<long long>(tsum));
#pragma unroll
                for (int q = 0; q < kFbApt / 4; ++q)
                    __stcs(reinterpret_cast<int4*>(a.w_out + a0) + q, make_int4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
            }
            // receivers of step t_prod's senders -> write-combining buffers
            const unsigned long long i0 = a.lo + static_cast<unsigned long long>(a0);  // even
#pragma unroll
            for (int p = 0; p < kFbApt / 2; ++p) {
                const uint4 x = stream_block(a.key, TAG_WEALTH_RECV, (i0 >> 1) + p, a.t_prod);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (v[2 * p + h] < a.amount) continue;
                    const unsigned long long xx = lane64_of(x, h);
                    unsigned long long r = (a.m >> 32) ? mulhi64(xx, a.m) : mulhi64_n32(xx, static_cast<uint32_t>(a.m));
                    if (a.exclude_self) r += (r >= i0 + 2 * p + h);
                    const int d = static_cast<int>(r >> kBinShift);
                    const uint16_t off = static_cast<uint16_t>(r & (kBinRange - 1));
                    const uint32_t slot = atomicAdd(&wcn[d], 1u);
                    if (slot < static_cast<uint32_t>(a.S)) {
                        wc[d * a.S + slot] = off;
                    } else {  // buffer full within this phase (rare): straight to the tail region
                        const uint32_t pos = atomicAdd(a.out_hi + d, 1u);
                        if (pos < a.cap_hi) a.out_data[static_cast<size_t>(d) * stride + a.cap_lo + pos] = off;
                    }
                    ++sent;
                }
            }
            __syncthreads();
            // flush full chunks, keep the remainder at the front of each buffer.
            // All reservation atomics of a thread are issued before any result is
            // used, so their round trips overlap.
            constexpr int kMaxOwned = 8;  // ranges per thread: ceil(K / 512) <= 8 (K <= 4096)
            uint32_t cnt_d[kMaxOwned], pos_d[kMaxOwned];
#pragma unroll
            for (int j = 0; j < kMaxOwned; ++j) {
                const int d = tid + j * kFbThreads;
                cnt_d[j] = d < a.K ? min(wcn[d], static_cast<uint32_t>(a.S)) : 0u;
                const uint32_t nfull = cnt_d[j] / kChunk;
                pos_d[j] = nfull ? atomicAdd(a.out_lo + d, nfull * kChunk) : 0u;
            }
#pragma unroll
            for (int j = 0; j < kMaxOwned; ++j) {
                const int d = tid + j * kFbThreads;
                if (d >= a.K) continue;
                const uint32_t c = cnt_d[j], nfull = c / kChunk, pos = pos_d[j];
                const uint16_t* b = wc + d * a.S;
                uint16_t* dst = a.out_data + static_cast<size_t>(d) * stride;
                for (uint32_t q = 0; q < nfull; ++q) {
                    if (pos + (q + 1) * kChunk <= a.cap_lo) {
                        uint4 chunk;
                        uint32_t* cw = reinterpret_cast<uint32_t*>(&chunk);
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj)
                            cw[jj] = static_cast<uint32_t>(b[q * kChunk + 2 * jj]) |
                                     (static_cast<uint32_t>(b[q * kChunk + 2 * jj + 1]) << 16);
                        reinterpret_cast<uint4*>(dst)[(pos >> 3) + q] = chunk;
                    }
                }
                const uint32_t rem = c - nfull * kChunk;
                if (nfull)
                    for (uint32_t jj = 0; jj < rem; ++jj) wc[d * a.S + jj] = b[nfull * kChunk + jj];
                wcn[d] = rem;
            }
            __syncthreads();
        }
    }
    // partial buffers -> tail region
    for (int d = tid; d < a.K; d += kFbThreads) {
        const uint32_t c = min(wcn[d], static_cast<uint32_t>(a.S));
        if (!c) continue;
        const uint32_t pos = atomicAdd(a.out_hi + d, c);
        uint16_t* dst = a.out_data + static_cast<size_t>(d) * stride + a.cap_lo;
        for (uint32_t j = 0; j < c; ++j)
            if (pos + j < a.cap_hi) dst[pos + j] = wc[d * a.S + j];
    }
    unsigned long long vals[5] = {tot, act, dig, sent, got};
    unsigned long long* const outs[5] = {APPLY ? &a.slot_apply->total : nullptr, APPLY ? &a.slot_apply->active : nullptr,
                                         (APPLY && a.digest) ? &a.slot_apply->digest : nullptr, &a.slot_prod->sent,
                                         APPLY ? &a.slot_apply->got : nullptr};
    block_sum_atomic<5>(vals, outs);
}

}  // namespace

bool fb_plan(Runtime& rt, int64_t n, int64_t lo, int64_t n_pad, FbPlan& plan)
{
    const int64_t K = ceil_div(n, kBinRange);
    if (lo % kBinRange != 0 || n_pad % kBinRange != 0) return false;
    int smem_max = 0, smem_sm = 0;
    AMBER_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, rt.device));
    AMBER_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, rt.device));
    // two CTAs per SM: hist (64 KB) + K counters + K*S entries per CTA
    const int64_t budget = std::min<int64_t>(smem_max, smem_sm / 2 - 2048) - kHistWords * 4 - 4 * K - 1024;
    int64_t S = budget / (2 * K);
    S = std::min<int64_t>(S, 24);
    if (S < 12 || K < 1024 || K > 4096) return false;  // buffers sized for >= 1024 ranges (~8 entries/phase)
    plan.K = static_cast<int>(K);
    plan.k0 = static_cast<int>(lo / kBinRange);
    plan.k_loc = static_cast<int>(n_pad / kBinRange);
    plan.S = static_cast<int>(S);
    plan.cap_lo = static_cast<uint32_t>(kBinRange + 16 * 256 + 64) & ~7u;  // f <= 1 plus 16 sigma
    plan.cap_hi = 8192;
    plan.smem_apply = static_cast<size_t>(kHistWords) * 4 + 4 * K + 2 * K * S + 16;
    plan.smem_prod = 4 * K + 2 * K * S + 16;
    AMBER_CUDA(cudaFuncSetAttribute(wealth_fb_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(plan.smem_apply)));
    AMBER_CUDA(cudaFuncSetAttribute(wealth_fb_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(plan.smem_prod)));
    int per_sm = 0;
    AMBER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wealth_fb_kernel<true>, kFbThreads,
                                                             plan.smem_apply));
    plan.grid = std::max(per_sm, 1) * rt.num_sms;
    return true;
}

void fb_allocate(Runtime& rt, const FbPlan& plan, FbBuffers& b)
{
    const size_t stride = static_cast<size_t>(plan.cap_lo) + plan.cap_hi;
    for (int par = 0; par < 2; ++par) {
        b.data[par].allocate(&rt, static_cast<size_t>(plan.K) * stride);
        b.lo[par].allocate(&rt, plan.K);
        b.hi[par].allocate(&rt, plan.K);
        b.lo[par].zero_async(rt.stream);
        b.hi[par].zero_async(rt.stream);
    }
    b.queue.allocate(&rt, 2);
    b.queue.zero_async(rt.stream);
}

void fb_launch(Runtime& rt, Profiler& prof, const FbPlan& plan, FbBuffers& b, const WealthStepCfg& c, bool apply,
               uint32_t t_apply, uint32_t t_prod, const int32_t* w_in, int32_t* w_out, WealthSlot* slot_apply,
               WealthSlot* slot_prod, WealthSlot* slot_zero, int launch_parity)
{
    FbArgs a{};
    a.key = c.key;
    a.w_in = w_in;
    a.w_out = w_out;
    const int pin = t_apply & 1, pout = t_prod & 1;
    a.in_data = b.data[pin].p;
    a.in_lo = b.lo[pin].p;
    a.in_hi = b.hi[pin].p;
    a.out_data = b.data[pout].p;
    a.out_lo = b.lo[pout].p;
    a.out_hi = b.hi[pout].p;
    a.cap_lo = plan.cap_lo;
    a.cap_hi = plan.cap_hi;
    a.K = plan.K;
    a.k0 = plan.k0;
    a.k_loc = plan.k_loc;
    a.S = plan.S;
    a.n_loc = c.n_loc;
    a.lo = c.lo;
    a.m = c.n_glob - (c.exclude_self ? 1 : 0);
    a.amount = c.amount;
    a.exclude_self = c.exclude_self;
    a.t_apply = t_apply;
    a.t_prod = t_prod;
    a.queue = b.queue.p;
    a.q_use = launch_parity & 1;
    a.q_reset = (launch_parity + 1) & 1;
    a.slot_apply = slot_apply;
    a.slot_prod = slot_prod;
    a.slot_zero = slot_zero;
    a.digest = c.digest;
    if (apply) {
        prof.launch(rt.stream, "wealth_fb_step", [&] {
            wealth_fb_kernel<true><<<plan.grid, kFbThreads, plan.smem_apply, rt.stream>>>(a);
        });
    } else {
        prof.launch(rt.stream, "wealth_fb_prime", [&] {
            wealth_fb_kernel<false><<<plan.grid, kFbThreads, plan.smem_prod, rt.stream>>>(a);
        });
    }
    check_launch("wealth_fb_kernel");
}

}  // namespace amber
