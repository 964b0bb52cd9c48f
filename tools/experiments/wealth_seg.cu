// wealth_seg.cu -- segmented-bin wealth step ("seg").
//
// The transfer scatter w_i' = w_i - a*s_i + a*#{j : s_j, r_j = i} (contract W1)
// without one global atomic per transfer.  Evidence for the design
// (tools/scatter_probe.cu, profiles/r01_scatter_probe.txt): on this B200 a
// random 32-bit RED into L2 costs ~7x a random shared-memory atomic, and a
// random scatter store into shared memory is as cheap as a coalesced global
// store.  So every transfer is routed through shared memory twice and through
// HBM once, coalesced:
//
//   agents are split into K ranges of R agents (R = 42 x 8192 at N = 1e8,
//   K = 291, about two ranges per SM); one persistent CTA (1024 threads) per
//   SM takes ranges k = blockIdx.x, blockIdx.x + grid, ...  For range k:
//   1. (apply launches) consume: the entries of bin k written by the previous
//      launch -- K segments, one per producer range, plus an overflow tail --
//      go into a 4-bit shared-memory histogram (R/2 bytes, atomicAdd);
//   2. stream the range in chunks of 8192 agents (8 per thread, two 128-bit
//      loads, next chunk prefetched): w' = w - a*s + a*count;
//   3. produce: every sender of step t+1 (w' >= a, in registers) draws its
//      receiver r (Philox lane, R6), d = r / R, and takes a slot of the
//      chunk's per-destination staging row (S slots, shared-memory atomic);
//      after one barrier each warp copies whole rows out to the
//      (destination d, producer k) segment at the segment's cursor -- one
//      coalesced store of up to S*4 bytes per destination per chunk.  A row
//      that overflows within a chunk sends the excess to d's tail region
//      (global atomic cursor; rare: S is ~2x the mean row fill).
//   After the range, the K segment cursors are published as the next
//   launch's counts.  Every (destination, producer) count is rewritten by
//   every production, so nothing but the tails needs clearing.
//
// HBM traffic per agent-update: 8 B (column read + write) + 8 B per transfer
// (entry written + read back) = 8 + 8f B; no L2 atomics except tail overflow.
//
// Exactness (same contract as the packed counters): every produced entry is
// counted in `sent`, every decoded count in `got`.  A dropped entry (segment
// or tail full) lowers got by 1; a 4-bit carry lowers it by 15 or 16.  So any
// loss makes got < sent, and the model replays the window with exact 32-bit
// counters (wealth.cu).
#include <algorithm>
#include <cmath>

#include "wealth_experiments.cuh"

namespace amber {

namespace {

constexpr int kSegApt = 8;                              // agents per thread per chunk
constexpr int kOffBits = 19;                            // offsets within a range < 2^19

struct SegArgs {
    PhiloxKey key;
    const int32_t* w_in;
    int32_t* w_out;
    const uint32_t* in_data;   // bins consumed (step t_apply)
    const uint32_t* in_cnt;
    const uint32_t* in_tail;
    uint32_t* in_tcnt;         // zeroed after consumption
    uint32_t* out_data;        // bins produced (step t_prod)
    uint32_t* out_cnt;
    uint32_t* out_tail;
    uint32_t* out_tcnt;
    int64_t n_loc;
    uint32_t R;
    int K;
    uint32_t cap, tcap, kcap;  // kcap = K * cap (segment row stride of one destination)
    uint32_t magic, msh;       // d = umulhi(r, magic) >> msh == r / R  (r < 2^31)
    unsigned long long lo;     // global id of agent 0
    uint32_t m;                // receiver modulus (N or N-1)
    int32_t amount, exclude_self;
    uint32_t t_apply, t_prod;
    WealthSlot* slot_apply;
    WealthSlot* slot_prod;
    WealthSlot* slot_zero;
    int digest;
};

__device__ __forceinline__ void count_off(uint32_t* cnt4, uint32_t off)
{
    atomicAdd(cnt4 + (off >> 3), 1u << ((off & 7u) << 2));
}

template <bool APPLY, int NT, int S>
__global__ void __launch_bounds__(NT, 1024 / NT) wealth_seg_kernel(const SegArgs a)
{
    constexpr int kChunk = NT * kSegApt;
    constexpr int kWarps = NT / 32;
    extern __shared__ __align__(16) uint32_t sm[];
    const int R8 = static_cast<int>(a.R >> 3);
    uint32_t* cnt4 = sm;                       // R/8 words (4-bit counters, apply only)
    uint32_t* stage = sm + R8;                 // K rows of S offsets
    uint32_t* hist = stage + a.K * S;          // K: row fill of the current chunk
    uint32_t* cur = hist + a.K;                // K: segment cursors of the current range
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    if (blockIdx.x == 0 && tid == 0 && a.slot_zero) *a.slot_zero = WealthSlot{0, 0, 0, 0, 0};
    for (int d = tid; d < a.K; d += NT) {
        hist[d] = 0u;
        cur[d] = 0u;
    }
    unsigned long long tot = 0, act = 0, got = 0, sent = 0, dig = 0;
    const int nchunks = static_cast<int>(a.R / kChunk);

    for (int k = blockIdx.x; k < a.K; k += gridDim.x) {
        const int64_t base = static_cast<int64_t>(k) * a.R;
        if constexpr (APPLY) {
            // 1) consume bin k: K producer segments + the tail
            uint4* c4 = reinterpret_cast<uint4*>(cnt4);
            for (int j = tid; j < R8 / 4; j += NT) c4[j] = make_uint4(0u, 0u, 0u, 0u);
            __syncthreads();
            const uint32_t nt = min(a.in_tcnt[k], a.tcap);
            const uint32_t* segs = a.in_data + static_cast<size_t>(k) * a.kcap;
            for (int p = warp; p < a.K; p += kWarps) {
                const uint32_t n = min(a.in_cnt[static_cast<size_t>(k) * a.K + p], a.cap);
                const uint4* src = reinterpret_cast<const uint4*>(segs + static_cast<size_t>(p) * a.cap);
                for (uint32_t q0 = 0; q0 < n; q0 += 256) {  // two 128-bit loads in flight per lane
                    const uint32_t qa = q0 + lane * 4, qb = qa + 128;
                    uint4 ea = make_uint4(0u, 0u, 0u, 0u), eb = ea;
                    if (qa < n) ea = __ldcs(src + (qa >> 2));
                    if (qb < n) eb = __ldcs(src + (qb >> 2));
                    if (qa < n) count_off(cnt4, ea.x);
                    if (qa + 1 < n) count_off(cnt4, ea.y);
                    if (qa + 2 < n) count_off(cnt4, ea.z);
                    if (qa + 3 < n) count_off(cnt4, ea.w);
                    if (qb < n) count_off(cnt4, eb.x);
                    if (qb + 1 < n) count_off(cnt4, eb.y);
                    if (qb + 2 < n) count_off(cnt4, eb.z);
                    if (qb + 3 < n) count_off(cnt4, eb.w);
                }
            }
            const uint32_t* tsrc = a.in_tail + static_cast<size_t>(k) * a.tcap;
            for (uint32_t e = tid; e < nt; e += NT) count_off(cnt4, __ldcs(tsrc + e));
            __syncthreads();
            if (tid == 0) a.in_tcnt[k] = 0u;  // every thread read nt before the barrier
        }

        // 2)+3) stream the range
        int32_t nx[kSegApt];
        {
            const int4* p4 = reinterpret_cast<const int4*>(a.w_in + base + tid * kSegApt);
            const int4 x0 = __ldcs(p4), x1 = __ldcs(p4 + 1);
            nx[0] = x0.x; nx[1] = x0.y; nx[2] = x0.z; nx[3] = x0.w;
            nx[4] = x1.x; nx[5] = x1.y; nx[6] = x1.z; nx[7] = x1.w;
        }
        uint32_t* const dst_k = a.out_data + static_cast<size_t>(k) * a.cap;  // + d * kcap
        for (int c = 0; c < nchunks; ++c) {
            int32_t v[kSegApt];
#pragma unroll
            for (int i = 0; i < kSegApt; ++i) v[i] = nx[i];
            const int64_t a0 = base + static_cast<int64_t>(c) * kChunk + tid * kSegApt;  // local index
            if (c + 1 < nchunks) {
                const int4* p4 = reinterpret_cast<const int4*>(a.w_in + a0 + kChunk);
                const int4 x0 = __ldcs(p4), x1 = __ldcs(p4 + 1);
                nx[0] = x0.x; nx[1] = x0.y; nx[2] = x0.z; nx[3] = x0.w;
                nx[4] = x1.x; nx[5] = x1.y; nx[6] = x1.z; nx[7] = x1.w;
            }
            if constexpr (APPLY) {
                const uint32_t word = cnt4[c * NT + tid];
                int32_t tsum = 0;
                uint32_t gsum = 0, asum = 0;
#pragma unroll
                for (int i = 0; i < kSegApt; ++i) {
                    const int32_t ci = static_cast<int32_t>((word >> (4 * i)) & 15u);
                    v[i] = v[i] - (v[i] >= a.amount ? a.amount : 0) + a.amount * ci;
                    tsum += v[i];
                    asum += v[i] > 0;
                    if (a.digest) {
                        const int64_t loc = a0 + i;
                        if (loc < a.n_loc)
                            dig += digest_term(a.lo + static_cast<unsigned long long>(loc), static_cast<uint32_t>(v[i]));
                    }
                }
                gsum = __popc(word & 0x11111111u) + 2u * __popc(word & 0x22222222u) + 4u * __popc(word & 0x44444444u) +
                       8u * __popc(word & 0x88888888u);
                got += gsum;
                act += asum;
                tot += static_cast<unsigned long long>(static_cast<long long>(tsum));
                int4* o4 = reinterpret_cast<int4*>(a.w_out + a0);
                __stcs(o4, make_int4(v[0], v[1], v[2], v[3]));
                __stcs(o4 + 1, make_int4(v[4], v[5], v[6], v[7]));
            }
            // receivers of step t_prod's senders -> staging rows
            const unsigned long long i0 = a.lo + static_cast<unsigned long long>(a0);  // even
            uint32_t nsent = 0;
#pragma unroll
            for (int p = 0; p < kSegApt / 2; ++p) {
                const bool s0 = v[2 * p] >= a.amount, s1 = v[2 * p + 1] >= a.amount;
                if (!(s0 | s1)) continue;
                const uint4 x = stream_block(a.key, TAG_WEALTH_RECV, (i0 >> 1) + p, a.t_prod);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!(h ? s1 : s0)) continue;
                    uint32_t r = mulhi64_n32(lane64_of(x, h), a.m);
                    if (a.exclude_self) r += (r >= static_cast<uint32_t>(i0 + 2 * p + h));
                    const uint32_t d = __umulhi(r, a.magic) >> a.msh;
                    const uint32_t off = r - d * a.R;
                    const uint32_t slot = atomicAdd(&hist[d], 1u);
                    if (slot < static_cast<uint32_t>(S)) {
                        stage[d * S + slot] = off;
                    } else {  // row full within this chunk: overflow tail of d
                        const uint32_t pos = atomicAdd(a.out_tcnt + d, 1u);
                        if (pos < a.tcap) a.out_tail[static_cast<size_t>(d) * a.tcap + pos] = off;
                    }
                    ++nsent;
                }
            }
            sent += nsent;
            __syncthreads();
            // copy-out: lane -> (row d, slot j); 32/S rows per warp pass (S >= 32: S/32 passes per row)
            if constexpr (S <= 32) {
                constexpr int kRows = 32 / S;
                const int jr = lane % S;
                for (int d0 = warp * kRows; d0 < a.K; d0 += kWarps * kRows) {
                    const int d = d0 + lane / S;
                    uint32_t h = 0, c0 = 0;
                    if (d < a.K) {
                        h = min(hist[d], static_cast<uint32_t>(S));
                        c0 = cur[d];
                        if (jr < static_cast<int>(h) && c0 + jr < a.cap)
                            dst_k[static_cast<size_t>(d) * a.kcap + c0 + jr] = stage[d * S + jr];
                    }
                    __syncwarp();
                    if (d < a.K && jr == 0) {
                        cur[d] = c0 + h;
                        hist[d] = 0u;
                    }
                }
            } else {
                for (int d = warp; d < a.K; d += kWarps) {
                    const uint32_t h = min(hist[d], static_cast<uint32_t>(S)), c0 = cur[d];
#pragma unroll
                    for (int j0 = 0; j0 < S; j0 += 32) {
                        const uint32_t j = j0 + lane;
                        if (j < h && c0 + j < a.cap) dst_k[static_cast<size_t>(d) * a.kcap + c0 + j] = stage[d * S + j];
                    }
                    __syncwarp();
                    if (lane == 0) {
                        cur[d] = c0 + h;
                        hist[d] = 0u;
                    }
                }
            }
            __syncthreads();
        }
        // publish this range's segment sizes, reset the cursors
        for (int d = tid; d < a.K; d += NT) {
            a.out_cnt[static_cast<size_t>(d) * a.K + k] = cur[d];
            cur[d] = 0u;
        }
        __syncthreads();
    }
    unsigned long long vals[5] = {tot, act, dig, sent, got};
    unsigned long long* const outs[5] = {APPLY ? &a.slot_apply->total : nullptr, APPLY ? &a.slot_apply->active : nullptr,
                                         (APPLY && a.digest) ? &a.slot_apply->digest : nullptr, &a.slot_prod->sent,
                                         APPLY ? &a.slot_apply->got : nullptr};
    block_sum_atomic<5>(vals, outs);
}

using SegKernel = void (*)(SegArgs);

template <bool APPLY>
SegKernel seg_kernel_for(int nt, int s)
{
    if (nt == 1024) {
        switch (s) {
            case 16: return wealth_seg_kernel<APPLY, 1024, 16>;
            case 32: return wealth_seg_kernel<APPLY, 1024, 32>;
            case 64: return wealth_seg_kernel<APPLY, 1024, 64>;
        }
    } else if (nt == 512) {
        switch (s) {
            case 8: return wealth_seg_kernel<APPLY, 512, 8>;
            case 16: return wealth_seg_kernel<APPLY, 512, 16>;
            case 32: return wealth_seg_kernel<APPLY, 512, 32>;
        }
    }
    return nullptr;
}

}  // namespace

bool seg_plan(Runtime& rt, int64_t n, int64_t n_loc, SegPlan& plan)
{
    if (rt.world != 1 || n != n_loc || n < 32768 || n >= (1ll << 31)) return false;
    int smem_max = 0;
    AMBER_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, rt.device));
    const int sms = rt.num_sms;
    // ctas per SM: 1 (1024 threads, ranges of <= 344064 agents) or 2 (512 threads, half the
    // shared memory each); AMBER_SEG_CTAS overrides (measurement hook)
    const char* env = getenv("AMBER_SEG_CTAS");
    const int per_sm = (env && env[0] == '2') ? 2 : 1;
    const int NT = per_sm == 2 ? 512 : 1024;
    const int64_t chunk = static_cast<int64_t>(NT) * kSegApt;
    const int64_t smem_cta = per_sm == 2 ? std::min<int64_t>(smem_max, 113 * 1024) : smem_max;
    // about two ranges per CTA slot, R a multiple of the chunk, counters <= ~75% of the budget
    int64_t R = ceil_div(ceil_div(n, 2ll * sms * per_sm), chunk) * chunk;
    while (R > chunk && R / 2 > smem_cta * 3 / 4) R -= chunk;
    const int64_t K = ceil_div(n, R);
    if (R > (1ll << kOffBits) || K > 8192) return false;
    // staging rows: ~2x the mean fill of a chunk row at f = 0.6 (f = 1 only in the first step);
    // rows that overflow within a chunk spill to the destination's tail
    const double mean = static_cast<double>(chunk) * 0.6 / static_cast<double>(K);
    const int smin = NT == 1024 ? 16 : 8, smax = NT == 1024 ? 64 : 32;
    int S = smin;
    while (S < 2.0 * mean && S < smax) S *= 2;
    auto need = [&](int s) { return static_cast<size_t>(R / 8) * 4 + static_cast<size_t>(K) * s * 4 + static_cast<size_t>(K) * 8; };
    while (need(S) > static_cast<size_t>(smem_cta) && S > smin) S /= 2;
    if (need(S) > static_cast<size_t>(smem_cta)) return false;
    // segment capacity: f = 1 mean R*R/N plus 16 sigma, multiple of 4 (16-byte aligned rows)
    const double mu = static_cast<double>(R) * static_cast<double>(R) / static_cast<double>(n);
    const int64_t cap = (static_cast<int64_t>(mu + 16.0 * std::sqrt(mu) + 64.0) + 3) & ~3ll;
    if (K * K * cap >= (1ll << 32)) return false;
    // d = umulhi(r, magic) >> msh: with 2^msh < R <= 2^(msh+1), magic = ceil(2^(32+msh) / R) < 2^32
    // and the error r*(magic*R - 2^(32+msh)) < r*R < 2^(32+msh) for r < 2^31 (exact)
    int msh = 0;
    while ((2ll << msh) < R) ++msh;
    const unsigned long long magic = ((1ull << (32 + msh)) + static_cast<unsigned long long>(R) - 1) /
                                     static_cast<unsigned long long>(R);
    if (magic >= (1ull << 32)) return false;
    for (int64_t j = 1; j <= K; ++j)  // boundary check of the division on the host
        for (int64_t r : {j * R - 1, j * R})
            if (r < (1ll << 31) &&
                ((static_cast<unsigned long long>(r) * magic) >> (32 + msh)) != static_cast<unsigned long long>(r / R))
                return false;
    plan.R = R;
    plan.K = static_cast<int>(K);
    plan.S = S;
    plan.NT = NT;
    plan.grid = static_cast<int>(std::min<int64_t>(K, static_cast<int64_t>(sms) * per_sm));
    plan.cap = static_cast<uint32_t>(cap);
    plan.tcap = static_cast<uint32_t>(std::max<int64_t>(4096, K < 64 ? R : R / 4));
    plan.magic = magic;
    plan.msh = msh;
    plan.smem = need(S);
    auto ka = seg_kernel_for<true>(NT, S);
    auto kp = seg_kernel_for<false>(NT, S);
    if (!ka || !kp) return false;
    AMBER_CUDA(cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(plan.smem)));
    AMBER_CUDA(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(plan.smem)));
    return true;
}

void seg_allocate(Runtime& rt, const SegPlan& plan, SegBuffers& b)
{
    const size_t K = static_cast<size_t>(plan.K);
    for (int par = 0; par < 2; ++par) {
        b.data[par].allocate(&rt, K * K * plan.cap);
        b.cnt[par].allocate(&rt, K * K);
        b.cnt[par].zero_async(rt.stream);
        b.tail[par].allocate(&rt, K * plan.tcap);
        b.tcnt[par].allocate(&rt, K);
        b.tcnt[par].zero_async(rt.stream);
    }
}

void seg_reset(Runtime& rt, SegBuffers& b)
{
    for (auto& x : b.cnt) x.zero_async(rt.stream);
    for (auto& x : b.tcnt) x.zero_async(rt.stream);
}

void seg_launch(Runtime& rt, Profiler& prof, const SegPlan& plan, SegBuffers& b, const WealthStepCfg& c, bool apply,
                uint32_t t_apply, uint32_t t_prod, const int32_t* w_in, int32_t* w_out, WealthSlot* slot_apply,
                WealthSlot* slot_prod, WealthSlot* slot_zero)
{
    SegArgs a{};
    a.key = c.key;
    a.w_in = w_in;
    a.w_out = w_out;
    const int pin = t_apply & 1, pout = t_prod & 1;
    a.in_data = b.data[pin].p;
    a.in_cnt = b.cnt[pin].p;
    a.in_tail = b.tail[pin].p;
    a.in_tcnt = b.tcnt[pin].p;
    a.out_data = b.data[pout].p;
    a.out_cnt = b.cnt[pout].p;
    a.out_tail = b.tail[pout].p;
    a.out_tcnt = b.tcnt[pout].p;
    a.n_loc = c.n_loc;
    a.R = static_cast<uint32_t>(plan.R);
    a.K = plan.K;
    a.cap = plan.cap;
    a.tcap = plan.tcap;
    a.kcap = static_cast<uint32_t>(plan.K) * plan.cap;
    a.magic = static_cast<uint32_t>(plan.magic);
    a.msh = static_cast<uint32_t>(plan.msh);
    a.lo = c.lo;
    a.m = static_cast<uint32_t>(c.n_glob - (c.exclude_self ? 1 : 0));
    a.amount = c.amount;
    a.exclude_self = c.exclude_self;
    a.t_apply = t_apply;
    a.t_prod = t_prod;
    a.slot_apply = slot_apply;
    a.slot_prod = slot_prod;
    a.slot_zero = slot_zero;
    a.digest = c.digest;
    SegKernel kern = apply ? seg_kernel_for<true>(plan.NT, plan.S) : seg_kernel_for<false>(plan.NT, plan.S);
    prof.launch(rt.stream, apply ? "wealth_seg_step" : "wealth_seg_prime", [&] {
        kern<<<plan.grid, plan.NT, plan.smem, rt.stream>>>(a);
    });
    check_launch("wealth_seg_kernel");
}

}  // namespace amber
