// wealth_bulk_scatter.cu -- experiment (not built into libamber.so): the C4
// wealth scatter (Sec. 5.1.1 l.201; W1: each agent with
// w > 0 gives one unit to r = mulhi64(lane64(WEALTH_RECV, i, t), N)) WITHOUT a
// global atomic per transfer, using Blackwell bulk data movement, against the
// one-RED-per-transfer scatter the product ships.
//
//   red   : the product's scheme -- one red.add per transfer into packed
//           4-bit counters (N/2 bytes), L2 evict_last.
//   bulk  : pass 1 bins the receivers by 2^18-agent range in shared memory
//           (one shared atomic per transfer for the slot), flushing each full
//           32-entry run to the range's global segment with cp.async.bulk
//           (one global atomic per 32 transfers); pass 2 gives each range to
//           two CTAs, which build its 4-bit histogram (128 KB) with shared
//           atomics and add it into the packed counters with
//           cp.reduce.async.bulk .add.u32.
//
// Both are checked against exact 32-bit counters.  Timings by CUDA events;
// run under ncu for the instruction counts:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -I paper_2601_16292_b200/csrc -I include tools/experiments/wealth_bulk_scatter.cu \
//        -o tools/experiments/wealth_bulk_scatter
//   tools/experiments/wealth_bulk_scatter            (N = 1e8, t = 5)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "philox.cuh"

using namespace amber;

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) {                                                                 \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));     \
            exit(1);                                                                             \
        }                                                                                        \
    } while (0)

constexpr int kShift = 18;                 // receivers per range: 2^18
constexpr int kStage = 64;                 // staged entries per range (flush at 32)
constexpr int kHistWords = (1 << kShift) / 8;  // 4-bit counters, 8 per word: 128 KB

__device__ __forceinline__ uint32_t mix(uint32_t x)
{
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    return x ^ (x >> 16);
}

// synthetic column: ~59% of the agents hold wealth (the C4 equilibrium)
__global__ void fill_w(int32_t* w, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        w[i] = (mix(static_cast<uint32_t>(i) * 2654435761u + 17u) % 100u) < 59u ? 1 + static_cast<int32_t>(i % 3) : 0;
}

__device__ __forceinline__ uint32_t receiver(const PhiloxKey& K, uint64_t i, uint32_t t, uint64_t n, uint4& blk,
                                             bool fresh)
{
    if (fresh) blk = stream_block(K, TAG_WEALTH_RECV, i >> 1, t);
    return static_cast<uint32_t>(mulhi64(lane64_of(blk, static_cast<unsigned>(i & 1)), n));
}

// exact reference: 32-bit counters
__global__ void scatter_ref(const int32_t* __restrict__ w, int64_t n, PhiloxKey K, uint32_t t, uint32_t* cnt)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; 2 * p < n; p += (int64_t)gridDim.x * blockDim.x) {
        uint4 blk;
        bool fresh = true;
        for (int h = 0; h < 2; ++h) {
            const int64_t i = 2 * p + h;
            if (i >= n || w[i] <= 0) continue;
            atomicAdd(cnt + receiver(K, i, t, n, blk, fresh), 1u);
            fresh = false;
        }
    }
}

// the shipped scheme: one RED per transfer into packed 4-bit counters
__global__ void __launch_bounds__(256) scatter_red(const int32_t* __restrict__ w, int64_t n, PhiloxKey K, uint32_t t,
                                                   uint32_t* packed)
{
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; 2 * p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int2 v = 2 * p + 1 < n ? reinterpret_cast<const int2*>(w)[p] : make_int2(w[2 * p], 0);
        if (v.x <= 0 && v.y <= 0) continue;
        const uint4 blk = stream_block(K, TAG_WEALTH_RECV, static_cast<unsigned long long>(p), t);
        for (int h = 0; h < 2; ++h) {
            if ((h ? v.y : v.x) <= 0) continue;
            const uint32_t r = static_cast<uint32_t>(mulhi64(lane64_of(blk, h), n));
            asm volatile("red.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(packed + (r >> 3)),
                         "r"(1u << ((r & 7u) * 4u)), "l"(pol)
                         : "memory");
        }
    }
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ssrc))), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_reduce_add_u32(void* gdst, const void* ssrc, uint32_t bytes)
{
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u32 [%0], [%1], %2;" ::"l"(gdst),
                 "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ssrc))), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read()
{
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_commit_wait_all()
{
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Pass 1: bin the transfers by receiver range (dynamic smem: stage[nr][kStage] + scnt[nr]).
// Rounds of 2 agents per thread; after each round the ranges holding >= 32
// entries flush 32 of them (128 B) with one bulk copy.
__global__ void __launch_bounds__(512) bin_pass(const int32_t* __restrict__ w, int64_t n, PhiloxKey K, uint32_t t,
                                                int nr, uint32_t* __restrict__ seg, int64_t seg_cap,
                                                uint32_t* __restrict__ gcur)
{
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* stage = sm;                                  // nr * kStage
    uint32_t* scnt = sm + static_cast<int64_t>(nr) * kStage;  // nr
    for (int b = threadIdx.x; b < nr; b += blockDim.x) scnt[b] = 0;
    __syncthreads();
    const int64_t npairs = (n + 1) / 2;
    const int64_t per = (npairs + gridDim.x - 1) / gridDim.x;
    const int64_t p0 = blockIdx.x * per, p1 = min(npairs, p0 + per);
    for (int64_t base = p0; base < p1; base += blockDim.x) {
        const int64_t p = base + threadIdx.x;
        if (p < p1) {
            const int2 v = 2 * p + 1 < n ? reinterpret_cast<const int2*>(w)[p] : make_int2(w[2 * p], 0);
            if (v.x > 0 || v.y > 0) {
                const uint4 blk = stream_block(K, TAG_WEALTH_RECV, static_cast<unsigned long long>(p), t);
                for (int h = 0; h < 2; ++h) {
                    if ((h ? v.y : v.x) <= 0) continue;
                    const uint32_t r = static_cast<uint32_t>(mulhi64(lane64_of(blk, h), n));
                    const uint32_t b = r >> kShift;
                    const uint32_t s = atomicAdd(scnt + b, 1u);
                    if (s < kStage) stage[b * kStage + s] = r;
                    else atomicAdd(gcur + nr, 1u);  // overflow counter (reported; never hit at random receivers)
                }
            }
        }
        fence_proxy_async();  // this thread's staged stores -> visible to the bulk copies
        __syncthreads();
        // flush full runs (a range gets < 2 * 512 / nr entries per round, so < 64 after a flush)
        for (int b = threadIdx.x; b < nr; b += blockDim.x) {
            const uint32_t c = scnt[b];
            if (c >= 32) {
                const uint32_t off = atomicAdd(gcur + b, 32u);
                if (off + 32 <= seg_cap) bulk_store(seg + b * seg_cap + off, stage + b * kStage, 128);
                bulk_commit_wait_read();
                const uint32_t cc = c < kStage ? c : kStage;
                for (uint32_t k = 32; k < cc; ++k) stage[b * kStage + k - 32] = stage[b * kStage + k];
                scnt[b] = cc - 32;
            }
        }
        __syncthreads();
    }
    // partial runs: plain stores, padded to 4 entries with a sentinel (pass 2
    // skips it) so every segment offset stays 16-byte aligned for the bulk copies
    for (int b = threadIdx.x; b < nr; b += blockDim.x) {
        const uint32_t c = min(scnt[b], static_cast<uint32_t>(kStage));
        if (!c) continue;
        const uint32_t c4 = (c + 3) & ~3u;
        const uint32_t off = atomicAdd(gcur + b, c4);
        for (uint32_t k = 0; k < c4; ++k)
            if (off + k < seg_cap) seg[b * seg_cap + off + k] = k < c ? stage[b * kStage + k] : 0xffffffffu;
    }
}

// Pass 2: two CTAs per range; each builds the 4-bit histogram of its half of the
// range's entries in shared memory and adds it into the packed counters with
// one bulk reduce.
__global__ void __launch_bounds__(1024) hist_pass(const uint32_t* __restrict__ seg, int64_t seg_cap,
                                                  const uint32_t* __restrict__ gcur, int64_t n, uint32_t* packed)
{
    extern __shared__ __align__(16) uint32_t hist[];  // kHistWords
    const int b = blockIdx.x >> 1, half = blockIdx.x & 1;
    for (int k = threadIdx.x; k < kHistWords; k += blockDim.x) hist[k] = 0u;
    __syncthreads();
    const int64_t cnt = static_cast<int64_t>(gcur[b]) < seg_cap ? static_cast<int64_t>(gcur[b]) : seg_cap;
    const int64_t e0 = half ? cnt / 2 : 0, e1 = half ? cnt : cnt / 2;
    const uint32_t* s = seg + b * seg_cap;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const uint32_t r = s[e];
        if (r == 0xffffffffu) continue;  // padding
        const uint32_t loc = r & ((1u << kShift) - 1u);
        atomicAdd(hist + (loc >> 3), 1u << ((loc & 7u) * 4u));
    }
    fence_proxy_async();
    __syncthreads();
    const int64_t words_total = (n + 7) / 8;
    const int64_t w0 = static_cast<int64_t>(b) * kHistWords;
    const int64_t words = kHistWords < words_total - w0 ? kHistWords : words_total - w0;
    if (threadIdx.x == 0 && words > 0) {
        // 4096-byte pieces (bulk sizes are multiples of 16 B)
        for (int64_t k = 0; k < words; k += 1024) {
            const int64_t nw = words - k < 1024 ? words - k : 1024;
            bulk_reduce_add_u32(packed + w0 + k, hist + k, static_cast<uint32_t>(((nw * 4) + 15) & ~15ll));
        }
        bulk_commit_wait_all();
    }
}

__global__ void unpack_compare(const uint32_t* packed, const uint32_t* ref, int64_t n, unsigned long long* bad)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (packed[i >> 3] >> ((i & 7) * 4)) & 0xfu;
        if (v != ref[i]) atomicAdd(bad, 1ull);
    }
}

int main(int argc, char** argv)
{
    const int64_t n = argc > 1 ? atoll(argv[1]) : 100000000ll;
    const uint32_t t = 5;
    const PhiloxKey K = philox_key(11ull);
    const int nr = static_cast<int>((n + (1 << kShift) - 1) >> kShift);
    const int64_t seg_cap = ((static_cast<int64_t>(1) << kShift) * 3) / 2 + 4096;  // expected 0.59 * 2^18 per range
    int32_t* w;
    uint32_t *ref, *packed, *seg, *gcur;
    unsigned long long* bad;
    const int64_t pw = (n + 7) / 8 + 1024;
    CK(cudaMalloc(&w, n * 4));
    CK(cudaMalloc(&ref, n * 4));
    CK(cudaMalloc(&packed, pw * 4));
    CK(cudaMalloc(&seg, static_cast<size_t>(nr) * seg_cap * 4));
    CK(cudaMalloc(&gcur, (nr + 1) * 4));  // + the staging-overflow counter
    CK(cudaMalloc(&bad, 8));
    fill_w<<<148 * 8, 256>>>(w, n);
    CK(cudaMemset(ref, 0, n * 4));
    scatter_ref<<<148 * 8, 256>>>(w, n, K, t, ref);
    CK(cudaDeviceSynchronize());

    cudaEvent_t e0, e1, e2;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&e2));
    float best_red = 1e9f, best_bin = 1e9f, best_hist = 1e9f;
    const size_t smem1 = static_cast<size_t>(nr) * kStage * 4 + nr * 4;
    const size_t smem2 = static_cast<size_t>(kHistWords) * 4;
    CK(cudaFuncSetAttribute(bin_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem1)));
    CK(cudaFuncSetAttribute(hist_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2)));
    unsigned long long h_bad = 0;
    for (int rep = 0; rep < 5; ++rep) {
        CK(cudaMemset(packed, 0, pw * 4));
        CK(cudaEventRecord(e0));
        scatter_red<<<148 * 8, 256>>>(w, n, K, t, packed);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best_red = ms < best_red ? ms : best_red;
        CK(cudaMemset(bad, 0, 8));
        unpack_compare<<<148 * 8, 256>>>(packed, ref, n, bad);
        CK(cudaMemcpy(&h_bad, bad, 8, cudaMemcpyDeviceToHost));
        if (h_bad) { fprintf(stderr, "red: %llu mismatches\n", h_bad); return 1; }

        CK(cudaMemset(packed, 0, pw * 4));
        CK(cudaMemset(gcur, 0, (nr + 1) * 4));
        CK(cudaEventRecord(e0));
        bin_pass<<<148, 512, smem1>>>(w, n, K, t, nr, seg, seg_cap, gcur);
        CK(cudaEventRecord(e1));
        hist_pass<<<2 * nr, 1024, smem2>>>(seg, seg_cap, gcur, n, packed);
        CK(cudaEventRecord(e2));
        CK(cudaEventSynchronize(e2));
        float ms1, ms2;
        CK(cudaEventElapsedTime(&ms1, e0, e1));
        CK(cudaEventElapsedTime(&ms2, e1, e2));
        best_bin = ms1 < best_bin ? ms1 : best_bin;
        best_hist = ms2 < best_hist ? ms2 : best_hist;
        CK(cudaMemset(bad, 0, 8));
        unpack_compare<<<148 * 8, 256>>>(packed, ref, n, bad);
        CK(cudaMemcpy(&h_bad, bad, 8, cudaMemcpyDeviceToHost));
        if (h_bad) { fprintf(stderr, "bulk: %llu mismatches\n", h_bad); return 1; }
    }
    std::vector<uint32_t> hc(nr + 1);
    CK(cudaMemcpy(hc.data(), gcur, (nr + 1) * 4, cudaMemcpyDeviceToHost));
    uint32_t mx = 0;
    for (int b = 0; b < nr; ++b) mx = hc[b] > mx ? hc[b] : mx;
    if (hc[nr]) { fprintf(stderr, "staging overflow %u\n", hc[nr]); return 1; }
    printf("N=%lld ranges=%d (2^%d agents) max range entries %u (cap %lld)\n", static_cast<long long>(n), nr, kShift,
           mx, static_cast<long long>(seg_cap));
    printf("red  (one RED per transfer, packed 4-bit): %.4f ms  exact\n", best_red);
    printf("bulk (bin + cp.async.bulk, hist + cp.reduce.async.bulk): %.4f + %.4f = %.4f ms  exact\n", best_bin,
           best_hist, best_bin + best_hist);
    return 0;
}
