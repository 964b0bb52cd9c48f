// die_probe.cu -- microbenchmark: does die-local placement of L2 atomics pay on B200?
// (1) classify SMs by die and 2 KB pages of a pool by home die (L2 hit latency:
//     near-die lookups are faster than lookups forwarded across the die fabric);
// (2) time random 32-bit REDs over the pool (a) unrestricted, (b) restricted to
//     pages homed on the issuing SM's die.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o die_probe tools/die_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

// one warp per block; lane 0 times a dependent chain of L2 loads inside each probed page
__global__ void probe(const unsigned* pool, int npages, int page_words, int first, int count, unsigned* lat, unsigned* sm_of_block)
{
    if (threadIdx.x != 0) return;
    sm_of_block[blockIdx.x] = smid();
    for (int k = 0; k < count; ++k) {
        int p = first + k;
        if (p >= npages) break;
        const unsigned* base = pool + (size_t)p * page_words;
        unsigned idx = 0, sink = 0;
        // warm (bring into L2), then time 8 dependent loads (pool entries are 0 -> idx stays 0.. use offsets)
        for (int w = 0; w < 4; ++w) { unsigned v; asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(base + idx + w * 32)); sink += v; }
        unsigned dep;
        asm volatile("add.u32 %0, %1, 0;" : "=r"(dep) : "r"(sink));
        long long t0;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) :: "memory");
        for (int w = 0; w < 4; ++w) {
            unsigned v;
            asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(base + idx + w * 32) : "memory");
            idx += v;  // v == 0: dependency without moving
        }
        asm volatile("add.u32 %0, %1, 0;" : "=r"(dep) : "r"(idx));
        long long t1;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) :: "memory");
        sink += dep;
        lat[(size_t)blockIdx.x * npages + p] = (unsigned)((t1 - t0) / 4) + (sink == 0xDEADBEEFu ? 1u : 0u);
    }
}

__device__ __forceinline__ unsigned hash32(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

// precomputed word indices (streamed, coalesced): the only difference between runs is the target set
__global__ void red_list(unsigned* pool, const unsigned* idx0, const unsigned* idx1, const int* die_of_sm, size_t per_thread_stride, int iters)
{
    const int d = die_of_sm ? die_of_sm[smid()] : 0;
    const unsigned* idx = d ? idx1 : idx0;
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; ++i) atomicAdd(pool + idx[i * per_thread_stride + tid], 1u);
}

__global__ void red_any(unsigned* pool, size_t words, int iters)
{
    unsigned h = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < iters; ++i) { h = hash32(h + i); atomicAdd(pool + (h % words), 1u); }
}

__global__ void red_local(unsigned* pool, const int* die_of_sm, const int* pages0, int n0, const int* pages1, int n1, int page_words, int iters)
{
    const int d = die_of_sm[smid()];
    const int* pages = d ? pages1 : pages0;
    const int np = d ? n1 : n0;
    if (np == 0) return;
    unsigned h = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < iters; ++i) {
        h = hash32(h + i);
        const int p = pages[h % np];
        atomicAdd(pool + (size_t)p * page_words + (hash32(h) % page_words), 1u);
    }
}

// random L2 loads from precomputed lists, 8 independent loads in flight per thread
__global__ void ld_list(const unsigned* pool, const unsigned* idx0, const unsigned* idx1, const int* die_of_sm,
                        size_t per_thread_stride, int iters, unsigned* sink)
{
    const int d = die_of_sm ? die_of_sm[smid()] : 0;
    const unsigned* idx = d ? idx1 : idx0;
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    unsigned acc = 0;
    for (int i = 0; i + 8 <= iters; i += 8) {
        unsigned v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(pool + idx[(i + u) * per_thread_stride + tid]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
    }
    if (acc == 0xDEADBEEFu) sink[0] = acc;
}

int main()
{
    const size_t pool_bytes = 64ull << 20;     // 64 MB (32768 pages)
    const int page_words = 512;                // 2 KB
    const int npages = (int)(pool_bytes / 2048);
    unsigned* pool;
    CK(cudaMalloc(&pool, pool_bytes));
    CK(cudaMemset(pool, 0, pool_bytes));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    // --- step 1: SM die classification on 256 reference pages, one block per SM
    const int ref = 256, blocks = nsm * 2;
    unsigned *lat, *smb;
    CK(cudaMalloc(&lat, (size_t)blocks * npages * 4));
    CK(cudaMalloc(&smb, blocks * 4));
    probe<<<blocks, 32>>>(pool, npages, page_words, 0, ref, lat, smb);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned> h_lat((size_t)blocks * npages), h_sm(blocks);
    CK(cudaMemcpy(h_lat.data(), lat, h_lat.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h_sm.data(), smb, blocks * 4, cudaMemcpyDeviceToHost));
    // reference block 0: near pages = below its median
    std::vector<unsigned> l0(h_lat.begin(), h_lat.begin() + ref);
    std::vector<unsigned> s0 = l0; std::sort(s0.begin(), s0.end());
    const unsigned med0 = s0[ref / 2];
    printf("block0 on sm %u: latency min %u median %u max %u\n", h_sm[0], s0[0], med0, s0[ref - 1]);
    std::vector<int> die_of_sm(256, -1);
    for (int b = 0; b < blocks; ++b) {
        // correlation sign: agree with block 0 on near/far -> same die
        int agree = 0;
        std::vector<unsigned> lb(h_lat.begin() + (size_t)b * npages, h_lat.begin() + (size_t)b * npages + ref);
        std::vector<unsigned> sb = lb; std::sort(sb.begin(), sb.end());
        const unsigned medb = sb[ref / 2];
        for (int p = 0; p < ref; ++p) agree += ((l0[p] < med0) == (lb[p] < medb));
        die_of_sm[h_sm[b]] = agree > ref / 2 ? 0 : 1;
    }
    int n_die0 = 0, n_die1 = 0;
    for (int s = 0; s < nsm; ++s) { if (die_of_sm[s] == 0) ++n_die0; else if (die_of_sm[s] == 1) ++n_die1; }
    printf("SMs: die0 %d die1 %d (unclassified %d)\n", n_die0, n_die1, nsm - n_die0 - n_die1);
    // --- step 2: page homes, probed from one SM of die 0 (block 0's SM): near -> die 0
    const int chunk = (npages + blocks - 1) / blocks;
    probe<<<blocks, 32>>>(pool, npages, page_words, 0, 0, lat, smb);  // sm map only
    CK(cudaDeviceSynchronize());
    // probe all pages from block 0 only, in slices (one block, serial) -- use a single-block launch
    probe<<<1, 32>>>(pool, npages, page_words, 0, npages, lat, smb);
    CK(cudaDeviceSynchronize());
    unsigned sm_probe; CK(cudaMemcpy(&sm_probe, smb, 4, cudaMemcpyDeviceToHost));
    std::vector<unsigned> lp(npages);
    CK(cudaMemcpy(lp.data(), lat, npages * 4, cudaMemcpyDeviceToHost));
    std::vector<unsigned> sp = lp; std::sort(sp.begin(), sp.end());
    const unsigned medp = sp[npages / 2];
    std::vector<int> pages0, pages1;
    const int die_probe = die_of_sm[sm_probe];
    for (int p = 0; p < npages; ++p) ((lp[p] < medp) == (die_probe == 0) ? pages0 : pages1).push_back(p);
    printf("page probe from sm %u (die %d): lat p10 %u median %u p90 %u; pages die0 %zu die1 %zu\n", sm_probe,
           die_probe, sp[npages / 10], medp, sp[npages * 9 / 10], pages0.size(), pages1.size());
    (void)chunk;
    // --- step 3: RED throughput
    int *d_die, *d_p0, *d_p1;
    CK(cudaMalloc(&d_die, 256 * 4));
    CK(cudaMalloc(&d_p0, pages0.size() * 4));
    CK(cudaMalloc(&d_p1, pages1.size() * 4));
    CK(cudaMemcpy(d_die, die_of_sm.data(), 256 * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_p0, pages0.data(), pages0.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_p1, pages1.data(), pages1.size() * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int grid = nsm * 8, thr = 256, iters = 64;
    const double nred = (double)grid * thr * iters;
    for (int rep = 0; rep < 3; ++rep) {
        float ms1, ms2;
        cudaEventRecord(a); red_any<<<grid, thr>>>(pool, pool_bytes / 4, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms1, a, b);
        cudaEventRecord(a);
        red_local<<<grid, thr>>>(pool, d_die, d_p0, (int)pages0.size(), d_p1, (int)pages1.size(), page_words, iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms2, a, b);
        printf("REDs %.0f: any-die %.3f ms (%.2e/s)   die-local %.3f ms (%.2e/s)   speedup %.2fx\n", nred, ms1,
               nred / ms1 * 1e3, ms2, nred / ms2 * 1e3, ms1 / ms2);
    }
    // precomputed address lists: any-die (uniform over pool) and per-die lists (uniform over that die's pages)
    const size_t total = (size_t)grid * thr * iters;
    std::vector<unsigned> ia(total), i0(total), i1(total);
    unsigned long long st = 88172645463325252ull;
    auto rnd = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; };
    for (size_t k = 0; k < total; ++k) {
        ia[k] = (unsigned)(rnd() % (pool_bytes / 4));
        i0[k] = pages0[rnd() % pages0.size()] * page_words + (unsigned)(rnd() % page_words);
        i1[k] = pages1[rnd() % pages1.size()] * page_words + (unsigned)(rnd() % page_words);
    }
    unsigned *d_ia, *d_i0, *d_i1;
    CK(cudaMalloc(&d_ia, total * 4)); CK(cudaMalloc(&d_i0, total * 4)); CK(cudaMalloc(&d_i1, total * 4));
    CK(cudaMemcpy(d_ia, ia.data(), total * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_i0, i0.data(), total * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_i1, i1.data(), total * 4, cudaMemcpyHostToDevice));
    const size_t stride = (size_t)grid * thr;
    for (int rep = 0; rep < 3; ++rep) {
        float m1, m2, m3;
        cudaEventRecord(a); red_list<<<grid, thr>>>(pool, d_ia, d_ia, nullptr, stride, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&m1, a, b);
        cudaEventRecord(a); red_list<<<grid, thr>>>(pool, d_i0, d_i1, d_die, stride, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&m2, a, b);
        cudaEventRecord(a); red_list<<<grid, thr>>>(pool, d_i1, d_i0, d_die, stride, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&m3, a, b);
        printf("list REDs: any %.3f ms  die-local %.3f ms  die-remote %.3f ms\n", m1, m2, m3);
    }
    // random 4-byte L2 loads (the SIR walk's neighbour-bitmap probes): does a
    // die-local replica of a read-only L2-resident array pay?
    unsigned* d_sink;
    CK(cudaMalloc(&d_sink, 4));
    for (int rep = 0; rep < 3; ++rep) {
        float m1, m2, m3;
        cudaEventRecord(a); ld_list<<<grid, thr>>>(pool, d_ia, d_ia, nullptr, stride, iters, d_sink); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&m1, a, b);
        cudaEventRecord(a); ld_list<<<grid, thr>>>(pool, d_i0, d_i1, d_die, stride, iters, d_sink); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&m2, a, b);
        cudaEventRecord(a); ld_list<<<grid, thr>>>(pool, d_i1, d_i0, d_die, stride, iters, d_sink); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&m3, a, b);
        printf("list loads %.0f: any %.3f ms (%.2e/s)  die-local %.3f ms (%.2e/s)  die-remote %.3f ms (%.2e/s)\n",
               (double)total, m1, total / m1 * 1e3, m2, total / m2 * 1e3, m3, total / m3 * 1e3);
    }
    CK(cudaGetLastError());
    return 0;
}
