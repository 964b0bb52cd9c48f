// scatter_probe.cu -- per-element cost of the ways a random "increment
// counter r" can be delivered on B200 (evidence for the wealth-scatter design,
// DESIGN.md section 5).  Every variant issues the same number of random
// 32-bit updates from a full grid (148 SMs x 2048 threads); hashing is cheap
// and identical across variants, so differences are the update path.
//
//   redg      : red.global.add.u32 into a 32 MB L2-resident array (current design)
//   atoms     : atomicAdd on shared memory, random word of a 96 KB array
//   sts       : plain st.shared to a random word (no RMW; the cost of a scatter store)
//   rmw       : ld.shared + add + st.shared (racy; what a warp-private counter costs)
//   dsmem_red : red.shared::cluster.add.u32 to a random CTA of a cluster of 8
//   stg_coal  : coalesced 4-byte global stores (bin write reference)
//   nop       : hashing only
//   ldg_rand  : random 4-byte loads from a 16 MB (L2-resident) array, summed
//               (the neighbour-bitmap lookup of the SIR walk at large N)
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned hash32(unsigned x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

constexpr int kIters = 256;
constexpr int kWords = 12 * 1024;  // 48 KB of smem counters (static limit)

template <int MODE>
__global__ void __launch_bounds__(1024, 2) probe(unsigned* g, unsigned gmask, unsigned* sink)
{
    __shared__ unsigned s[kWords];
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) s[i] = 0;
    __syncthreads();
    unsigned h = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    unsigned acc = 0;
    const unsigned long long gi = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    for (int i = 0; i < kIters; ++i) {
        h = hash32(h + i);
        if constexpr (MODE == 0) atomicAdd(g + (h & gmask), 1u);
        if constexpr (MODE == 1) atomicAdd(s + (h % kWords), 1u);
        if constexpr (MODE == 2) s[h % kWords] = h;
        if constexpr (MODE == 3) { unsigned* p = s + (h % kWords); *(volatile unsigned*)p = *(volatile unsigned*)p + 1u; }
        if constexpr (MODE == 4) atomicAdd(s + (h % kWords), (h >> 30) | 1u);
        if constexpr (MODE == 5) g[(gi + (unsigned long long)i * gridDim.x * blockDim.x) & gmask] = h;
        if constexpr (MODE == 6) if (h == 0x12345678u) sink[0] = h;
        if constexpr (MODE == 7) acc += __ldcg(g + (h & gmask));
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[1 + blockIdx.x % 64] += s[h % kWords];
    if (acc == 0x9e3779b9u) sink[0] = acc;
}

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(1024, 2) probe_dsmem(unsigned* sink)
{
    __shared__ unsigned s[kWords];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) s[i] = 0;
    cl.sync();
    unsigned h = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < kIters; ++i) {
        h = hash32(h + i);
        unsigned* p = cl.map_shared_rank(s + (h % kWords), (h >> 24) & 7);
        atomicAdd(p, 1u);
    }
    cl.sync();
    if (threadIdx.x == 0) sink[1 + blockIdx.x % 64] += s[h % kWords];
}

int main()
{
    unsigned *g, *sink;
    cudaMalloc(&g, 64u << 20);
    cudaMalloc(&sink, 4096);
    cudaMemset(g, 0, 64u << 20);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int thr = 1024;
    const unsigned mask = (32u << 20) / 4 - 1;
    auto run = [&](const char* name, auto launch, int grid) {
        launch(grid);
        cudaEventRecord(a);
        launch(grid);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double n = (double)grid * thr * kIters;
        cudaError_t e = cudaGetLastError();
        printf("%-10s grid %4d: %.3f ms  %.3e updates/s  %.3f ns/update/SM  %s\n", name, grid, ms, n / ms * 1e3,
               ms * 1e6 / (n / nsm), e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    const int grid = nsm * 2;
    run("nop", [&](int gr) { probe<6><<<gr, thr>>>(g, mask, sink); }, grid);
    run("redg", [&](int gr) { probe<0><<<gr, thr>>>(g, mask, sink); }, grid);
    run("atoms", [&](int gr) { probe<1><<<gr, thr>>>(g, mask, sink); }, grid);
    run("atoms_var", [&](int gr) { probe<4><<<gr, thr>>>(g, mask, sink); }, grid);
    run("sts", [&](int gr) { probe<2><<<gr, thr>>>(g, mask, sink); }, grid);
    run("rmw", [&](int gr) { probe<3><<<gr, thr>>>(g, mask, sink); }, grid);
    run("ldg_rand", [&](int gr) { probe<7><<<gr, thr>>>(g, (16u << 20) / 4 - 1, sink); }, grid);
    run("stg_coal", [&](int gr) { probe<5><<<gr, thr>>>(g, (16u << 20) - 1, sink); }, grid);
    int ncl = 0;
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(8 * 64);
        cfg.blockDim = dim3(thr);
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = 8;
        at.val.clusterDim.y = 1;
        at.val.clusterDim.z = 1;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        cudaOccupancyMaxActiveClusters(&ncl, probe_dsmem, &cfg);
    }
    printf("max active clusters of 8 (2 CTA/SM possible): %d\n", ncl);
    run("dsmem_red", [&](int gr) { probe_dsmem<<<gr, thr>>>(sink); }, (ncl > 0 ? ncl : 16) * 8);
    return 0;
}
