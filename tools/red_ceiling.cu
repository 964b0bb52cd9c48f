// red_ceiling.cu -- random 32-bit RED throughput vs target-set size on B200
// (the ceiling for the packed-counter wealth scatter).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hash32(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__global__ void red_any(unsigned* pool, unsigned words_mask, int iters)
{
    unsigned h = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < iters; ++i) { h = hash32(h + i); atomicAdd(pool + (h & words_mask), 1u); }
}
int main()
{
    unsigned* pool; cudaMalloc(&pool, 512u << 20); cudaMemset(pool, 0, 512u << 20);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int grid = nsm * 8, thr = 256, iters = 128;
    const double n = (double)grid * thr * iters;
    for (unsigned mb : {1u, 4u, 16u, 32u, 64u, 128u, 512u}) {
        const unsigned mask = (mb << 20) / 4 - 1;
        red_any<<<grid, thr>>>(pool, mask, iters);
        cudaEventRecord(a); red_any<<<grid, thr>>>(pool, mask, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("target %4u MB: %.3f ms  %.3e REDs/s\n", mb, ms, n / ms * 1e3);
    }
    return 0;
}
