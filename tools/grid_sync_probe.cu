// Cost of one grid-wide barrier in a cooperative launch on this B200:
// cooperative_groups grid.sync() vs a sense-reversing barrier (one atomic per
// block + a spin on a flag, fences around it), for several grid sizes.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/grid_sync_probe tools/grid_sync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void cg_sync(int iters, unsigned* sink)
{
    cg::grid_group g = cg::this_grid();
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += threadIdx.x ^ i;
        g.sync();
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
}

__device__ __forceinline__ void bar_sync(unsigned* count, volatile unsigned* gen, unsigned nblocks)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(const_cast<unsigned*>(gen), 1u);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void my_sync(int iters, unsigned* count, unsigned* gen, unsigned* sink)
{
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += threadIdx.x ^ i;
        bar_sync(count, gen, gridDim.x);
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
}

int main()
{
    unsigned *sink, *cnt, *gen;
    cudaMalloc(&sink, 64);
    cudaMalloc(&cnt, 4);
    cudaMalloc(&gen, 4);
    cudaMemset(cnt, 0, 4);
    cudaMemset(gen, 0, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000;
    for (int blocks : {148, 296, 391, 444, 592}) {
        for (int mode = 0; mode < 2; ++mode) {
            int it = iters;
            void* a0[] = {&it, &sink};
            void* a1[] = {&it, &cnt, &gen, &sink};
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) cudaLaunchCooperativeKernel((void*)cg_sync, blocks, 256, a0, 0, 0);
                else cudaLaunchCooperativeKernel((void*)my_sync, blocks, 256, a1, 0, 0);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%-8s blocks %4d: %.3f us per barrier (%s)\n", mode ? "custom" : "cg", blocks, ms * 1e3 / iters,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
