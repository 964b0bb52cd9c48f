// T1 RNG cross-check: the product's device Philox4x32-10
// (paper_2601_16292_b200/csrc/philox.cuh, hoisted round keys) against cuRAND's
// device routine curand_Philox4x32_10 on 2^20 pseudo-random (counter, key)
// pairs, plus the receiver arithmetic: mulhi64_n32 against __umul64hi and
// lane64_of against the R4 word layout.  Prints the mismatch counts; exit 0
// iff all are zero.  Test infrastructure (tests/test_gpu_rng_pin.py).
#include <cstdio>
#include <curand_kernel.h>

#include "philox.cuh"

__device__ __forceinline__ unsigned h32(unsigned x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__global__ void check(int n, unsigned long long* bad)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint4 c = make_uint4(h32(4 * i), h32(4 * i + 1), h32(4 * i + 2), h32(4 * i + 3));
        const unsigned long long seed = (static_cast<unsigned long long>(h32(i ^ 0x55555555u)) << 32) | h32(i + 77u);
        const uint2 k = make_uint2(static_cast<unsigned>(seed), static_cast<unsigned>(seed >> 32));
        const amber::PhiloxKey K = amber::philox_key(seed);
        const uint4 a = amber::philox(c, K);
        const uint4 b = curand_Philox4x32_10(c, k);
        if (a.x != b.x || a.y != b.y || a.z != b.z || a.w != b.w) atomicAdd(bad + 0, 1ull);
        const unsigned long long x = (static_cast<unsigned long long>(a.y) << 32) | a.x;
        const unsigned nn = h32(i * 3u + 1u) | 1u;
        if (amber::mulhi64_n32(x, nn) != static_cast<uint32_t>(__umul64hi(x, nn))) atomicAdd(bad + 1, 1ull);
        if (amber::lane64_of(a, 0) != x || amber::lane64_of(a, 1) != ((static_cast<unsigned long long>(a.w) << 32) | a.z))
            atomicAdd(bad + 2, 1ull);
    }
}

int main()
{
    unsigned long long* bad;
    cudaMalloc(&bad, 3 * sizeof(unsigned long long));
    cudaMemset(bad, 0, 3 * sizeof(unsigned long long));
    const int n = 1 << 20;
    check<<<1184, 256>>>(n, bad);
    unsigned long long h[3] = {1, 1, 1};
    cudaMemcpy(h, bad, sizeof(h), cudaMemcpyDeviceToHost);
    const cudaError_t e = cudaGetLastError();
    printf("pairs %d philox_mismatch %llu mulhi_mismatch %llu lane_mismatch %llu %s\n", n, h[0], h[1], h[2],
           cudaGetErrorString(e));
    return (e == cudaSuccess && !h[0] && !h[1] && !h[2]) ? 0 : 1;
}
