// red_stream_ceiling.cu -- the C4 wealth step's real roof on this B200: the
// random-RED stream (one 32-bit RED per transfer into L2-resident packed
// counters) issued WHILE the int32 column streams through HBM (read + write),
// as the fused wealth kernel does.  Three kernels over N = 1e8 agents:
//   stream  -- w_out[i] = f(w_in[i]) with 16-byte streaming loads/stores (800 MB)
//   red     -- f*N random REDs into a 50 MB packed-counter array (4-bit lanes)
//   fused   -- both in one pass: each agent's column word is streamed and, with
//              probability f (a hash of the id, no Philox), one RED is issued
// f = 0.587 (the equilibrium sender fraction of BASELINE config 4).  The fused
// time is the roof of wealth_step_fused (which also runs Philox and the apply).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_stream_ceiling tools/red_stream_ceiling.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__device__ __forceinline__ void red_hint(uint32_t* a, uint32_t v, unsigned long long pol)
{
    asm volatile("red.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
}

constexpr uint32_t kThresh = 2521204635u;  // 0.587 * 2^32

template <bool STREAM, bool RED>
__global__ void __launch_bounds__(256) pass(const int4* __restrict__ in, int4* __restrict__ out, uint32_t* inc,
                                            int64_t nq, uint32_t n, uint32_t salt)
{
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q0 < nq; q0 += 8 * stride) {
        int4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t q = q0 + j * stride;
            if (STREAM && q < nq) v[j] = __ldcs(in + q);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t q = q0 + j * stride;
            if (q >= nq) break;
            if (RED) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t i = static_cast<uint32_t>(4 * q + k);
                    const uint32_t h = hash32(i ^ salt);
                    if (h < kThresh) {
                        const uint32_t r = __umulhi(hash32(h + 0x9e3779b9u), n);
                        red_hint(inc + (r >> 3), 1u << ((r & 7u) * 4u), pol);
                    }
                }
            }
            if (STREAM) {
                int4 w = v[j];
                w.x += 1; w.y += 1; w.z += 1; w.w += 1;
                __stcs(out + q, w);
            }
        }
    }
}

int main()
{
    const uint32_t n = 100000000u;
    const int64_t nq = n / 4;
    int4 *a, *b;
    uint32_t* inc;
    cudaMalloc(&a, n * 4ull);
    cudaMalloc(&b, n * 4ull);
    cudaMalloc(&inc, n / 2);
    cudaMemset(a, 0, n * 4ull);
    cudaMemset(inc, 0, n / 2);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double reds = 0.587 * n;
    printf("# red_stream_ceiling: N = %u, f = 0.587 (%.3g REDs into a %u MB 4-bit counter array), %d SMs\n", n, reds,
           n / 2 >> 20, nsm);
    for (int grid_mult : {1, 2, 4, 8}) {
        const int grid = nsm * grid_mult;
        float t[3] = {0, 0, 0};
        for (int rep = 0; rep < 6; ++rep) {
            for (int kind = 0; kind < 3; ++kind) {
                cudaEventRecord(e0);
                if (kind == 0) pass<true, false><<<grid, 256>>>(a, b, inc, nq, n, rep);
                if (kind == 1) pass<false, true><<<grid, 256>>>(a, b, inc, nq, n, rep);
                if (kind == 2) pass<true, true><<<grid, 256>>>(a, b, inc, nq, n, rep);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep >= 2) t[kind] += ms / 4;  // 2 warm-ups
                cudaMemsetAsync(inc, 0, n / 2);  // keep counters from wrapping (not timed)
            }
        }
        printf("grid %4d x 256: stream %.4f ms (%.0f GB/s)  red %.4f ms (%.3g REDs/s)  fused %.4f ms "
               "(%.0f GB/s alg with 8 B/transfer)\n",
               grid, t[0], 8.0 * n / (t[0] * 1e6), t[1], reds / (t[1] * 1e-3), t[2],
               (8.0 * n + 8.0 * reds) / (t[2] * 1e6));
    }
    cudaError_t err = cudaGetLastError();
    printf("%s\n", err == cudaSuccess ? "ok" : cudaGetErrorString(err));
    return 0;
}
