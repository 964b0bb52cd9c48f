// alu_ceiling.cu -- measured ALU ceilings for the Boids stencil (SURVEY 8(d):
// "report against a measured FFMA ceiling ... measure it").
//
// Part 1: issue throughput of the instruction classes the stencil is made of
// (FADD, FMUL, 32-bit IADD, 64-bit IADD, F2I.S32, F2I.S64), in lane-ops per
// clock per SM, from chains of 8 independent accumulators per thread at full
// occupancy.
// Part 2: the stencil's own candidate loop (the B2/B3 accumulate of
// boids.cu, both the float-velocity form and the pre-quantised-velocity form)
// over candidates staged in shared memory -- memory latency hidden, so the
// rate is the ALU/issue ceiling of that exact instruction sequence.  The
// candidates are uniform in the 3x3-cell stencil box (cells of side R), so a
// fraction pi/9 = 0.35 of them are neighbours, as at BASELINE config 3.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/alu_ceiling tools/alu_ceiling.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(256) op_kernel(float seed, long long* sink, unsigned long long* cyc)
{
    const long long t0 = clock64();
    float f[8];
    int i32[8];
    long long i64[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        f[k] = seed + k + threadIdx.x * 1e-3f;
        i32[k] = threadIdx.x + k;
        i64[k] = threadIdx.x * 3 + k;
    }
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (OP == 0) f[k] = __fadd_rn(f[k], 1.0001f);
            if (OP == 1) f[k] = __fmul_rn(f[k], 0.99999f);
            if (OP == 2) i32[k] = i32[k] + it;
            if (OP == 3) i64[k] = i64[k] + (long long)it;
            if (OP == 4) i32[k] += __float2int_rn(__int_as_float(i32[k] & 0x4affffff));
            if (OP == 5) i64[k] += __float2ll_rn(__int_as_float(static_cast<int>(i64[k]) & 0x4affffff));
        }
    }
    long long s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += static_cast<long long>(f[k]) + i32[k] + i64[k];
    if (s == 42) sink[0] = s;
    if (threadIdx.x == 0) atomicMax(cyc, static_cast<unsigned long long>(clock64() - t0));
}

struct Acc {
    long long n, sdx, sdy, svx, svy, ssx, ssy;
};
__device__ __forceinline__ long long q24(float f) { return __float2ll_rn(__fmul_rn(f, 16777216.0f)); }

// boids.cu boid_accumulate<false> (interior: no minimum image)
__device__ __forceinline__ void acc_float(const float4 o, const float4 me, float R2, float rs2, Acc& a)
{
    const float dx = __fsub_rn(o.x, me.x), dy = __fsub_rn(o.y, me.y);
    const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
    if (d2 <= R2) {
        const long long qx = q24(dx), qy = q24(dy);
        a.n += 1; a.sdx += qx; a.sdy += qy; a.svx += q24(o.z); a.svy += q24(o.w);
        if (d2 <= rs2) { a.ssx += qx; a.ssy += qy; }
    }
}

// the pre-quantised form: o.z/o.w carry q24(v) as int32 bits; dx, dy convert
// with a 32-bit F2I (|dx| <= R < 128)
__device__ __forceinline__ void acc_qv(const float4 o, const float4 me, float R2, float rs2, Acc& a)
{
    const float dx = __fsub_rn(o.x, me.x), dy = __fsub_rn(o.y, me.y);
    const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
    if (d2 <= R2) {
        const int qx = __float2int_rn(__fmul_rn(dx, 16777216.0f)), qy = __float2int_rn(__fmul_rn(dy, 16777216.0f));
        a.n += 1; a.sdx += qx; a.sdy += qy; a.svx += __float_as_int(o.z); a.svy += __float_as_int(o.w);
        if (d2 <= rs2) { a.ssx += qx; a.ssy += qy; }
    }
}

__device__ __forceinline__ unsigned hash32(unsigned x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }

template <bool QV>
__global__ void __launch_bounds__(256, 4) stencil_kernel(int K, int reps, float R, long long* out, unsigned long long* cyc)
{
    extern __shared__ float4 cand[];
    const long long t0 = clock64();
    const float box = 3.0f * R;
    for (int q = threadIdx.x; q < K; q += blockDim.x) {
        const unsigned h = hash32(q * 7919u + blockIdx.x * 131u);
        const float x = box * ((h & 0xffff) / 65536.0f), y = box * ((h >> 16) / 65536.0f);
        const float vx = ((hash32(h) & 0xffff) / 32768.0f) - 1.0f, vy = ((hash32(h + 1) & 0xffff) / 32768.0f) - 1.0f;
        cand[q] = QV ? make_float4(x, y, __int_as_float(__float2int_rn(vx * 16777216.0f)),
                                   __int_as_float(__float2int_rn(vy * 16777216.0f)))
                     : make_float4(x, y, vx, vy);
    }
    __syncthreads();
    const float R2 = R * R, rs2 = 0.04f * R2;
    constexpr int G = 4;
    const int sub = threadIdx.x & (G - 1);
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
        const unsigned h = hash32(threadIdx.x / G + r * 977u + blockIdx.x);
        const float4 me = make_float4(R + R * ((h & 0xffff) / 65536.0f), R + R * ((h >> 16) / 65536.0f), 0.f, 0.f);
        Acc acc{0, 0, 0, 0, 0, 0, 0};
        int q = sub;
        for (; q + G < K; q += 2 * G) {
            const float4 o0 = cand[q], o1 = cand[q + G];
            if (QV) { acc_qv(o0, me, R2, rs2, acc); acc_qv(o1, me, R2, rs2, acc); }
            else { acc_float(o0, me, R2, rs2, acc); acc_float(o1, me, R2, rs2, acc); }
        }
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            acc.n += __shfl_xor_sync(0xffffffffu, acc.n, off);
            acc.sdx += __shfl_xor_sync(0xffffffffu, acc.sdx, off);
            acc.sdy += __shfl_xor_sync(0xffffffffu, acc.sdy, off);
            acc.svx += __shfl_xor_sync(0xffffffffu, acc.svx, off);
            acc.svy += __shfl_xor_sync(0xffffffffu, acc.svy, off);
            acc.ssx += __shfl_xor_sync(0xffffffffu, acc.ssx, off);
            acc.ssy += __shfl_xor_sync(0xffffffffu, acc.ssy, off);
        }
        tot += acc.n + acc.sdx + acc.sdy + acc.svx + acc.svy + acc.ssx + acc.ssy;
    }
    if (tot == 42) out[0] = tot;
    if (threadIdx.x == 0) atomicMax(cyc, static_cast<unsigned long long>(clock64() - t0));
}

int main()
{
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    long long* sink;
    unsigned long long* cyc;
    CK(cudaMalloc(&sink, 64));
    CK(cudaMalloc(&cyc, 8));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"FADD", "FMUL", "IADD (32-bit)", "IADD (64-bit)", "F2I.S32 (+IADD)", "F2I.S64 (+IADD.64)"};
    const int blocks = nsm * 8, thr = 256;  // 2048 threads per SM
    printf("# alu_ceiling: %d SMs; lane-ops per clock per SM (8 independent chains per thread, 64 warps/SM)\n", nsm);
    for (int op = 0; op < 6; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaMemset(cyc, 0, 8));
            cudaEventRecord(a);
            switch (op) {
                case 0: op_kernel<0><<<blocks, thr>>>(1.f, sink, cyc); break;
                case 1: op_kernel<1><<<blocks, thr>>>(1.f, sink, cyc); break;
                case 2: op_kernel<2><<<blocks, thr>>>(1.f, sink, cyc); break;
                case 3: op_kernel<3><<<blocks, thr>>>(1.f, sink, cyc); break;
                case 4: op_kernel<4><<<blocks, thr>>>(1.f, sink, cyc); break;
                case 5: op_kernel<5><<<blocks, thr>>>(1.f, sink, cyc); break;
            }
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long c = 0;
            CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
            const double ops_per_sm = 8.0 * thr * 8.0 * kIters;  // 8 blocks per SM, 8 chains, kIters
            if (rep) printf("%-22s %7.1f lane-ops/clk/SM   (%.3f ms, %llu cycles per block, %.0f MHz)\n", names[op],
                            ops_per_sm / c, ms, c, c / (ms * 1e3));
        }
    }
    const int K = 2048, reps = 64;
    const float R = 10.0f;
    CK(cudaFuncSetAttribute(stencil_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, K * 16));
    CK(cudaFuncSetAttribute(stencil_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, K * 16));
    const int sblocks = nsm * 4;  // 4 x 256 threads per SM (the stencil kernel's residency)
    for (int qv = 0; qv < 2; ++qv) {
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaMemset(cyc, 0, 8));
            cudaEventRecord(a);
            if (qv) stencil_kernel<true><<<sblocks, 256, K * 16>>>(K, reps, R, sink, cyc);
            else stencil_kernel<false><<<sblocks, 256, K * 16>>>(K, reps, R, sink, cyc);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long c = 0;
            CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
            // candidate visits: per agent (4 lanes) all K candidates, 64 agents per block per rep
            const double visits = static_cast<double>(sblocks) * (256 / 4) * reps * K;
            if (rep)
                printf("stencil %-26s %.3e candidate-visits/s  (%.2f per clk per SM; %.3f ms, %.0f MHz)\n",
                       qv ? "(pre-quantised v, F2I.S32)" : "(float v, F2I.S64)", visits / (ms * 1e-3),
                       visits / nsm / c, ms, c / (ms * 1e3));
        }
    }
    return 0;
}
