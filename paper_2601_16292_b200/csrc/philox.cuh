// philox.cuh -- device counter-based generator (DESIGN.md "Contract" R1-R8).
//
// Philox4x32-10 (Salmon et al., SC'11).  The ten round keys depend only on
// the seed, so the host expands them once into a kernel-parameter struct: in
// SASS each round is then 2 IMAD.WIDE.U32 + 2 LOP3 with the key read straight
// from the constant bank (no per-thread key schedule).
#pragma once

#ifdef __CUDACC_RTC__  // runtime-compiled expression kernels (population.cu JIT): no host headers
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#else
#include <cstdint>
#endif

namespace amber {

// R5: stream tags (counter word 3).
enum : uint32_t {
    TAG_WEALTH_RECV = 0x01u,
    TAG_SIR_TX = 0x10u,
    TAG_SIR_REC = 0x11u,
    TAG_SIR_INIT = 0x12u,
    TAG_GRAPH = 0x13u,
    TAG_BOIDS_POS = 0x20u,
    TAG_BOIDS_VEL = 0x21u,
};

struct PhiloxKey {
    uint32_t k0[10];
    uint32_t k1[10];
};

// R2: key = (lo32(seed), hi32(seed)); round r uses key + r*(W0, W1).
__host__ __device__ inline PhiloxKey philox_key(uint64_t seed)
{
    PhiloxKey k;
    uint32_t a = static_cast<uint32_t>(seed), b = static_cast<uint32_t>(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        k.k0[r] = a;
        k.k1[r] = b;
        a += 0x9E3779B9u;
        b += 0xBB67AE85u;
    }
    return k;
}

__device__ __forceinline__ PhiloxKey philox_key_dev(uint64_t seed) { return philox_key(seed); }

// R1: the block function.
__device__ __forceinline__ uint4 philox(uint4 c, const PhiloxKey& K)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const unsigned long long p0 = static_cast<unsigned long long>(0xD2511F53u) * c.x;
        const unsigned long long p1 = static_cast<unsigned long long>(0xCD9E8D57u) * c.z;
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
        c = make_uint4(hi1 ^ c.y ^ K.k0[r], lo1, hi0 ^ c.w ^ K.k1[r], lo0);
    }
    return c;
}

// R3: counter (lo32(b), hi32(b), t, tag) of block b of a per-unit stream.
__device__ __forceinline__ uint4 stream_block(const PhiloxKey& K, uint32_t tag, unsigned long long b,
                                              uint32_t t)
{
    return philox(make_uint4(static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32), t, tag), K);
}

// R4: 64-bit lane u -> words (2(u%2), 2(u%2)+1) of block u/2, low word first.
__device__ __forceinline__ unsigned long long lane64_of(uint4 w, unsigned odd)
{
    return odd ? (static_cast<unsigned long long>(w.w) << 32) | w.z
               : (static_cast<unsigned long long>(w.y) << 32) | w.x;
}

// R6: floor(x * n / 2^64).
__device__ __forceinline__ unsigned long long mulhi64(unsigned long long x, unsigned long long n)
{
    return __umul64hi(x, n);
}

// R6 specialised for n < 2^32 (two 32x32->64 products).
__device__ __forceinline__ uint32_t mulhi64_n32(unsigned long long x, uint32_t n)
{
    const unsigned long long lo = static_cast<unsigned long long>(static_cast<uint32_t>(x)) * n;
    const unsigned long long hi = static_cast<unsigned long long>(static_cast<uint32_t>(x >> 32)) * n;
    return static_cast<uint32_t>((hi + (lo >> 32)) >> 32);
}

// R7: T(p) = ceil(p * 2^32) (host); Bernoulli draw is [x32 < T] compared in 64 bits.
#ifndef __CUDACC_RTC__
inline unsigned long long bernoulli_threshold_host(double p)
{
    if (!(p >= 0.0)) return 0ull;
    if (p >= 1.0) return 4294967296ull;
    double v = p * 4294967296.0;
    unsigned long long f = static_cast<unsigned long long>(v);
    return (static_cast<double>(f) < v) ? f + 1 : f;
}
#endif

// R8: uniform float in [0, 1).
__device__ __forceinline__ float u01(uint32_t x) { return static_cast<float>(x >> 8) * (1.0f / 16777216.0f); }

}  // namespace amber
