// walk.cu -- Random Walk (Sec. 5.1.1: "agents move in
// continuous 2D space according to random velocity vectors with boundary
// handling"; Sec. 5.3: "vector additions ... boundary handling
// applied as vectorized clipping"; K1-K3).
//
// One streaming kernel per step: each thread owns 4 consecutive agents (one
// float4 of x, one of y, two Philox blocks -- agent 2m uses words 0-1 of
// block m, agent 2m+1 words 2-3), writes the clipped positions in place and
// accumulates the mean displacement from the origin columns.  Algorithmic
// bytes per agent-update: 16 B (x, y in and out) + 8 B (origin read for the
// observable) = 24 B; HBM-bound at scale.
#include <algorithm>
#include <cmath>

#include "internal.cuh"
#include "philox.cuh"

namespace amber {

namespace {

constexpr uint32_t TAG_WALK_POS = 0x30u, TAG_WALK_VEL = 0x31u;

__global__ void walk_init_kernel(PhiloxKey key, int64_t n, int64_t n_pad, float L, float* px, float* py, float* ox,
                                 float* oy)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pad; i += (int64_t)gridDim.x * blockDim.x) {
        float x = 0.f, y = 0.f;
        if (i < n) {
            const uint4 w = stream_block(key, TAG_WALK_POS, static_cast<unsigned long long>(i) >> 1, 0u);
            x = __fmul_rn(L, u01((i & 1) ? w.z : w.x));
            y = __fmul_rn(L, u01((i & 1) ? w.w : w.y));
        }
        px[i] = x;
        py[i] = y;
        ox[i] = x;
        oy[i] = y;
    }
}

struct WalkSlot {
    double disp;
};

__device__ __forceinline__ float walk_comp(float p, uint32_t u, float vmax, float hi)
{
    const float v = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u01(u)), 1.0f), vmax);
    float x = __fadd_rn(p, v);
    x = x < 0.0f ? 0.0f : x;
    return x > hi ? hi : x;
}

__global__ void __launch_bounds__(256) walk_step_kernel(PhiloxKey key, int64_t n, int64_t nq, float vmax, float hi,
                                                        uint32_t t, float* __restrict__ px, float* __restrict__ py,
                                                        const float* __restrict__ ox, const float* __restrict__ oy,
                                                        WalkSlot* slot, double* __restrict__ part,
                                                        unsigned int* __restrict__ done)
{
    double disp = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // two quads per iteration: all eight 16-byte loads are issued before any use
    for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q0 < nq; q0 += 2 * stride) {
      float4 X[2], Y[2], A[2], B[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t q = q0 + h * stride;
        if (q < nq) {
            X[h] = __ldcs(reinterpret_cast<const float4*>(px) + q);
            Y[h] = __ldcs(reinterpret_cast<const float4*>(py) + q);
            A[h] = __ldcs(reinterpret_cast<const float4*>(ox) + q);
            B[h] = __ldcs(reinterpret_cast<const float4*>(oy) + q);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t q = q0 + h * stride;
        if (q >= nq) break;
        const float4 x4 = X[h], y4 = Y[h], a4 = A[h], b4 = B[h];
        const unsigned long long blk = 2ull * static_cast<unsigned long long>(q);
        const uint4 w0 = stream_block(key, TAG_WALK_VEL, blk, t);      // agents 4q, 4q+1
        const uint4 w1 = stream_block(key, TAG_WALK_VEL, blk + 1, t);  // agents 4q+2, 4q+3
        float4 nx, ny;
        nx.x = walk_comp(x4.x, w0.x, vmax, hi);
        ny.x = walk_comp(y4.x, w0.y, vmax, hi);
        nx.y = walk_comp(x4.y, w0.z, vmax, hi);
        ny.y = walk_comp(y4.y, w0.w, vmax, hi);
        nx.z = walk_comp(x4.z, w1.x, vmax, hi);
        ny.z = walk_comp(y4.z, w1.y, vmax, hi);
        nx.w = walk_comp(x4.w, w1.z, vmax, hi);
        ny.w = walk_comp(y4.w, w1.w, vmax, hi);
        __stcs(reinterpret_cast<float4*>(px) + q, nx);
        __stcs(reinterpret_cast<float4*>(py) + q, ny);
        const float xs[4] = {nx.x, nx.y, nx.z, nx.w}, ys[4] = {ny.x, ny.y, ny.z, ny.w};
        const float as[4] = {a4.x, a4.y, a4.z, a4.w}, bs[4] = {b4.x, b4.y, b4.z, b4.w};
        float part = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (4 * q + k < n) {
                const float dx = __fsub_rn(xs[k], as[k]), dy = __fsub_rn(ys[k], bs[k]);
                part = __fadd_rn(part, __fsqrt_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy))));
            }
        }
        disp += static_cast<double>(part);
      }
    }
    // Deterministic reduction (no floating-point atomics): each block writes its
    // partial; the last block to finish sums the partials in a fixed order, so
    // the metric is bit-reproducible from run to run for a given launch geometry.
    __shared__ double red[8];
    __shared__ bool last;
    disp = warp_sum_f64(disp);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = disp;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
        part[blockIdx.x] = s;
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s = 0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) s += __ldcg(part + b);
    s = warp_sum_f64(s);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += red[w];
        slot->disp = tot;
        *done = 0u;  // ready for the next launch (stream-ordered)
    }
}

__global__ void walk_zero_slots(WalkSlot* ring, int64_t cap, int64_t s0, int64_t count)
{
    for (int64_t k = threadIdx.x; k < count && k < cap; k += blockDim.x) ring[(s0 + k) % cap] = WalkSlot{0.0};
}

}  // namespace

class WalkModel final : public Model {
public:
    int64_t n = 0, n_pad = 0;
    amber_walk_params p{};
    PhiloxKey key{};
    DevBuf<float> col[4];  // pos_x, pos_y, origin_x, origin_y
    DevBuf<WalkSlot> ring;
    DevBuf<double> part;       // per-block partials of the step's displacement sum
    DevBuf<unsigned int> done; // blocks finished (last-block reduction)
    int64_t m_first = 0;

    WalkModel(int64_t n_, const amber_walk_params& p_, uint64_t seed, const amber_runtime* r)
    {
        rt.init(r);
        n = n_;
        p = p_;
        AMBER_REQUIRE(n >= 1, "walk needs n_agents >= 1");
        AMBER_REQUIRE(p.L > 0 && p.vmax >= 0, "walk needs L > 0, vmax >= 0");
        key = philox_key(seed);
        n_pad = ceil_div(n, 4) * 4;
        for (auto& c : col) c.allocate(&rt, n_pad);
        ring.allocate(&rt, metrics_cap);
        ring.zero_async(rt.stream);
        done.allocate(&rt, 1);
        done.zero_async(rt.stream);
        walk_init_kernel<<<rt.num_sms * 8, 256, 0, rt.stream>>>(key, n, n_pad, p.L, col[0].p, col[1].p, col[2].p,
                                                               col[3].p);
        check_launch("walk_init_kernel");
        rt.sync();
    }

    ~WalkModel() override
    {
        if (rt.stream) cudaStreamSynchronize(rt.stream);
        for (auto& c : col) c.reset();
        ring.reset();
        part.reset();
        done.reset();
        rt.destroy();
    }

    void step(int64_t nsteps) override
    {
        AMBER_REQUIRE(nsteps >= 0 && t + nsteps < (1ll << 32), "bad n_steps");
        const float hi = std::nextafter(p.L, 0.0f);
        const int threads = block ? static_cast<int>(std::min<int64_t>(block, 256)) : 256;
        const int64_t nq = n_pad / 4;
        const int g = grid ? static_cast<int>(grid)
                           : static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nq, threads),
                                                                                     rt.num_sms * 8)));
        if (part.n < static_cast<size_t>(g)) part.allocate(&rt, g);
        int64_t ndone = 0;
        while (ndone < nsteps) {
            const int64_t chunk = std::min<int64_t>(nsteps - ndone, metrics_cap);
            walk_zero_slots<<<1, 256, 0, rt.stream>>>(ring.p, metrics_cap, t, chunk);
            check_launch("walk_zero_slots");
            for (int64_t k = 0; k < chunk; ++k) {
                prof.launch(rt.stream, "walk_step", [&] {
                    walk_step_kernel<<<g, threads, 0, rt.stream>>>(key, n, nq, p.vmax, hi, static_cast<uint32_t>(t),
                                                                   col[0].p, col[1].p, col[2].p, col[3].p,
                                                                   ring.p + (t % metrics_cap), part.p, done.p);
                });
                check_launch("walk_step_kernel");
                ++t;
            }
            ndone += chunk;
        }
    }

    int idx(const std::string& k) const
    {
        if (k == "pos_x") return 0;
        if (k == "pos_y") return 1;
        if (k == "origin_x") return 2;
        if (k == "origin_y") return 3;
        return -1;
    }

    bool column_info(const char* name, amber_dtype* dt, int64_t* glen, int64_t* off, int64_t* len) override
    {
        if (idx(name) < 0) return false;
        if (dt) *dt = AMBER_F32;
        if (glen) *glen = n;
        if (off) *off = 0;
        if (len) *len = n;
        return true;
    }

    void read_column(const char* name, void* dst, size_t bytes, bool on_dev) override
    {
        const int k = idx(name);
        if (k < 0) fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        if (bytes < static_cast<size_t>(n) * 4) fail(AMBER_E_BUFFER_TOO_SMALL, "dst too small");
        copy_out(rt, dst, col[k].p, n * 4, on_dev);
    }

    void write_column(const char* name, const void* src, size_t bytes, bool on_dev) override
    {
        const int k = idx(name);
        if (k < 0) fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        if (bytes < static_cast<size_t>(n) * 4) fail(AMBER_E_BUFFER_TOO_SMALL, "src too small");
        copy_in(rt, col[k].p, src, n * 4, on_dev);
    }

    void read_metrics(const char* name, void* dst, size_t bytes, int64_t* n_out) override
    {
        if (std::string(name) != "mean_displacement") fail(AMBER_E_UNKNOWN_NAME, std::string("no metric ") + name);
        std::vector<WalkSlot> h(metrics_cap);
        AMBER_CUDA(cudaMemcpyAsync(h.data(), ring.p, metrics_cap * sizeof(WalkSlot), cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        const int64_t first = std::max(m_first, t - metrics_cap + 1);
        const int64_t cnt = std::max<int64_t>(t - first, 0);
        if (bytes < static_cast<size_t>(cnt) * 8) fail(AMBER_E_BUFFER_TOO_SMALL, "metrics dst too small");
        for (int64_t s = first; s < t; ++s)
            static_cast<double*>(dst)[s - first] = h[s % metrics_cap].disp / static_cast<double>(n);
        if (n_out) *n_out = cnt;
    }

    void reset_metrics() override
    {
        rt.sync();
        m_first = t;
    }

    uint64_t digest(const char* name) override
    {
        const int k = idx(name);
        if (k < 0) fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        return device_digest_u32(rt, reinterpret_cast<const uint32_t*>(col[k].p), n, 0);
    }

    void set_step(int64_t s) override
    {
        AMBER_REQUIRE(s >= 0 && s < (1ll << 32), "step out of range");
        rt.sync();
        t = s;
        m_first = s;
    }

    bool set_option(const char* key_, int64_t v) override
    {
        std::string k(key_);
        if (k == "block") AMBER_REQUIRE(v <= 256, "walk kernel is built for <= 256 threads per block");
        return Model::set_option(key_, v);
    }
};

Model* make_walk(int64_t n, const amber_walk_params& p, uint64_t seed, const amber_runtime* rt)
{
    return new WalkModel(n, p, seed, rt);
}

}  // namespace amber
