// sirs.cu -- SIR in continuous space, the paper's SIR benchmark (PAPER.md
// Sec. 5.1.1: "agents in continuous 2D space ... transition between
// Susceptible, Infected, and Recovered states based on contact with infected
// neighbors within a fixed radius"; Listing 2: one draw per
// susceptible with >= 1 infected neighbour; C1-C4).
//
// Positions are static, so the contact graph is built ONCE at creation:
// uniform-grid binning (cell side >= r*1.001, bounded box: the stencil is
// clipped at the walls, not wrapped), a per-agent neighbour count over the
// 3x3 stencil, an exclusive scan, and a per-agent fill + row sort (the
// paper's SpatialIndex radius query, done as a grid instead of a KD-tree).
// Each step is then a pure CSR update in one cooperative launch per call
// (grid barrier per step): a susceptible checks its contacts for any I and
// takes ONE Philox draw; infected agents take a recovery draw.
#include <cooperative_groups.h>

#include <algorithm>
#include <cub/cub.cuh>

#include "graph.cuh"
#include "internal.cuh"
#include "philox.cuh"

namespace cg = cooperative_groups;

namespace amber {

namespace {

constexpr uint8_t kS = 0, kI = 1, kR = 2;
constexpr uint32_t TAG_SIRS_POS = 0x40u, TAG_SIRS_TX = 0x41u, TAG_SIRS_INIT = 0x42u, TAG_SIRS_REC = 0x43u;

struct Grid2 {
    int nc;
    float inv_cs;
};

__device__ __forceinline__ int cc(float x, const Grid2& g)
{
    int c = static_cast<int>(__fmul_rn(x, g.inv_cs));
    return c < 0 ? 0 : (c >= g.nc ? g.nc - 1 : c);
}

__global__ void sirs_pos_kernel(PhiloxKey key, int64_t n, float L, float* px, float* py)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 w = stream_block(key, TAG_SIRS_POS, static_cast<unsigned long long>(i) >> 1, 0u);
        px[i] = __fmul_rn(L, u01((i & 1) ? w.z : w.x));
        py[i] = __fmul_rn(L, u01((i & 1) ? w.w : w.y));
    }
}

__global__ void sirs_cell_kernel(const float* px, const float* py, int64_t n, Grid2 g, int* cell, int* cnt)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = cc(py[i], g) * g.nc + cc(px[i], g);
        cell[i] = c;
        atomicAdd(cnt + c, 1);
    }
}

__global__ void sirs_place_kernel(const float* px, const float* py, int64_t n, const int* cell, int* cursor,
                                  float2* sp, int32_t* sid)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int q = atomicAdd(cursor + cell[i], 1);
        sp[q] = make_float2(px[i], py[i]);
        sid[q] = static_cast<int32_t>(i);
    }
}

// C2: for agent i (id order) count (pass 0) or write (pass 1) its contacts.
template <bool FILL>
__global__ void sirs_contacts_kernel(const float* px, const float* py, int64_t n, Grid2 g, float r2,
                                     const int* start, const float2* sp, const int32_t* sid, int* deg,
                                     const int32_t* row_ptr, int32_t* col)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float xi = px[i], yi = py[i];
        const int cx = cc(xi, g), cy = cc(yi, g);
        const int span = g.nc >= 3 ? 1 : 0;
        int k = 0;
        const int32_t base = FILL ? row_ptr[i] : 0;
        for (int dy = -span; dy <= span; ++dy) {
            const int yy = cy + dy;
            if (yy < 0 || yy >= g.nc) continue;
            for (int dx = -span; dx <= span; ++dx) {
                const int xx = cx + dx;
                if (xx < 0 || xx >= g.nc) continue;
                const int c = yy * g.nc + xx;
                for (int q = start[c]; q < start[c + 1]; ++q) {
                    const int32_t j = sid[q];
                    if (j == static_cast<int32_t>(i)) continue;
                    const float ddx = __fsub_rn(sp[q].x, xi), ddy = __fsub_rn(sp[q].y, yi);
                    if (__fadd_rn(__fmul_rn(ddx, ddx), __fmul_rn(ddy, ddy)) <= r2) {
                        if (FILL) col[base + k] = j;
                        ++k;
                    }
                }
            }
        }
        if (!FILL) {
            deg[i] = k;
        } else {  // ascending row (insertion sort; rows are ~ rho*pi*r^2 long)
            for (int a = 1; a < k; ++a) {
                const int32_t v = col[base + a];
                int b = a - 1;
                while (b >= 0 && col[base + b] > v) {
                    col[base + b + 1] = col[base + b];
                    --b;
                }
                col[base + b + 1] = v;
            }
        }
    }
}

struct SirsSlot {
    unsigned long long S, I, R, digest;
};

struct SirsArgs {
    PhiloxKey key;
    const int32_t* row_ptr;  // internal (cell-ordered) CSR: neighbours as internal indices
    const int32_t* col;
    const int32_t* sid;      // internal index -> agent id (the draws are keyed by id)
    uint8_t* x[2];           // state in internal order (n_pad, padding = 3)
    int64_t n, n_pad;
    unsigned long long t_inf, t_rec;
    uint32_t t0;
    int64_t steps;
    int cur;
    SirsSlot* ring;
    int64_t ring_cap;
    int digest;
};

__device__ __forceinline__ uint32_t lane32_word(const uint4& w, uint32_t k)
{
    return k == 0 ? w.x : (k == 1 ? w.y : (k == 2 ? w.z : w.w));
}

// Steps on the internal layout: agents renumbered in grid-cell order at
// creation, so an agent's contacts are a few cells away in memory (state
// gathers hit L1/L2 lines already in use) -- the result is independent of the
// numbering because every draw is keyed by the agent id (sid).  A warp owns 32
// consecutive internal agents; the susceptible lanes' rows are walked
// cooperatively (graph.cuh walk_rows) and an owner stops at its first infected
// contact (Listing 2: one draw per exposed susceptible, so only existence
// matters).
__global__ void __launch_bounds__(256) sirs_persistent_kernel(const SirsArgs a)
{
    cg::grid_group grid = cg::this_grid();
    __shared__ int32_t sq[8][3][32];  // per warp: compacted rows (start, end) and their lanes
    int cur = a.cur;
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    // 32-bit agent indices (n < 2^31: int32 CSR)
    const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
    const int n = static_cast<int>(a.n), n_pad = static_cast<int>(a.n_pad);
    for (int64_t k = 0; k < a.steps; ++k) {
        const uint32_t t = a.t0 + static_cast<uint32_t>(k);
        const uint8_t* x = a.x[cur];
        uint8_t* y = a.x[cur ^ 1];
        unsigned long long cnt[4] = {0, 0, 0, 0};
        for (int a0 = gw * 32; a0 < n_pad; a0 += nw * 32) {
            const int u = a0 + lane;
            const bool real = u < n;
            const uint8_t st = x[u];
            const uint32_t s_mask = __ballot_sync(0xffffffffu, real && st == kS);
            uint32_t exposed = 0;
            if (s_mask) {
                // the susceptible lanes' rows compacted to lanes 0 .. k-1 (rank =
                // popc of the lower S lanes, through shared memory), so the walk
                // finds arc owners by row-end bits (graph.cuh kFast) instead of
                // the five-step shuffle search; hits map back to the lanes
                const bool mine = (s_mask >> lane) & 1u;
                const int rank = __popc(s_mask & ((1u << lane) - 1u)), cnt = __popc(s_mask);
                if (mine) {
                    sq[wq][0][rank] = a.row_ptr[u];
                    sq[wq][1][rank] = a.row_ptr[u + 1];
                    sq[wq][2][rank] = lane;
                }
                __syncwarp();
                const bool oc = lane < cnt;
                const int32_t rb = oc ? sq[wq][0][lane] : 0, re = oc ? sq[wq][1][lane] : 0;
                const int src = oc ? sq[wq][2][lane] : 0;
                __syncwarp();  // the next chunk rewrites sq
                const uint32_t own = cnt == 32 ? 0xffffffffu : (1u << cnt) - 1u;
                const uint32_t hit = walk_rows_probe<4, true>(
                    [&](int32_t e) { return static_cast<uint32_t>(__ldg(a.col + e)); }, own, rb, re,
                    [&](uint32_t j) {
                        AMBER_DCHECK(j < static_cast<uint64_t>(a.n), "SIR-space: contact id >= n");
                        return static_cast<uint32_t>(x[j] == kI);
                    },
                    [](uint32_t, int32_t, int) { return true; });
                exposed = __reduce_or_sync(0xffffffffu, ((hit >> lane) & 1u) ? 1u << src : 0u);
            }
            uint8_t o = st;
            if (real && (st == kI || ((exposed >> lane) & 1u))) {
                const uint32_t id = static_cast<uint32_t>(a.sid[u]);
                const uint4 w = stream_block(a.key, st == kI ? TAG_SIRS_REC : TAG_SIRS_TX, id >> 2, t);
                const uint32_t d = lane32_word(w, id & 3u);
                if (st == kI) {
                    if (static_cast<unsigned long long>(d) < a.t_rec) o = kR;
                } else if (static_cast<unsigned long long>(d) < a.t_inf) {
                    o = kI;
                }
            }
            y[u] = o;
            if (real) {
                cnt[0] += o == kS;
                cnt[1] += o == kI;
                cnt[2] += o == kR;
                if (a.digest) cnt[3] += digest_term(static_cast<unsigned long long>(a.sid[u]), o);
            }
        }
        SirsSlot* sl = a.ring + (t % a.ring_cap);
        unsigned long long* const outs[4] = {&sl->S, &sl->I, &sl->R, a.digest ? &sl->digest : nullptr};
        block_sum_atomic<4>(cnt, outs);
        cur ^= 1;
        grid.sync();
    }
}

// id order <-> internal order
__global__ void sirs_to_internal(const uint8_t* __restrict__ src, const int32_t* __restrict__ sid, int64_t n,
                                 uint8_t* __restrict__ dst)
{
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        dst[u] = src[sid[u]];
}

__global__ void sirs_to_ids(const uint8_t* __restrict__ src, const int32_t* __restrict__ sid, int64_t n,
                            uint8_t* __restrict__ dst)
{
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        dst[sid[u]] = src[u];
}

// Internal CSR from the id-order CSR: row u = row of agent sid[u], neighbours
// relabelled through inv (id -> internal index).
__global__ void sirs_int_deg(const int32_t* __restrict__ rp_id, const int32_t* __restrict__ sid, int64_t n,
                             int* __restrict__ deg)
{
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = sid[u];
        deg[u] = rp_id[i + 1] - rp_id[i];
    }
}

__global__ void sirs_int_fill(const int32_t* __restrict__ rp_id, const int32_t* __restrict__ col_id,
                              const int32_t* __restrict__ sid, const int32_t* __restrict__ inv, int64_t n,
                              const int32_t* __restrict__ rp_int, int32_t* __restrict__ col_int)
{
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = sid[u];
        const int32_t b = rp_id[i], e = rp_id[i + 1], o = rp_int[u];
        for (int32_t p = b; p < e; ++p) col_int[o + (p - b)] = inv[col_id[p]];
    }
}

__global__ void sirs_inv(const int32_t* __restrict__ sid, int64_t n, int32_t* __restrict__ inv)
{
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        inv[sid[u]] = static_cast<int32_t>(u);
}

__global__ void sirs_zero_slots(SirsSlot* ring, int64_t cap, int64_t s0, int64_t count)
{
    for (int64_t k = threadIdx.x; k < count && k < cap; k += blockDim.x) ring[(s0 + k) % cap] = SirsSlot{0, 0, 0, 0};
}

}  // namespace

class SirSpaceModel final : public Model {
public:
    int64_t n = 0, n_pad = 0, arcs = 0, k_inf = 0;
    amber_sir_space_params p{};
    PhiloxKey key{};
    DevBuf<float> px, py;
    DevBuf<int32_t> row_ptr, col;      // id-order contact CSR (the public columns)
    DevBuf<int32_t> row_int, col_int;  // the same graph on the internal (cell-ordered) numbering
    DevBuf<int32_t> sid;               // internal index -> agent id
    DevBuf<uint8_t> x[2];              // state, internal order
    DevBuf<uint8_t> tmp;               // id-order staging for column I/O
    int cur = 0;
    DevBuf<SirsSlot> ring;
    int64_t m_first = 0;

    SirSpaceModel(int64_t n_, const amber_sir_space_params& p_, uint64_t seed, const amber_runtime* r)
    {
        rt.init(r);
        n = n_;
        p = p_;
        AMBER_REQUIRE(n >= 1 && n < (1ll << 31), "SIR-space needs 1 <= n_agents < 2^31");
        AMBER_REQUIRE(p.L > 0 && p.r > 0 && p.p_infect >= 0 && p.p_infect <= 1 && p.p_recover >= 0 &&
                          p.p_recover <= 1 && p.init_frac >= 0 && p.init_frac <= 1,
                      "SIR-space params out of range");
        key = philox_key(seed);
        k_inf = static_cast<int64_t>(std::floor(p.init_frac * static_cast<double>(n) + 0.5));
        cudaStream_t s = rt.stream;
        const int gsz = rt.num_sms * 8;
        px.allocate(&rt, n);
        py.allocate(&rt, n);
        sirs_pos_kernel<<<gsz, 256, 0, s>>>(key, n, p.L, px.p, py.p);
        check_launch("sirs_pos_kernel");
        n_pad = ceil_div(n, 32) * 32;
        for (auto& b : x) {
            b.allocate(&rt, n_pad + 16);
            AMBER_CUDA(cudaMemsetAsync(b.p, 3, n_pad + 16, s));  // padding agents (never S or I)
        }
        tmp.allocate(&rt, n + 16);
        std::vector<unsigned long long> seeds{seed};
        build_init_state(rt, seeds, n, n, k_inf, tmp.p, TAG_SIRS_INIT);
        // contact graph, once
        Grid2 g{};
        double ncd = std::floor(static_cast<double>(p.L) / (static_cast<double>(p.r) * 1.001));
        ncd = std::min(ncd, 4096.0);
        g.nc = static_cast<int>(ncd >= 3 ? ncd : 1);
        g.inv_cs = static_cast<float>(g.nc / static_cast<double>(p.L));
        const int ncell = g.nc * g.nc;
        DevBuf<int> cell, cnt, start, cursor, deg;
        DevBuf<float2> sp;
        cell.allocate(&rt, n);
        cnt.allocate(&rt, ncell + 1);
        cnt.zero_async(s);
        start.allocate(&rt, ncell + 1);
        cursor.allocate(&rt, ncell + 1);
        sp.allocate(&rt, n);
        sid.allocate(&rt, n);
        deg.allocate(&rt, n + 1);
        deg.zero_async(s);
        sirs_cell_kernel<<<gsz, 256, 0, s>>>(px.p, py.p, n, g, cell.p, cnt.p);
        check_launch("sirs_cell_kernel");
        scan(cnt.p, start.p, ncell + 1);
        AMBER_CUDA(cudaMemcpyAsync(cursor.p, start.p, (ncell + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s));
        sirs_place_kernel<<<gsz, 256, 0, s>>>(px.p, py.p, n, cell.p, cursor.p, sp.p, sid.p);
        check_launch("sirs_place_kernel");
        const float r2 = p.r * p.r;
        sirs_contacts_kernel<false><<<gsz, 256, 0, s>>>(px.p, py.p, n, g, r2, start.p, sp.p, sid.p, deg.p, nullptr,
                                                        nullptr);
        check_launch("sirs_contacts_kernel<count>");
        row_ptr.allocate(&rt, n + 1);
        scan(deg.p, row_ptr.p, n + 1);
        int32_t total = 0;
        AMBER_CUDA(cudaMemcpyAsync(&total, row_ptr.p + n, 4, cudaMemcpyDeviceToHost, s));
        AMBER_CUDA(cudaStreamSynchronize(s));
        arcs = total;
        col.allocate(&rt, std::max<int64_t>(arcs, 1));
        sirs_contacts_kernel<true><<<gsz, 256, 0, s>>>(px.p, py.p, n, g, r2, start.p, sp.p, sid.p, nullptr,
                                                       row_ptr.p, col.p);
        check_launch("sirs_contacts_kernel<fill>");
        // internal numbering = the cell order of the binning (sid): contacts become
        // near indices, so the per-step state gathers are local
        {
            DevBuf<int32_t> inv;
            inv.allocate(&rt, n);
            sirs_inv<<<gsz, 256, 0, s>>>(sid.p, n, inv.p);
            check_launch("sirs_inv");
            deg.zero_async(s);
            sirs_int_deg<<<gsz, 256, 0, s>>>(row_ptr.p, sid.p, n, deg.p);
            check_launch("sirs_int_deg");
            row_int.allocate(&rt, n + 1);
            scan(deg.p, row_int.p, n + 1);
            col_int.allocate(&rt, std::max<int64_t>(arcs, 1));
            sirs_int_fill<<<gsz, 256, 0, s>>>(row_ptr.p, col.p, sid.p, inv.p, n, row_int.p, col_int.p);
            check_launch("sirs_int_fill");
        }
        sirs_to_internal<<<gsz, 256, 0, s>>>(tmp.p, sid.p, n, x[0].p);
        check_launch("sirs_to_internal");
        ring.allocate(&rt, metrics_cap);
        ring.zero_async(s);
        AMBER_CUDA(cudaStreamSynchronize(s));
    }

    void scan(const int* in, int* out, int64_t count)
    {
        size_t tmp = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, count, rt.stream);
        DevBuf<char> t;
        t.allocate(&rt, tmp + 16);
        AMBER_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, count, rt.stream));
        rt.sync();
    }

    ~SirSpaceModel() override
    {
        if (rt.stream) cudaStreamSynchronize(rt.stream);
        px.reset(); py.reset(); row_ptr.reset(); col.reset(); row_int.reset(); col_int.reset(); sid.reset();
        tmp.reset();
        for (auto& b : x) b.reset();
        ring.reset();
        rt.destroy();
    }

    void step(int64_t nsteps) override
    {
        AMBER_REQUIRE(nsteps >= 0 && t + nsteps < (1ll << 32), "bad n_steps");
        int64_t done = 0;
        while (done < nsteps) {
            const int64_t chunk = std::min<int64_t>(nsteps - done, metrics_cap);
            sirs_zero_slots<<<1, 256, 0, rt.stream>>>(ring.p, metrics_cap, t, chunk);
            check_launch("sirs_zero_slots");
            int per_sm = 0;
            AMBER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sirs_persistent_kernel, 256, 0));
            int blocks = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(n_pad > (1 << 22) ? per_sm : std::min(per_sm, 3)) * rt.num_sms,
                                                            std::max<int64_t>(1, ceil_div(n_pad, 256))));
            if (grid) blocks = static_cast<int>(std::min<int64_t>(grid, static_cast<int64_t>(per_sm) * rt.num_sms));
            SirsArgs a{key, row_int.p, col_int.p, sid.p, {x[0].p, x[1].p}, n, n_pad,
                       bernoulli_threshold_host(p.p_infect), bernoulli_threshold_host(p.p_recover),
                       static_cast<uint32_t>(t), chunk, cur, ring.p, metrics_cap, digest_on ? 1 : 0};
            void* kargs[] = {&a};
            prof.launch(rt.stream, "sirs_persistent", [&] {
                AMBER_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(sirs_persistent_kernel), blocks, 256,
                                                       kargs, 0, rt.stream));
            });
            check_launch("sirs_persistent_kernel");
            t += chunk;
            if (chunk & 1) cur ^= 1;
            done += chunk;
        }
    }

    bool column_info(const char* name, amber_dtype* dt, int64_t* glen, int64_t* off, int64_t* len) override
    {
        std::string k(name);
        amber_dtype d;
        int64_t L;
        if (k == "state") { d = AMBER_U8; L = n; }
        else if (k == "pos_x" || k == "pos_y") { d = AMBER_F32; L = n; }
        else if (k == "row_ptr") { d = AMBER_I32; L = n + 1; }
        else if (k == "col_idx") { d = AMBER_I32; L = arcs; }
        else return false;
        if (dt) *dt = d;
        if (glen) *glen = L;
        if (off) *off = 0;
        if (len) *len = L;
        return true;
    }

    void read_column(const char* name, void* dst, size_t bytes, bool on_dev) override
    {
        std::string k(name);
        const void* src;
        size_t nb;
        if (k == "state") { src = state_ids(); nb = n; }
        else if (k == "pos_x") { src = px.p; nb = n * 4; }
        else if (k == "pos_y") { src = py.p; nb = n * 4; }
        else if (k == "row_ptr") { src = row_ptr.p; nb = (n + 1) * 4; }
        else if (k == "col_idx") { src = col.p; nb = arcs * 4; }
        else fail(AMBER_E_UNKNOWN_NAME, "no column " + k);
        if (bytes < nb) fail(AMBER_E_BUFFER_TOO_SMALL, "dst too small for column " + k);
        copy_out(rt, dst, src, nb, on_dev);
    }

    void write_column(const char* name, const void* src, size_t bytes, bool on_dev) override
    {
        std::string k(name);
        if (k != "state") fail(AMBER_E_INVALID_ARG, "only the state column is writable (positions are static)");
        if (bytes < static_cast<size_t>(n)) fail(AMBER_E_BUFFER_TOO_SMALL, "src smaller than state column");
        copy_in(rt, tmp.p, src, n, on_dev);
        sirs_to_internal<<<rt.num_sms * 8, 256, 0, rt.stream>>>(tmp.p, sid.p, n, x[cur].p);
        check_launch("sirs_to_internal");
        rt.sync();
    }

    // the current state in id order (staging buffer)
    const uint8_t* state_ids()
    {
        sirs_to_ids<<<rt.num_sms * 8, 256, 0, rt.stream>>>(x[cur].p, sid.p, n, tmp.p);
        check_launch("sirs_to_ids");
        return tmp.p;
    }

    void read_metrics(const char* name, void* dst, size_t bytes, int64_t* n_out) override
    {
        std::string k(name);
        size_t off;
        if (k == "S") off = offsetof(SirsSlot, S);
        else if (k == "I") off = offsetof(SirsSlot, I);
        else if (k == "R") off = offsetof(SirsSlot, R);
        else if (k == "digest" && digest_on) off = offsetof(SirsSlot, digest);
        else fail(AMBER_E_UNKNOWN_NAME, "no metric " + k);
        std::vector<SirsSlot> h(metrics_cap);
        AMBER_CUDA(cudaMemcpyAsync(h.data(), ring.p, metrics_cap * sizeof(SirsSlot), cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        const int64_t first = std::max(m_first, t - metrics_cap);
        const int64_t cnt = std::max<int64_t>(t - first, 0);
        if (bytes < static_cast<size_t>(cnt) * 8) fail(AMBER_E_BUFFER_TOO_SMALL, "metrics dst too small");
        for (int64_t s = first; s < t; ++s)
            std::memcpy(static_cast<char*>(dst) + (s - first) * 8, reinterpret_cast<const char*>(&h[s % metrics_cap]) + off, 8);
        if (n_out) *n_out = cnt;
    }

    void reset_metrics() override
    {
        rt.sync();
        m_first = t;
    }

    uint64_t digest(const char* name) override
    {
        if (std::string(name) != "state") fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        return device_digest_u8(rt, state_ids(), n, 0);
    }

    void set_step(int64_t s) override
    {
        AMBER_REQUIRE(s >= 0 && s < (1ll << 32), "step out of range");
        rt.sync();
        t = s;
        m_first = s;
    }

    bool get_option(const char* key_, int64_t* v) override
    {
        if (std::string(key_) == "edges") {
            *v = arcs / 2;
            return true;
        }
        return Model::get_option(key_, v);
    }
};

Model* make_sir_space(int64_t n, const amber_sir_space_params& p, uint64_t seed, const amber_runtime* rt)
{
    return new SirSpaceModel(n, p, seed, rt);
}

}  // namespace amber
