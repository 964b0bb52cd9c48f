// sir.cu -- SIR on Erdos-Renyi contact graphs (Sec. 5.1.1,
// Listing 2, network environment Sec. 4.1;
// DESIGN.md G1-G4, S1-S6) and the batched replicate sweep (Sec. 4.2).
//
// Setup (not the hot path): a batched graph builder makes R independent
// G(n, M) graphs at once as one global CSR over R*n vertices (radix sorts of
// packed (replicate, min, max) keys, de-duplication, both arc directions,
// degree scan), and the K initial infected per replicate (segmented sort of
// the 64-bit init keys).
//
// Hot path: the per-step synchronous update.  Model (one replicate): each
// launch is one step, pull direction, one thread per 4 agents; or, with the
// "persistent" option, one cooperative launch runs all n steps with a grid
// barrier between steps.  Sweep: one CTA per replicate at a time (dynamic work
// queue), its graph, both state buffers and row offsets resident in shared
// memory for all steps, early exit once no agent is infected.
#include <cooperative_groups.h>

#include <algorithm>
#include <cub/cub.cuh>

#include "graph.cuh"
#include "internal.cuh"
#include "philox.cuh"

namespace cg = cooperative_groups;

namespace amber {

namespace {

constexpr uint8_t kS = 0, kI = 1, kR = 2, kPad = 3;

int bits_for(int64_t n)
{
    int b = 1;
    while ((1ll << b) < n) ++b;
    return b;
}

// ---------------------------------------------------------------- graph build
struct GraphBuildArgs {
    const unsigned long long* seeds;  // [R]
    int64_t R, n, m;
    int bn;  // bits per vertex id
};

// G2: e-th draw of replicate r -> packed key (r, min, max).
__global__ void er_keys_kernel(GraphBuildArgs a, unsigned long long* keys)
{
    const int64_t total = a.R * a.m;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = k / a.m, e = k - r * a.m;
        const PhiloxKey K = philox_key_dev(a.seeds[r]);
        const uint4 w = stream_block(K, TAG_GRAPH, static_cast<unsigned long long>(e), 0u);
        const unsigned long long xu = (static_cast<unsigned long long>(w.y) << 32) | w.x;
        const unsigned long long xv = (static_cast<unsigned long long>(w.w) << 32) | w.z;
        const unsigned long long u = mulhi64(xu, static_cast<unsigned long long>(a.n));
        unsigned long long v = mulhi64(xv, static_cast<unsigned long long>(a.n - 1));
        v += (v >= u);
        const unsigned long long lo = u < v ? u : v, hi = u < v ? v : u;
        keys[k] = (static_cast<unsigned long long>(r) << (2 * a.bn)) | (lo << a.bn) | hi;
    }
}

// G3: unique edges -> two arcs each (r, src, dst); duplicates -> sentinel.
__global__ void er_arcs_kernel(GraphBuildArgs a, const unsigned long long* keys, unsigned long long* arcs)
{
    const int64_t total = a.R * a.m;
    const unsigned long long mask = (1ull << a.bn) - 1;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[k];
        const bool uniq = (k == 0) || keys[k - 1] != key;
        if (uniq) {
            const unsigned long long r = key >> (2 * a.bn), lo = (key >> a.bn) & mask, hi = key & mask;
            arcs[2 * k] = (r << (2 * a.bn)) | (lo << a.bn) | hi;
            arcs[2 * k + 1] = (r << (2 * a.bn)) | (hi << a.bn) | lo;
        } else {
            arcs[2 * k] = ~0ull;
            arcs[2 * k + 1] = ~0ull;
        }
    }
}

// Degree count over the sorted valid arcs (vertex id = r*n + src), col fill.
__global__ void er_csr_kernel(GraphBuildArgs a, const unsigned long long* arcs, int64_t n_arcs, int* deg, int32_t* col)
{
    const unsigned long long mask = (1ull << a.bn) - 1;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_arcs; p += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = arcs[p];
        const unsigned long long r = key >> (2 * a.bn), src = (key >> a.bn) & mask, dst = key & mask;
        atomicAdd(deg + r * a.n + src, 1);
        col[p] = static_cast<int32_t>(dst);
    }
}

__global__ void count_valid_kernel(const unsigned long long* arcs, int64_t total, unsigned long long* n_valid)
{
    // arcs are sorted with sentinels last: find the first sentinel (binary search by one thread)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int64_t lo = 0, hi = total;
        while (lo < hi) {
            int64_t mid = (lo + hi) / 2;
            if (arcs[mid] == ~0ull) hi = mid;
            else lo = mid + 1;
        }
        *n_valid = static_cast<unsigned long long>(lo);
    }
}

// S1: init keys (64-bit lane of SIR_INIT, step 0) and ids per replicate.
__global__ void init_keys_kernel(const unsigned long long* seeds, int64_t R, int64_t n, unsigned long long* keys,
                                 int32_t* ids, uint32_t tag)
{
    const int64_t total = R * n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = k / n, i = k - r * n;
        const PhiloxKey K = philox_key_dev(seeds[r]);
        const uint4 w = stream_block(K, tag, static_cast<unsigned long long>(i / 2), 0u);
        keys[k] = lane64_of(w, static_cast<unsigned>(i & 1));
        ids[k] = static_cast<int32_t>(i);
    }
}

__global__ void init_state_kernel(const int32_t* sorted_ids, int64_t R, int64_t n, int64_t n_pad, int64_t k_inf,
                                  uint8_t* state)
{
    const int64_t total = R * n_pad;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = k % n_pad;
        state[k] = i < n ? kS : kPad;
    }
}

__global__ void init_mark_kernel(const int32_t* sorted_ids, int64_t R, int64_t n, int64_t n_pad, int64_t k_inf,
                                 uint8_t* state)
{
    const int64_t total = R * k_inf;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = k / k_inf, j = k - r * k_inf;
        state[r * n_pad + sorted_ids[r * n + j]] = kI;
    }
}

}  // namespace

void build_graphs(Runtime& rt, const std::vector<unsigned long long>& seeds, int64_t n, int64_t m, Graphs& g)
{
    const int64_t R = static_cast<int64_t>(seeds.size());
    AMBER_REQUIRE(n >= 2 && m >= 0, "graph needs n >= 2, M >= 0");
    const int bn = bits_for(n);
    const int br = R > 1 ? bits_for(R) : 0;
    AMBER_REQUIRE(2 * bn + br <= 64, "graph too large for packed 64-bit keys");
    AMBER_REQUIRE(R * 2 * m < (1ll << 31), "graph batch exceeds 2^31 arcs; use smaller batches");
    g.R = R;
    g.n = n;
    g.m = m;
    cudaStream_t s = rt.stream;
    DevBuf<unsigned long long> d_seeds, keys, keys2, arcs, arcs2, n_valid;
    DevBuf<int> deg;
    d_seeds.allocate(&rt, std::max<int64_t>(R, 1));
    AMBER_CUDA(cudaMemcpyAsync(d_seeds.p, seeds.data(), R * 8, cudaMemcpyHostToDevice, s));
    const int64_t total = R * m;
    GraphBuildArgs a{d_seeds.p, R, n, m, bn};
    const int grid = rt.num_sms * 8;
    keys.allocate(&rt, std::max<int64_t>(total, 1));
    keys2.allocate(&rt, std::max<int64_t>(total, 1));
    if (total) {
        er_keys_kernel<<<grid, 256, 0, s>>>(a, keys.p);
        check_launch("er_keys_kernel");
        size_t tmp = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.p, keys2.p, total, 0, 2 * bn + br, s);
        DevBuf<char> t;
        t.allocate(&rt, tmp + 16);
        AMBER_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, keys.p, keys2.p, total, 0, 2 * bn + br, s));
    }
    arcs.allocate(&rt, std::max<int64_t>(2 * total, 1));
    arcs2.allocate(&rt, std::max<int64_t>(2 * total, 1));
    n_valid.allocate(&rt, 1);
    n_valid.zero_async(s);
    if (total) {
        er_arcs_kernel<<<grid, 256, 0, s>>>(a, keys2.p, arcs.p);
        check_launch("er_arcs_kernel");
        keys.reset();
        keys2.reset();
        size_t tmp = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tmp, arcs.p, arcs2.p, 2 * total, 0, 64, s);
        DevBuf<char> t;
        t.allocate(&rt, tmp + 16);
        AMBER_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, arcs.p, arcs2.p, 2 * total, 0, 64, s));
        count_valid_kernel<<<1, 32, 0, s>>>(arcs2.p, 2 * total, n_valid.p);
        check_launch("count_valid_kernel");
    }
    unsigned long long nv = 0;
    AMBER_CUDA(cudaMemcpyAsync(&nv, n_valid.p, 8, cudaMemcpyDeviceToHost, s));
    AMBER_CUDA(cudaStreamSynchronize(s));
    g.arcs = static_cast<int64_t>(nv);
    deg.allocate(&rt, R * n + 1);
    deg.zero_async(s);
    g.col.allocate(&rt, std::max<int64_t>(g.arcs, 1) + 8);
    if (g.arcs) {
        er_csr_kernel<<<grid, 256, 0, s>>>(a, arcs2.p, g.arcs, deg.p, g.col.p);
        check_launch("er_csr_kernel");
    }
    g.row_ptr.allocate(&rt, R * n + 1);
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, deg.p, g.row_ptr.p, R * n + 1, s);
    DevBuf<char> t;
    t.allocate(&rt, tmp + 16);
    AMBER_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, deg.p, g.row_ptr.p, R * n + 1, s));
    AMBER_CUDA(cudaStreamSynchronize(s));
}

// S1: initial state for R replicates (row stride n_pad, padding = kPad).
void build_init_state(Runtime& rt, const std::vector<unsigned long long>& seeds, int64_t n, int64_t n_pad,
                      int64_t k_inf, uint8_t* state, uint32_t tag)
{
    const int64_t R = static_cast<int64_t>(seeds.size());
    cudaStream_t s = rt.stream;
    DevBuf<unsigned long long> d_seeds, keys, keys2;
    DevBuf<int32_t> ids, ids2;
    DevBuf<int> offsets;
    d_seeds.allocate(&rt, R);
    AMBER_CUDA(cudaMemcpyAsync(d_seeds.p, seeds.data(), R * 8, cudaMemcpyHostToDevice, s));
    keys.allocate(&rt, R * n);
    keys2.allocate(&rt, R * n);
    ids.allocate(&rt, R * n);
    ids2.allocate(&rt, R * n);
    const int grid = rt.num_sms * 8;
    init_keys_kernel<<<grid, 256, 0, s>>>(d_seeds.p, R, n, keys.p, ids.p, tag);
    check_launch("init_keys_kernel");
    std::vector<int> h_off(R + 1);
    for (int64_t r = 0; r <= R; ++r) h_off[r] = static_cast<int>(r * n);
    offsets.allocate(&rt, R + 1);
    AMBER_CUDA(cudaMemcpyAsync(offsets.p, h_off.data(), (R + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
    // stable by construction: equal keys keep ascending id order -> (key, id) order (S1)
    size_t tmp = 0;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp, keys.p, keys2.p, ids.p, ids2.p, R * n, R, offsets.p,
                                             offsets.p + 1, 0, 64, s);
    DevBuf<char> t;
    t.allocate(&rt, tmp + 16);
    AMBER_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(t.p, tmp, keys.p, keys2.p, ids.p, ids2.p, R * n, R,
                                                        offsets.p, offsets.p + 1, 0, 64, s));
    init_state_kernel<<<grid, 256, 0, s>>>(ids2.p, R, n, n_pad, k_inf, state);
    check_launch("init_state_kernel");
    if (k_inf > 0) {
        init_mark_kernel<<<grid, 256, 0, s>>>(ids2.p, R, n, n_pad, k_inf, state);
        check_launch("init_mark_kernel");
    }
    AMBER_CUDA(cudaStreamSynchronize(s));
}

namespace {

// ---------------------------------------------------------------- step kernel
struct SirSlot {
    unsigned long long S, I, R, digest;
};

struct SirStepArgs {
    PhiloxKey key;
    const int32_t* row_ptr;  // n + 1 (replicate-local offsets)
    const int32_t* col;
    uint8_t* x[2];           // ping-pong state (n_pad, padding = kPad)
    int64_t n, n_pad;
    unsigned long long t_beta, t_gamma;
    uint32_t t0;             // first step index
    int64_t n_steps;         // steps in this launch (persistent) or 1
    int cur;                 // index of the buffer holding the state at t0
    SirSlot* ring;
    int64_t ring_cap;
    int digest;
};

// One step, warp-cooperative pull.  A warp owns 32 consecutive agents
// (lane = agent).  Their CSR rows are contiguous, so the warp walks the
// concatenated arc range 32 arcs at a time (coalesced col loads, 32 independent
// neighbour-state gathers in flight); each lane finds the owner of its arc by a
// 5-step shuffle search over the row starts, draws the pair-keyed Bernoulli
// (S3) for S-owner / I-neighbour arcs, and ORs a hit into the owner's bit of a
// per-warp mask.  Owners already infected skip further draws (early exit is
// legal because the result is the OR over all S-I edges).
__device__ __forceinline__ void sir_step_body(const SirStepArgs& a, const uint8_t* __restrict__ x, uint8_t* __restrict__ y,
                                              uint32_t t, unsigned long long (&cnt)[4], uint32_t* wmask)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int32_t arcs_end = a.row_ptr[a.n];
    for (int64_t a0 = gw * 32; a0 < a.n_pad; a0 += nw * 32) {
        const int64_t i = a0 + lane;
        const bool real = i < a.n;
        const uint8_t st = x[i];
        const int32_t rb = real ? a.row_ptr[i] : arcs_end;
        const int32_t we = __shfl_sync(0xffffffffu, real ? a.row_ptr[i + 1] : arcs_end, 31);
        const int32_t wb = __shfl_sync(0xffffffffu, rb, 0);
        const bool is_s = st == kS;
        const unsigned s_lanes = __ballot_sync(0xffffffffu, is_s);
        if (lane == 0) *wmask = 0u;
        __syncwarp();
        if (s_lanes) {
            for (int32_t e0 = wb; e0 < we; e0 += 32) {
                const int32_t e = e0 + lane;
                // owner = largest lane L with rb_L <= e (rows are contiguous)
                int L = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int cand = L + step;
                    const int32_t rbc = __shfl_sync(0xffffffffu, rb, cand & 31);
                    if (cand < 32 && rbc <= e) L = cand;
                }
                const unsigned done = *wmask;
                if (e < we && ((s_lanes >> L) & 1u) && !((done >> L) & 1u)) {
                    const uint32_t j = static_cast<uint32_t>(__ldg(a.col + e));
                    if (x[j] == kI) {
                        const uint32_t s = static_cast<uint32_t>(a0 + L);
                        const uint4 w = philox(make_uint4(min(s, j), max(s, j), t, TAG_SIR_TX), a.key);
                        if (static_cast<unsigned long long>(w.x) < a.t_beta) atomicOr(wmask, 1u << L);
                    }
                }
                __syncwarp();
            }
        }
        uint8_t o = st;
        if (is_s) {
            if ((*wmask >> lane) & 1u) o = kI;
        } else if (st == kI) {
            const uint4 rec = stream_block(a.key, TAG_SIR_REC, static_cast<unsigned long long>(i >> 2), t);  // R4
            const uint32_t k = static_cast<uint32_t>(i & 3);
            const uint32_t d = k == 0 ? rec.x : (k == 1 ? rec.y : (k == 2 ? rec.z : rec.w));
            if (static_cast<unsigned long long>(d) < a.t_gamma) o = kR;
        }
        y[i] = o;
        if (real) {
            cnt[o] += 1;
            if (a.digest) cnt[3] += digest_term(static_cast<unsigned long long>(i), o);
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(256) sir_step_kernel(const SirStepArgs a)
{
    __shared__ uint32_t wmask[8];
    const uint32_t t = a.t0;
    unsigned long long cnt[4] = {0, 0, 0, 0};
    sir_step_body(a, a.x[a.cur], a.x[a.cur ^ 1], t, cnt, &wmask[threadIdx.x >> 5]);
    SirSlot* sl = a.ring + (t % a.ring_cap);
    unsigned long long* const outs[4] = {&sl->S, &sl->I, &sl->R, a.digest ? &sl->digest : nullptr};
    block_sum_atomic<4>(cnt, outs);
}

// All n_steps steps in one cooperative launch (grid barrier between steps).
// Push step (direction-optimizing, persistent kernel only).  x = state t,
// y = the other ping-pong buffer, which holds state t-1 because the previous
// step of this launch wrote it.  Every agent that is S at t was S at t-1, so y
// already reads S there; only I/R agents and newly infected agents change.
// All updates of y are 32-bit atomics on the byte's word (exact new-infection
// count from the returned old value; duplicates from several infected
// neighbours are harmless).  Result identical to pull by S3.
__device__ __forceinline__ void sir_push_body(const SirStepArgs& a, const uint8_t* __restrict__ x, uint8_t* y, uint32_t t,
                                              long long (&d)[3])
{
    uint32_t* yw = reinterpret_cast<uint32_t*>(y);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t st = x[i];
        if (st == kS || st == kPad) continue;
        const uint32_t sh = static_cast<uint32_t>(i & 3) * 8;
        const uint8_t old = y[i];  // state t-1 of agent i: nobody else writes this byte in this step
        uint8_t nw = kR;
        if (st == kI) {
            const uint4 rec = stream_block(a.key, TAG_SIR_REC, static_cast<unsigned long long>(i >> 2), t);
            const uint32_t k = static_cast<uint32_t>(i & 3);
            const uint32_t dr = k == 0 ? rec.x : (k == 1 ? rec.y : (k == 2 ? rec.z : rec.w));
            nw = (static_cast<unsigned long long>(dr) < a.t_gamma) ? kR : kI;
            if (nw == kR) {
                d[1] -= 1;
                d[2] += 1;
            }
            const int32_t b = a.row_ptr[i], e = a.row_ptr[i + 1];
            const uint32_t ii = static_cast<uint32_t>(i);
            for (int32_t p = b; p < e; ++p) {
                const uint32_t j = static_cast<uint32_t>(__ldg(a.col + p));
                if (x[j] != kS) continue;
                const uint4 w = philox(make_uint4(min(ii, j), max(ii, j), t, TAG_SIR_TX), a.key);
                if (static_cast<unsigned long long>(w.x) < a.t_beta) {
                    const uint32_t sj = (j & 3u) * 8u;
                    const uint32_t prev = atomicOr(yw + (j >> 2), 1u << sj);
                    if (((prev >> sj) & 0xFFu) == kS) {
                        d[0] -= 1;
                        d[1] += 1;
                    }
                }
            }
        }
        if (nw != old) atomicAdd(yw + (i >> 2), static_cast<uint32_t>(nw - old) << sh);
    }
}

// All n_steps steps in one cooperative launch (grid barrier between steps).
// Step k > 0 pushes from the infected agents when they are fewer than the
// susceptible ones (counts of the previous step, read from its ring slot after
// the barrier, so every block takes the same decision); otherwise it pulls.
__global__ void __launch_bounds__(256) sir_persistent_kernel(const SirStepArgs a)
{
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t wmask[8];
    int cur = a.cur;
    for (int64_t k = 0; k < a.n_steps; ++k) {
        const uint32_t t = a.t0 + static_cast<uint32_t>(k);
        SirSlot* sl = a.ring + (t % a.ring_cap);
        bool push = false;
        unsigned long long prev_s = 0, prev_i = 0, prev_r = 0;
        if (k > 0 && !a.digest) {
            const SirSlot* pv = a.ring + ((t - 1) % a.ring_cap);
            prev_s = pv->S;
            prev_i = pv->I;
            prev_r = pv->R;
            push = prev_i < prev_s;
        }
        if (push) {
            long long d[3] = {0, 0, 0};
            sir_push_body(a, a.x[cur], a.x[cur ^ 1], t, d);
            unsigned long long v[3] = {static_cast<unsigned long long>(d[0]), static_cast<unsigned long long>(d[1]),
                                       static_cast<unsigned long long>(d[2])};
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                v[0] += prev_s;
                v[1] += prev_i;
                v[2] += prev_r;
            }
            unsigned long long* const outs[3] = {&sl->S, &sl->I, &sl->R};
            block_sum_atomic<3>(v, outs);
        } else {
            unsigned long long cnt[4] = {0, 0, 0, 0};
            sir_step_body(a, a.x[cur], a.x[cur ^ 1], t, cnt, &wmask[threadIdx.x >> 5]);
            unsigned long long* const outs[4] = {&sl->S, &sl->I, &sl->R, a.digest ? &sl->digest : nullptr};
            block_sum_atomic<4>(cnt, outs);
        }
        cur ^= 1;
        grid.sync();
    }
}

__global__ void sir_zero_slots(SirSlot* ring, int64_t cap, int64_t s0, int64_t count)
{
    for (int64_t k = threadIdx.x; k < count && k < cap; k += blockDim.x) ring[(s0 + k) % cap] = SirSlot{0, 0, 0, 0};
}

}  // namespace

// ---------------------------------------------------------------- model
class SirModel final : public Model {
public:
    int64_t n = 0, n_pad = 0, m_draws = 0, k_inf = 0;
    amber_sir_params p{};
    uint64_t seed = 0;
    PhiloxKey key{};
    Graphs g;
    DevBuf<uint8_t> x[2];
    int cur = 0;
    DevBuf<SirSlot> ring;
    int64_t m_first = 0;

    SirModel(int64_t n_, const amber_sir_params& p_, uint64_t seed_, const amber_runtime* r)
    {
        rt.init(r);
        n = n_;
        p = p_;
        seed = seed_;
        key = philox_key(seed);
        AMBER_REQUIRE(n >= 2 && n < (1ll << 31), "SIR needs 2 <= n_agents < 2^31");
        AMBER_REQUIRE(p.mean_degree >= 0 && p.beta >= 0 && p.beta <= 1 && p.gamma >= 0 && p.gamma <= 1 &&
                          p.init_frac >= 0 && p.init_frac <= 1,
                      "SIR params out of range");
        m_draws = static_cast<int64_t>(std::floor(static_cast<double>(n) * p.mean_degree / 2.0 + 0.5));
        k_inf = static_cast<int64_t>(std::floor(p.init_frac * static_cast<double>(n) + 0.5));
        n_pad = ceil_div(n, 32) * 32;
        std::vector<unsigned long long> seeds{seed};
        build_graphs(rt, seeds, n, m_draws, g);
        for (auto& b : x) b.allocate(&rt, n_pad);
        build_init_state(rt, seeds, n, n_pad, k_inf, x[0].p);
        ring.allocate(&rt, metrics_cap);
        ring.zero_async(rt.stream);
        AMBER_CUDA(cudaStreamSynchronize(rt.stream));
    }

    ~SirModel() override
    {
        if (rt.stream) cudaStreamSynchronize(rt.stream);
        g.row_ptr.reset();
        g.col.reset();
        for (auto& b : x) b.reset();
        ring.reset();
        rt.destroy();
    }

    SirStepArgs args(int64_t nsteps)
    {
        SirStepArgs a{};
        a.key = key;
        a.row_ptr = g.row_ptr.p;
        a.col = g.col.p;
        a.x[0] = x[0].p;
        a.x[1] = x[1].p;
        a.n = n;
        a.n_pad = n_pad;
        a.t_beta = bernoulli_threshold_host(p.beta);
        a.t_gamma = bernoulli_threshold_host(p.gamma);
        a.t0 = static_cast<uint32_t>(t);
        a.n_steps = nsteps;
        a.cur = cur;
        a.ring = ring.p;
        a.ring_cap = metrics_cap;
        a.digest = digest_on ? 1 : 0;
        return a;
    }

    void step(int64_t nsteps) override
    {
        AMBER_REQUIRE(nsteps >= 0, "n_steps must be >= 0");
        AMBER_REQUIRE(t + nsteps < (1ll << 32), "step index would exceed 2^32");
        int64_t done = 0;
        while (done < nsteps) {
            const int64_t chunk = std::min<int64_t>(nsteps - done, metrics_cap);
            sir_zero_slots<<<1, 256, 0, rt.stream>>>(ring.p, metrics_cap, t, chunk);
            check_launch("sir_zero_slots");
            const int threads = block ? static_cast<int>(std::min<int64_t>(block, 256)) : 256;
            if (persistent && chunk > 1) {
                int per_sm = 0;
                AMBER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sir_persistent_kernel, threads, 0));
                // latency-bound: many resident warps help, but the grid barrier
                // cost grows with the block count; 3 blocks/SM measured best (C2)
                int blocks = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(std::min(per_sm, 3)) * rt.num_sms,
                                                                ceil_div(n_pad, threads)));
                if (grid) blocks = static_cast<int>(std::min<int64_t>(grid, static_cast<int64_t>(per_sm) * rt.num_sms));
                blocks = std::max(blocks, 1);
                SirStepArgs a = args(chunk);
                void* kargs[] = {&a};
                prof.launch(rt.stream, "sir_persistent", [&] {
                    AMBER_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(sir_persistent_kernel), blocks,
                                                           threads, kargs, 0, rt.stream));
                });
                check_launch("sir_persistent_kernel");
                t += chunk;
                if (chunk & 1) cur ^= 1;
            } else {
                for (int64_t k = 0; k < chunk; ++k) {
                    SirStepArgs a = args(1);
                    int blocks = static_cast<int>(ceil_div(n_pad, threads));
                    if (grid) blocks = static_cast<int>(grid);
                    prof.launch(rt.stream, "sir_step", [&] { sir_step_kernel<<<blocks, threads, 0, rt.stream>>>(a); });
                    check_launch("sir_step_kernel");
                    cur ^= 1;
                    ++t;
                }
            }
            done += chunk;
        }
    }

    bool column_info(const char* name, amber_dtype* dt, int64_t* glen, int64_t* off, int64_t* len) override
    {
        std::string k(name);
        int64_t L;
        amber_dtype d;
        if (k == "state") { d = AMBER_U8; L = n; }
        else if (k == "row_ptr") { d = AMBER_I32; L = n + 1; }
        else if (k == "col_idx") { d = AMBER_I32; L = g.arcs; }
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
        if (k == "state") { src = x[cur].p; nb = n; }
        else if (k == "row_ptr") { src = g.row_ptr.p; nb = (n + 1) * 4; }
        else if (k == "col_idx") { src = g.col.p; nb = g.arcs * 4; }
        else fail(AMBER_E_UNKNOWN_NAME, "no column " + k);
        if (bytes < nb) fail(AMBER_E_BUFFER_TOO_SMALL, "dst too small for column " + k);
        copy_out(rt, dst, src, nb, on_dev);
    }

    void write_column(const char* name, const void* src, size_t bytes, bool on_dev) override
    {
        std::string k(name);
        if (k == "row_ptr" || k == "col_idx") fail(AMBER_E_INVALID_ARG, "column " + k + " is read-only");
        if (k != "state") fail(AMBER_E_UNKNOWN_NAME, "no column " + k);
        if (bytes < static_cast<size_t>(n)) fail(AMBER_E_BUFFER_TOO_SMALL, "src smaller than state column");
        copy_in(rt, x[cur].p, src, n, on_dev);
    }

    void read_metrics(const char* name, void* dst, size_t bytes, int64_t* n_out) override
    {
        std::string k(name);
        size_t off;
        if (k == "S") off = offsetof(SirSlot, S);
        else if (k == "I") off = offsetof(SirSlot, I);
        else if (k == "R") off = offsetof(SirSlot, R);
        else if (k == "digest" && digest_on) off = offsetof(SirSlot, digest);
        else fail(AMBER_E_UNKNOWN_NAME, "no metric " + k);
        std::vector<SirSlot> h(metrics_cap);
        AMBER_CUDA(cudaMemcpyAsync(h.data(), ring.p, metrics_cap * sizeof(SirSlot), cudaMemcpyDeviceToHost, rt.stream));
        AMBER_CUDA(cudaStreamSynchronize(rt.stream));
        const int64_t first = std::max(m_first, t - metrics_cap);
        const int64_t cnt = std::max<int64_t>(t - first, 0);
        if (bytes < static_cast<size_t>(cnt) * 8) fail(AMBER_E_BUFFER_TOO_SMALL, "metrics dst too small");
        for (int64_t s = first; s < t; ++s)
            std::memcpy(static_cast<char*>(dst) + (s - first) * 8, reinterpret_cast<const char*>(&h[s % metrics_cap]) + off, 8);
        if (n_out) *n_out = cnt;
    }

    void reset_metrics() override
    {
        AMBER_CUDA(cudaStreamSynchronize(rt.stream));
        m_first = t;
    }

    uint64_t digest(const char* name) override
    {
        if (std::string(name) != "state") fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        return device_digest_u8(rt, x[cur].p, n, 0);
    }

    void set_step(int64_t s) override
    {
        AMBER_REQUIRE(s >= 0 && s < (1ll << 32), "step out of range");
        AMBER_CUDA(cudaStreamSynchronize(rt.stream));
        t = s;
        m_first = s;
    }

    bool set_option(const char* key, int64_t v) override
    {
        std::string k(key);
        if (k == "metrics_capacity") {
            AMBER_REQUIRE(v >= 16, "metrics_capacity must be >= 16");
            AMBER_CUDA(cudaStreamSynchronize(rt.stream));
            metrics_cap = v;
            ring.allocate(&rt, metrics_cap);
            ring.zero_async(rt.stream);
            m_first = t;
            return true;
        }
        if (k == "block") AMBER_REQUIRE(v <= 256, "SIR kernels are built for <= 256 threads per block");
        return Model::set_option(key, v);
    }

    bool get_option(const char* key, int64_t* v) override
    {
        std::string k(key);
        if (k == "edges") { *v = g.arcs / 2; return true; }
        return Model::get_option(key, v);
    }
};

Model* make_sir(int64_t n, const amber_sir_params& p, uint64_t seed, const amber_runtime* rt)
{
    return new SirModel(n, p, seed, rt);
}

}  // namespace amber
