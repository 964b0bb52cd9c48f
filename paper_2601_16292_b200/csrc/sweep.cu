// sweep.cu -- batched SIR replicate sweep (Sec. 4.2
// "configurable replication counts", Sec. 4.4 line 191 ParallelRunner;
// BASELINE config 5; S5-S6).
//
// All replicates' graphs and initial states are built on the device in one
// batch (sir.cu builders).  The stepping kernel is persistent: a CTA takes
// the next replicate from a work queue (ordered by beta, largest first, so the
// longest epidemics start first), stages its CSR (row offsets as u32, column
// ids as u16 when n <= 65536) and both state buffers in shared memory, runs
// all steps there, and stops early once no agent is infected (later steps
// cannot change the state: S needs an I neighbour and only I agents move).
// Both directions walk rows warp-cooperatively (graph.cuh walk_rows): the
// owners' rows of a 32-agent chunk are concatenated so every lane works on
// arcs (the thread-per-agent walk was divergence-bound, 44 -> 30 ms at C5).
// Final R / n goes to out[r].
#include <algorithm>
#include <numeric>

#include "graph.cuh"
#include "internal.cuh"
#include "philox.cuh"

namespace amber {

struct Comm;
Comm* make_comm(const amber_runtime* r);
void destroy_comm(Comm* c);
void comm_allgather_f64(Comm* c, cudaStream_t s, const double* send, double* recv, size_t n_per_rank);
void comm_allreduce_u64(Comm* c, cudaStream_t s, unsigned long long* d, size_t n);
bool loopback_allgather_f64(const amber_runtime* r, const std::vector<double>& mine, std::vector<double>& all);

namespace {

constexpr uint8_t kS = 0, kI = 1, kR = 2;
#ifndef AMBER_SWEEP_WALK_U
#define AMBER_SWEEP_WALK_U 1
#endif
constexpr int kSweepU = AMBER_SWEEP_WALK_U;  // 32-arc batches per walk iteration (shared-memory latency is short)

struct SweepArgs {
    const int32_t* row_ptr;  // R*n + 1 (global offsets)
    const int32_t* col;      // replicate-local ids
    const uint8_t* state0;   // R * n_pad
    const unsigned long long* seeds;
    const unsigned long long* t_beta;  // per replicate
    const int* order;        // processing order
    unsigned long long t_gamma;
    int64_t R, n, n_pad, steps;
    int* next;               // work-queue counter
    double* out;             // final R fraction per replicate
    unsigned long long* active_updates;
    int col_smem;            // 1: stage col as u16 in shared memory
    int64_t col_cap;         // u16 entries reserved in shared memory
};

// max over replicates k of row_ptr[(k+1) n] - row_ptr[k n] (arcs per replicate)
__global__ void sweep_max_arcs_kernel(const int32_t* __restrict__ row_ptr, int64_t R, int64_t n,
                                      unsigned int* __restrict__ out)
{
    unsigned int m = 0;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < R;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        m = max(m, static_cast<unsigned int>(row_ptr[(k + 1) * n] - row_ptr[k * n]));
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// enqueue (graph.cuh) with the queue in shared memory: the owners of `mask`
// (agents a0 + b) are appended at slots qc + rank; at 32 queued, lane l's
// owner is slot l and the walk runs; the remainder moves to the front.
template <class W>
__device__ __forceinline__ void enqueue_sq(uint32_t mask, uint32_t a0, uint16_t* sq, uint32_t& qid, uint32_t& qc,
                                           W&& walk)
{
    const uint32_t lane = threadIdx.x & 31, k = __popc(mask);
    if (!k) return;
    if ((mask >> lane) & 1u) sq[qc + __popc(mask & ((1u << lane) - 1u))] = static_cast<uint16_t>(a0 + lane);
    __syncwarp();
    qc += k;
    if (qc < 32) return;
    qid = sq[lane];
    walk(32u);
    const uint32_t rem = qc - 32;
    const uint16_t v = lane < rem ? sq[32 + lane] : 0;
    __syncwarp();
    if (lane < rem) sq[lane] = v;
    __syncwarp();
    qc = rem;
}

template <bool COL_SMEM>
__global__ void __launch_bounds__(1024, 1) sir_sweep_kernel(const SweepArgs a)
{
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* rp = reinterpret_cast<uint32_t*>(smem);                  // n + 1
    uint16_t* cs = reinterpret_cast<uint16_t*>(rp + ((a.n + 4) & ~3ll));  // col_cap (COL_SMEM)
    uint8_t* xs = reinterpret_cast<uint8_t*>(cs + (COL_SMEM ? ((a.col_cap + 7) & ~7ll) : 0));
    // COL_SMEM (n <= 65536): each warp's owner queue as 64 u16 slots in shared
    // memory -- queued by rank (popc of the lower set bits), one STS per owner,
    // instead of a register queue filled with __fns (r02 ncu: __fns and its
    // enqueue were 16% of the sweep's instructions)
    uint16_t* sq = COL_SMEM ? reinterpret_cast<uint16_t*>(xs + ((2 * a.n_pad + 15) & ~15ll)) + (threadIdx.x >> 5) * 64
                            : nullptr;
    __shared__ int rep_s;
    __shared__ int cnt_s[2][2];  // [parity][I, S]
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    // (Measured, not kept, r02: the push's owner scan from an infected-agent
    // bitmap written by the copy pass, one set bit per lane per round over 32
    // words: C5 28.1 vs 24.3 ms -- a round per owner rank costs more than the
    // byte load + ballot per 32 agents it replaces.)
    // 32-bit indices inside a replicate (its state lives in shared memory, so
    // n_pad < 2^17; 64-bit loop counters cost two instructions per compare /
    // increment: C5 25.5 -> 24.1 ms)
    const int n = static_cast<int>(a.n), n_pad = static_cast<int>(a.n_pad);
    const int nq = n_pad / 4;

    for (;;) {
        if (tid == 0) rep_s = atomicAdd(a.next, 1);
        __syncthreads();
        const int slot = rep_s;
        __syncthreads();
        if (slot >= a.R) break;
        const int r = a.order[slot];
        const int32_t base = a.row_ptr[static_cast<int64_t>(r) * a.n];
        const int32_t* gcol = a.col + base;
        for (int64_t v = tid; v <= a.n; v += nt) rp[v] = static_cast<uint32_t>(a.row_ptr[r * a.n + v] - base);
        __syncthreads();
        if constexpr (COL_SMEM) {
            const uint32_t na = rp[a.n];
            for (uint32_t p = tid; p < na; p += nt) cs[p] = static_cast<uint16_t>(gcol[p]);
        }
        const uchar4* s0 = reinterpret_cast<const uchar4*>(a.state0 + static_cast<int64_t>(r) * a.n_pad);
        for (int q = tid; q < nq; q += nt) reinterpret_cast<uchar4*>(xs)[q] = s0[q];
        if (tid == 0) cnt_s[0][0] = cnt_s[0][1] = cnt_s[1][0] = cnt_s[1][1] = 0;
        __syncthreads();
        const PhiloxKey key = philox_key(a.seeds[r]);
        auto col_at = [&](int32_t e) {
            AMBER_DCHECK(e >= 0 && (!COL_SMEM || e < a.col_cap), "sweep: arc index out of the staged columns");
            const uint32_t j = COL_SMEM ? static_cast<uint32_t>(cs[e]) : static_cast<uint32_t>(gcol[e]);
            AMBER_DCHECK(j < static_cast<uint64_t>(a.n), "sweep: neighbour id >= n");
            return j;
        };
        const unsigned long long tb = a.t_beta[r];
        int cur = 0;
        int64_t executed = a.steps;
        // initial S / I counts (direction choice of the first step)
        {
            int ni = 0, ns = 0;
            for (int i = tid; i < n; i += nt) {
                ni += xs[i] == kI;
                ns += xs[i] == kS;
            }
            ni = __reduce_add_sync(0xffffffffu, ni);
            ns = __reduce_add_sync(0xffffffffu, ns);
            if ((tid & 31) == 0) {
                atomicAdd(&cnt_s[0][0], ni);
                atomicAdd(&cnt_s[0][1], ns);
            }
            __syncthreads();
        }
        for (int64_t t = 0; t < a.steps; ++t) {
            // derived from the shared-memory base, so the accesses stay LDS/STS
            const uint8_t* x = xs + (cur ? n_pad : 0);
            uint8_t* y = xs + (cur ? 0 : n_pad);
            const int par = static_cast<int>(t & 1);
            const int prev_inf = cnt_s[par][0], prev_sus = cnt_s[par][1];
            if (prev_inf == 0) {  // no infected agent: nothing can change any more
                executed = t;
                break;
            }
            int n_inf = 0, n_sus = 0;
            if (prev_inf < prev_sus) {
                // push: recoveries + copy, then each infected agent tries its susceptible
                // neighbours (S3: the pair-keyed draw makes this identical to pull).
                // (A one-pass push on the back-buffer invariant, as in sir.cu, measured
                // slower here: 35.7 vs 29.7 ms for C5 -- in shared memory the vectorised
                // copy pass is cheap and the extra atomics are not.)
                for (int q = tid; q < nq; q += nt) {
                    const uchar4 v = reinterpret_cast<const uchar4*>(x)[q];
                    uint8_t o[4] = {v.x, v.y, v.z, v.w};
                    if (o[0] == kI || o[1] == kI || o[2] == kI || o[3] == kI) {
                        const uint4 rec = stream_block(key, TAG_SIR_REC, static_cast<unsigned long long>(q), static_cast<uint32_t>(t));
                        const uint32_t rw[4] = {rec.x, rec.y, rec.z, rec.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (o[k] == kI && static_cast<unsigned long long>(rw[k]) < a.t_gamma) o[k] = kR;
                    }
                    reinterpret_cast<uchar4*>(y)[q] = make_uchar4(o[0], o[1], o[2], o[3]);
                }
                __syncthreads();
                // warp-cooperative: the infected agents of the warp's chunks are
                // queued (one per lane, compacted across chunks) and walk their
                // concatenated rows 32 owners at a time (graph.cuh walk_rows), so
                // the walk's lanes are full even when few agents are infected
                uint32_t qid = 0, qc = 0;  // lane's queued owner; queued count (warp-uniform)
                auto walk_push = [&](uint32_t nown) {
                    const bool mine = static_cast<uint32_t>(lane) < nown;
                    const int32_t rb = mine ? static_cast<int32_t>(rp[qid]) : 0, re = mine ? static_cast<int32_t>(rp[qid + 1]) : 0;
                    const uint32_t own = nown >= 32 ? 0xffffffffu : ((1u << nown) - 1u);
                    walk_rows_pay<kSweepU, true>(col_at, own, rb, re, qid,
                                     [&](uint32_t j) { return static_cast<uint32_t>(x[j] == kS && y[j] == kS); },
                                     [&](uint32_t j, int32_t, int, uint32_t ii) {  // y: already hit this step
                        const uint4 w = philox(make_uint4(min(ii, j), max(ii, j), static_cast<uint32_t>(t), TAG_SIR_TX), key);
                        if (static_cast<unsigned long long>(w.x) < tb) y[j] = kI;
                        return false;
                    });
                };
                for (int a0 = warp * 32; a0 < n_pad; a0 += nwarps * 32) {
                    const int i = a0 + lane;
                    const uint32_t own = __ballot_sync(0xffffffffu, i < n && x[i] == kI);
                    if constexpr (COL_SMEM) enqueue_sq(own, static_cast<uint32_t>(a0), sq, qid, qc, walk_push);
                    else enqueue(own, static_cast<uint32_t>(a0), qid, qc, walk_push);
                }
                if (qc) {
                    if constexpr (COL_SMEM) qid = static_cast<uint32_t>(lane) < qc ? sq[lane] : 0u;
                    walk_push(qc);
                }
                __syncthreads();
                // counts of the pushed state, four bytes per load (padding bytes are 3)
                for (int q = tid; q < nq; q += nt) {
                    const uint32_t v = reinterpret_cast<const uint32_t*>(y)[q];
                    n_inf += __popc(__vcmpeq4(v, 0x01010101u)) >> 3;
                    n_sus += __popc(__vcmpeq4(v, 0x00000000u)) >> 3;
                }
            } else {
                // pull, warp-cooperative: the susceptible agents of the warp's chunks
                // are queued (compacted across chunks) and walk their concatenated
                // rows 32 owners at a time; an owner stops at its first transmitting
                // arc and writes its own next state
                uint32_t qid = 0, qc = 0;
                auto walk_pull = [&](uint32_t nown) {
                    const bool mine = static_cast<uint32_t>(lane) < nown;
                    const int32_t rb = mine ? static_cast<int32_t>(rp[qid]) : 0, re = mine ? static_cast<int32_t>(rp[qid + 1]) : 0;
                    const uint32_t own = nown >= 32 ? 0xffffffffu : ((1u << nown) - 1u);
                    const uint32_t hit = walk_rows_pay<kSweepU, true>(col_at, own, rb, re, qid,
                                                          [&](uint32_t j) { return static_cast<uint32_t>(x[j] == kI); },
                                                          [&](uint32_t j, int32_t, int, uint32_t ii) {
                        const uint4 w = philox(make_uint4(min(ii, j), max(ii, j), static_cast<uint32_t>(t), TAG_SIR_TX), key);
                        return static_cast<unsigned long long>(w.x) < tb;
                    });
                    if (mine) {
                        const bool h = (hit >> lane) & 1u;
                        y[qid] = h ? kI : kS;
                        n_inf += h;
                        n_sus += !h;
                    }
                };
                for (int a0 = warp * 32; a0 < n_pad; a0 += nwarps * 32) {
                    const int i = a0 + lane;
                    const bool real = i < n;
                    const uint8_t in = i < n_pad ? x[i] : static_cast<uint8_t>(3);  // 3 = padding
                    const uint32_t s_mask = __ballot_sync(0xffffffffu, real && in == kS);
                    const uint32_t i_mask = __ballot_sync(0xffffffffu, real && in == kI);
                    // R4 recovery draws: one Philox block per 4 agents, computed by the
                    // group's first lane and shuffled to the other three
                    uint32_t rw = 0;
                    if (i_mask) {
                        uint4 rec = make_uint4(0u, 0u, 0u, 0u);
                        if ((lane & 3) == 0 && ((i_mask >> lane) & 0xFu))
                            rec = stream_block(key, TAG_SIR_REC, static_cast<unsigned long long>(i >> 2), static_cast<uint32_t>(t));
                        const int src = lane & ~3;
                        const uint32_t r0 = __shfl_sync(0xffffffffu, rec.x, src), r1 = __shfl_sync(0xffffffffu, rec.y, src);
                        const uint32_t r2 = __shfl_sync(0xffffffffu, rec.z, src), r3 = __shfl_sync(0xffffffffu, rec.w, src);
                        const int k = lane & 3;
                        rw = k == 0 ? r0 : (k == 1 ? r1 : (k == 2 ? r2 : r3));
                    }
                    // susceptible agents are written by their walk
                    if (!((s_mask >> lane) & 1u)) {
                        uint8_t o = in;
                        if (real && in == kI && static_cast<unsigned long long>(rw) < a.t_gamma) o = kR;
                        if (i < n_pad) y[i] = o;
                        n_inf += real && o == kI;
                    }
                    if constexpr (COL_SMEM) enqueue_sq(s_mask, static_cast<uint32_t>(a0), sq, qid, qc, walk_pull);
                    else enqueue(s_mask, static_cast<uint32_t>(a0), qid, qc, walk_pull);
                }
                if (qc) {
                    if constexpr (COL_SMEM) qid = static_cast<uint32_t>(lane) < qc ? sq[lane] : 0u;
                    walk_pull(qc);
                }
            }
            n_inf = __reduce_add_sync(0xffffffffu, n_inf);
            n_sus = __reduce_add_sync(0xffffffffu, n_sus);
            if ((tid & 31) == 0) {
                if (n_inf) atomicAdd(&cnt_s[par ^ 1][0], n_inf);
                if (n_sus) atomicAdd(&cnt_s[par ^ 1][1], n_sus);
            }
            __syncthreads();
            if (tid == 0) cnt_s[par][0] = cnt_s[par][1] = 0;
            cur ^= 1;
            __syncthreads();
        }
        // final R count
        int n_rec = 0;
        for (int i = tid; i < n; i += nt) n_rec += (xs[(cur ? n_pad : 0) + i] == kR);
        n_rec = __reduce_add_sync(0xffffffffu, n_rec);
        if (tid == 0) cnt_s[0][0] = 0;
        __syncthreads();
        if ((tid & 31) == 0 && n_rec) atomicAdd(&cnt_s[0][0], n_rec);
        __syncthreads();
        if (tid == 0) {
            a.out[r] = static_cast<double>(cnt_s[0][0]) / static_cast<double>(a.n);
            atomicAdd(a.active_updates, static_cast<unsigned long long>(executed) * a.n);
        }
        __syncthreads();
    }
}

}  // namespace

void run_sweep(int64_t n, const amber_sir_params& base, const amber_replicate* reps, int64_t n_reps, int64_t n_steps,
               const amber_runtime* r, double* out, amber_sweep_stats* stats)
{
    Runtime rt;
    rt.init(r);
    struct Guard {
        Runtime& rt;
        ~Guard() { rt.destroy(); }
    } guard{rt};
    AMBER_REQUIRE(n >= 2 && n < (1ll << 31), "sweep needs 2 <= n_agents < 2^31");
    AMBER_REQUIRE(base.gamma >= 0 && base.gamma <= 1 && base.init_frac >= 0 && base.init_frac <= 1 &&
                      base.mean_degree >= 0,
                  "sweep params out of range");
    const int W = rt.world, me = rt.rank;
    const int64_t per = ceil_div(std::max<int64_t>(n_reps, 1), W);
    int64_t r0, r1;
    sweep_range(n_reps, W, me, &r0, &r1);
    const int64_t R = r1 - r0;
    const int64_t m = static_cast<int64_t>(std::floor(static_cast<double>(n) * base.mean_degree / 2.0 + 0.5));
    const int64_t k_inf = static_cast<int64_t>(std::floor(base.init_frac * static_cast<double>(n) + 0.5));
    const int64_t n_pad = ceil_div(n, 16) * 16;
    std::vector<double> local(std::max<int64_t>(per, 1), 0.0);
    double build_ms = 0, step_ms = 0;
    unsigned long long active = 0;
    cudaEvent_t e0, e1, e2;
    AMBER_CUDA(cudaEventCreate(&e0));
    AMBER_CUDA(cudaEventCreate(&e1));
    AMBER_CUDA(cudaEventCreate(&e2));
    // batches bound the setup memory (sort buffers) for very large sweeps
    const int64_t batch_cap = std::max<int64_t>(1, std::min<int64_t>(R, ((1ll << 31) - 1) / std::max<int64_t>(2 * m, 1)));
    for (int64_t b0 = 0; b0 < R; b0 += batch_cap) {
        const int64_t B = std::min(batch_cap, R - b0);
        std::vector<unsigned long long> seeds(B), tb(B);
        std::vector<std::pair<double, int>> ord(B);
        for (int64_t k = 0; k < B; ++k) {
            const amber_replicate& rep = reps[r0 + b0 + k];
            AMBER_REQUIRE(rep.beta >= 0 && rep.beta <= 1, "replicate beta out of [0,1]");
            seeds[k] = rep.seed;
            tb[k] = bernoulli_threshold_host(rep.beta);
            ord[k] = {-rep.beta, static_cast<int>(k)};
        }
        std::stable_sort(ord.begin(), ord.end());
        std::vector<int> order(B);
        for (int64_t k = 0; k < B; ++k) order[k] = ord[k].second;
        AMBER_CUDA(cudaEventRecord(e0, rt.stream));
        Graphs g;
        build_graphs(rt, seeds, n, m, g);
        DevBuf<uint8_t> st0;
        st0.allocate(&rt, B * n_pad);
        build_init_state(rt, seeds, n, n_pad, k_inf, st0.p);
        DevBuf<unsigned long long> d_seeds, d_tb, d_active;
        DevBuf<int> d_order, d_next;
        DevBuf<double> d_out;
        d_seeds.allocate(&rt, B);
        d_tb.allocate(&rt, B);
        d_order.allocate(&rt, B);
        d_next.allocate(&rt, 1);
        d_out.allocate(&rt, B);
        d_active.allocate(&rt, 1);
        AMBER_CUDA(cudaMemcpyAsync(d_seeds.p, seeds.data(), B * 8, cudaMemcpyHostToDevice, rt.stream));
        AMBER_CUDA(cudaMemcpyAsync(d_tb.p, tb.data(), B * 8, cudaMemcpyHostToDevice, rt.stream));
        AMBER_CUDA(cudaMemcpyAsync(d_order.p, order.data(), B * sizeof(int), cudaMemcpyHostToDevice, rt.stream));
        d_next.zero_async(rt.stream);
        d_active.zero_async(rt.stream);
        // max arcs of any replicate in the batch (for the shared-memory column
        // stage), reduced on the device: 4 bytes back instead of the row offsets
        DevBuf<unsigned int> d_max;
        d_max.allocate(&rt, 1);
        d_max.zero_async(rt.stream);
        sweep_max_arcs_kernel<<<static_cast<int>(std::min<int64_t>(ceil_div(B, 256), 1024)), 256, 0, rt.stream>>>(
            g.row_ptr.p, B, n, d_max.p);
        check_launch("sweep_max_arcs_kernel");
        unsigned int h_max = 0;
        AMBER_CUDA(cudaMemcpyAsync(&h_max, d_max.p, 4, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        const int64_t max_arcs = h_max;
        AMBER_CUDA(cudaEventRecord(e1, rt.stream));
        SweepArgs a{};
        a.row_ptr = g.row_ptr.p;
        a.col = g.col.p;
        a.state0 = st0.p;
        a.seeds = d_seeds.p;
        a.t_beta = d_tb.p;
        a.order = d_order.p;
        a.t_gamma = bernoulli_threshold_host(base.gamma);
        a.R = B;
        a.n = n;
        a.n_pad = n_pad;
        a.steps = n_steps;
        a.next = d_next.p;
        a.out = d_out.p;
        a.active_updates = d_active.p;
        int smem_max = 0;
        AMBER_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, rt.device));
        const size_t rp_bytes = ((n + 4) & ~3ll) * 4, st_bytes = 2 * n_pad;
        const size_t col_bytes = ((max_arcs + 7) & ~7ll) * 2;
        const size_t sq_bytes = 32 * 64 * 2 + 16;  // the warps' owner queues (COL_SMEM), 16-byte aligned
        const bool col_smem =
            n <= 65536 && rp_bytes + col_bytes + st_bytes + sq_bytes + 64 <= static_cast<size_t>(smem_max);
        a.col_smem = col_smem;
        a.col_cap = col_smem ? max_arcs : 0;
        size_t smem = rp_bytes + (col_smem ? col_bytes + sq_bytes : 0) + st_bytes;
        AMBER_REQUIRE(smem + 64 <= static_cast<size_t>(smem_max), "sweep: replicate state does not fit shared memory");
        auto kern = col_smem ? sir_sweep_kernel<true> : sir_sweep_kernel<false>;
        AMBER_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int per_sm = 0;
        AMBER_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 1024, smem));
        const int blocks = static_cast<int>(std::min<int64_t>(std::max(per_sm, 1) * rt.num_sms, B));
        if (B > 0) {
            kern<<<blocks, 1024, smem, rt.stream>>>(a);
            check_launch("sir_sweep_kernel");
        }
        AMBER_CUDA(cudaEventRecord(e2, rt.stream));
        AMBER_CUDA(cudaMemcpyAsync(local.data() + b0, d_out.p, B * 8, cudaMemcpyDeviceToHost, rt.stream));
        unsigned long long act = 0;
        AMBER_CUDA(cudaMemcpyAsync(&act, d_active.p, 8, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        float f1 = 0, f2 = 0;
        AMBER_CUDA(cudaEventElapsedTime(&f1, e0, e1));
        AMBER_CUDA(cudaEventElapsedTime(&f2, e1, e2));
        build_ms += f1;
        step_ms += f2;
        active += act;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    std::vector<double> lb_all;
    if (W > 1 && loopback_allgather_f64(r, local, lb_all)) {
        for (int64_t k = 0; k < n_reps; ++k) out[k] = lb_all[k];
    } else if (W > 1) {
        Comm* c = make_comm(r);
        DevBuf<double> d_loc, d_all;
        d_loc.allocate(&rt, per);
        d_all.allocate(&rt, per * W);
        AMBER_CUDA(cudaMemcpyAsync(d_loc.p, local.data(), per * 8, cudaMemcpyHostToDevice, rt.stream));
        comm_allgather_f64(c, rt.stream, d_loc.p, d_all.p, per);
        std::vector<double> all(per * W);
        AMBER_CUDA(cudaMemcpyAsync(all.data(), d_all.p, per * W * 8, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        destroy_comm(c);
        for (int64_t k = 0; k < n_reps; ++k) out[k] = all[k];  // rank g's block starts at g*per
    } else {
        for (int64_t k = 0; k < n_reps; ++k) out[k] = local[k];
    }
    if (stats) {
        stats->build_ms = build_ms;
        stats->step_ms = step_ms;
        stats->agent_updates = n * n_steps * R;
        stats->active_updates = static_cast<int64_t>(active);
    }
}

}  // namespace amber
