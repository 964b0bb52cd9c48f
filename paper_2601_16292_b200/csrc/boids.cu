// boids.cu -- flocking in a periodic 2-D box (BASELINE config 3; continuous
// wrapped space per PAPER.md Sec. 4.1; B1-B8).
//
// Per step (all on the model stream):
//   1. bin     : cell of every agent (uniform grid, cell side >= R with margin)
//                -> per-cell counts (atomics)
//   2. scan    : exclusive scan of the counts -> cell_start (one CTA)
//   3. scatter : counting-sort placement; gathers (x, y, vx, vy) into a
//                cell-sorted float4 array and carries the agent ids along
//   4. step    : one thread per sorted agent scans the 3x3 cell stencil
//                (contiguous ranges of the sorted array, L1-resident), sums
//                neighbour terms in int64 fixed point (exact, so independent
//                of traversal order), applies the rules and writes the next
//                state in sorted order (coalesced).
// The columns therefore live in "current order" with an id array; reads and
// writes of the id-ordered columns go through an un-permute / permute kernel.
// Float contract B7: every float/double op below is an explicit _rn intrinsic
// (no FMA contraction, IEEE division and square root), so the step equals the
// oracle's bit for bit.
#include <cooperative_groups.h>

#include <algorithm>
#include <cub/block/block_reduce.cuh>
#include <cub/cub.cuh>

#include "internal.cuh"
#include "philox.cuh"

namespace amber {

namespace {

constexpr float kFix = 16777216.0f;  // 2^24 (B3)
#ifndef AMBER_BOIDS_INFLIGHT
#define AMBER_BOIDS_INFLIGHT 2  // candidate loads in flight per lane in interior row runs
#endif
#ifndef AMBER_BOIDS_MINB
// resident 256-thread blocks per SM for the stencil kernel: 3 (register cap 80)
// for small populations, 6 (cap 40) for large ones -- V3 stencil 18.3 -> 17.5 ms
// (more warps to hide the candidate loads), C3 slightly slower (60.9 -> 63.9 us).
// r02 C3 A/B (tools/c3_lib_probe.py, same box, alternating runs): 2 / 3 / 4 / 5
// blocks per SM 42.4 / 42.4 / 43.6 / 42.7 us/step.
#define AMBER_BOIDS_MINB 3
#endif
#ifndef AMBER_BOIDS_MINB_LARGE
// r02 V3 A/B (tools/v3_run.py 10, alternating runs): 5 / 6 / 7 / 8 blocks per
// SM 18.11 / 17.93 / 18.25 / 18.24 ms/step (incl. the first step from init)
#define AMBER_BOIDS_MINB_LARGE 6
#endif

struct BoidsArgs {
    float L, R, rs, wc, wa, ws, vmax, dt;
    int nc;       // cells per side (y; and x for the sharded slabs)
    float inv_cs; // nc / L
    int span = 1; // stencil half-width in cells: 1 (cells >= R) or 2 (cells >= R/2)
    // one-GPU grid: rows of nc cells of height cs >= R in y, each split into
    // ncx = sx * nc columns of width cs / sx in x; the stencil of an agent in
    // column hx covers columns hx - sx .. hx + sx of three rows (one contiguous
    // run per row, (2 + 1/sx) cs wide instead of 3 cs)
    int ncx = 0;
    float inv_csx = 0.f;  // ncx / L
    int sx = 1;
    // 0.5 L, R^2, r_s^2 rounded once on the host (float rn, as the device
    // would): constant-bank operands of the candidate loop's compares instead
    // of per-agent products held in registers
    float halfL = 0.f, R2 = 0.f, rs2 = 0.f;
};

inline void boids_derived(BoidsArgs& a)
{
    volatile float L = a.L, R = a.R, rs = a.rs;  // plain IEEE single products
    a.halfL = 0.5f * L;
    a.R2 = R * R;
    a.rs2 = rs * rs;
}

__device__ __forceinline__ int cell_coord(float x, const BoidsArgs& a)
{
    int c = static_cast<int>(__fmul_rn(x, a.inv_cs));
    return c < 0 ? 0 : (c >= a.nc ? a.nc - 1 : c);
}

// x column of the one-GPU grid (width cs / sx)
__device__ __forceinline__ int cell_x(float x, const BoidsArgs& a)
{
    int c = static_cast<int>(__fmul_rn(x, a.inv_csx));
    return c < 0 ? 0 : (c >= a.ncx ? a.ncx - 1 : c);
}

// B1: initial positions and rejection-sampled unit velocities (id order).
__global__ void boids_init_kernel(PhiloxKey key, int64_t n, float L, float4* st, int32_t* ids)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        // R4: 32-bit lanes 2i, 2i+1 of tag BOIDS_POS = words (2i%4, 2i%4+1) of block i/2
        const uint4 w = stream_block(key, TAG_BOIDS_POS, static_cast<unsigned long long>(i) >> 1, 0u);
        const uint32_t ux = (i & 1) ? w.z : w.x, uy = (i & 1) ? w.w : w.y;
        const float x = __fmul_rn(L, u01(ux)), y = __fmul_rn(L, u01(uy));
        float vx = 0.f, vy = 0.f;
        for (uint32_t attempt = 0;; ++attempt) {
            const uint4 v = philox(make_uint4(static_cast<uint32_t>(i), static_cast<uint32_t>(static_cast<unsigned long long>(i) >> 32),
                                              attempt, TAG_BOIDS_VEL),
                                   key);
            const float a = __fsub_rn(__fmul_rn(2.0f, u01(v.x)), 1.0f);
            const float b = __fsub_rn(__fmul_rn(2.0f, u01(v.y)), 1.0f);
            const float s2 = __fadd_rn(__fmul_rn(a, a), __fmul_rn(b, b));
            if (s2 > 0.0f && s2 <= 1.0f) {
                const float s = __fsqrt_rn(s2);
                vx = __fdiv_rn(a, s);
                vy = __fdiv_rn(b, s);
                break;
            }
        }
        st[i] = make_float4(x, y, vx, vy);
        ids[i] = static_cast<int32_t>(i);
    }
}

struct BoidsSlot {
    double mean_speed, polar_x, polar_y;
    unsigned long long digest;
};

// Runs of equal keys in consecutive lanes (key < 0: no item, never merged):
// the lane of the run's head, the lane's rank in its run and the run length.
// The state is in the previous step's cell order, so consecutive agents mostly
// share their new cell: one atomic per run instead of one per agent.  All 32
// lanes call it.
__device__ __forceinline__ void lane_runs(int key, int& head, int& rank, int& len)
{
    const uint32_t lane = threadIdx.x & 31;
    const int prev = __shfl_up_sync(0xffffffffu, key, 1);
    const uint32_t heads = __ballot_sync(0xffffffffu, lane == 0 || key < 0 || prev != key);
    const uint32_t le = 0xffffffffu >> (31 - lane);  // lanes <= this one
    head = 31 - __clz(heads & le);
    rank = static_cast<int>(lane) - head;
    const uint32_t above = heads & ~le;
    len = (above ? __ffs(above) - 1 : 32) - head;
}

__global__ void boids_count_kernel(const float4* __restrict__ st, int64_t n, BoidsArgs a, int* __restrict__ cnt,
                                   int* __restrict__ cell_of, BoidsSlot* slot_zero)
{
    if (slot_zero && blockIdx.x == 0 && threadIdx.x == 0) *slot_zero = BoidsSlot{0.0, 0.0, 0.0, 0ull};  // this step's record
    const int64_t nt = (int64_t)gridDim.x * blockDim.x, rounds = (n + nt - 1) / nt;
    for (int64_t r = 0; r < rounds; ++r) {  // uniform trip count: the lanes cooperate
        const int64_t p = r * nt + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        int c = -1;
        if (p < n) {
            const float4 s = st[p];
            c = cell_coord(s.y, a) * a.ncx + cell_x(s.x, a);
            if (cell_of) cell_of[p] = c;
        }
        int head, rank, len;
        lane_runs(c, head, rank, len);
        if (c >= 0 && rank == 0) atomicAdd(cnt + c, len);
    }
}

// Exclusive scan of the ncell + 1 counts by one CTA (ncell <= 2^16), register
// resident: each thread loads 16 consecutive counts (four 16-byte loads), one
// block scan of the thread sums (warp shuffles + the 32 warp totals), then 16
// starts per thread with 16-byte stores -- one global round trip per 16,384
// cells (r02: replaced a two-pass segment scan, 8.7 -> 6.5 us cold; grids up
// to kScanSmemCells now fold the scan into the scatter, below).
__global__ void __launch_bounds__(1024) boids_scan_reg_kernel(const int* __restrict__ cnt, int* __restrict__ start,
                                                              int* __restrict__ cursor, int ncell)
{
    __shared__ int wsum[32];
    __shared__ int carry_s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    const int total = ncell + 1;  // cnt[ncell] = 0, so start[ncell] = n
    for (int base = 0; base < total; base += 1024 * 16) {
        const int c0 = base + threadIdx.x * 16;
        int v[16];
        const bool full = c0 + 16 <= total;
        if (full) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int4 q = reinterpret_cast<const int4*>(cnt + c0)[k];
                v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = c0 + k < total ? cnt[c0 + k] : 0;
        }
        int sum = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) sum += v[k];
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) wsum[w] = incl;
        __syncthreads();
        if (w == 0) {
            const int x = wsum[lane];
            int xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += u;
            }
            wsum[lane] = xi - x;
        }
        __syncthreads();
        const int carry = carry_s;
        int run = carry + wsum[w] + incl - sum;
        if (full && c0 + 16 <= ncell) {  // 16 real cells: 16-byte stores
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int4 o;
                o.x = run; run += v[4 * k];
                o.y = run; run += v[4 * k + 1];
                o.z = run; run += v[4 * k + 2];
                o.w = run; run += v[4 * k + 3];
                reinterpret_cast<int4*>(start + c0)[k] = o;
                reinterpret_cast<int4*>(cursor + c0)[k] = o;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int c = c0 + k;
                if (c < total) {
                    start[c] = run;
                    if (c < ncell) cursor[c] = run;
                }
                run += v[k];
            }
        }
        __syncthreads();
        if (threadIdx.x == 1023) carry_s = run;  // the pass's running total
        __syncthreads();
    }
}

// Exclusive scan of the ncell + 1 counts for large grids (> 2^16 cells), by
// hand in three launches (no library scan on the step path): (1) each
// 1024-thread block sums a chunk of kScanChunk cells; (1b) one CTA scans the
// chunk totals into offsets; (2) each block scans its chunk from its offset
// (four cells per thread, warp shuffles + one shared-memory pass over the 32
// warp totals), writes start / cursor and re-zeroes the counts.
constexpr int kScanChunk = 4096;

__device__ __forceinline__ int block_sum_1024(int v, int* red)
{
    v = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int t = threadIdx.x < 32 ? red[threadIdx.x] : 0;
    if (threadIdx.x < 32) t = __reduce_add_sync(0xffffffffu, t);
    __syncthreads();
    return t;  // valid in warp 0
}

__global__ void __launch_bounds__(1024) boids_chunk_sums_kernel(const int* __restrict__ cnt, int ncell1,
                                                                int* __restrict__ sums)
{
    __shared__ int red[32];
    const int c0 = blockIdx.x * kScanChunk + threadIdx.x * 4;
    int s = 0;
    if (c0 + 4 <= ncell1) {  // one 16-byte load (cnt is 256-byte aligned, c0 a multiple of 4)
        const int4 v = *reinterpret_cast<const int4*>(cnt + c0);
        s = v.x + v.y + v.z + v.w;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) s += c0 + k < ncell1 ? cnt[c0 + k] : 0;
    }
    s = block_sum_1024(s, red);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
}

// (1b) one CTA turns the chunk totals into exclusive chunk offsets, in place
// (1024 totals per pass: warp shuffles + the 32 warp totals + a running carry)
__global__ void __launch_bounds__(1024) boids_chunk_offsets_kernel(int* __restrict__ sums, int nch)
{
    __shared__ int wex[32];
    __shared__ int carry_s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < nch; base += 1024) {
        const int c = base + threadIdx.x;
        const int v = c < nch ? sums[c] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) wex[w] = incl;
        __syncthreads();
        if (w == 0) {
            const int x = wex[lane];
            int xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += u;
            }
            wex[lane] = xi - x;
        }
        __syncthreads();
        const int carry = carry_s;
        if (c < nch) sums[c] = carry + wex[w] + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry_s = carry + wex[31] + incl;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) boids_chunk_scan_kernel(int* __restrict__ cnt, const int* __restrict__ offs,
                                                                int ncell, int* __restrict__ start,
                                                                int* __restrict__ cursor)
{
    __shared__ int wex[32];
    const int carry = offs[blockIdx.x];
    const int c0 = blockIdx.x * kScanChunk + threadIdx.x * 4;
    int v[4], tsum = 0;
    const bool full = c0 + 4 <= ncell;  // all four cells real (and not the terminal entry)
    if (full) {
        const int4 q = *reinterpret_cast<const int4*>(cnt + c0);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
        tsum = q.x + q.y + q.z + q.w;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = c0 + k <= ncell ? cnt[c0 + k] : 0;
            tsum += v[k];
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wex[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int x = wex[lane];
        int xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += u;
        }
        wex[lane] = xi - x;
    }
    __syncthreads();
    int run = carry + wex[w] + incl - tsum;
    if (full) {  // 16-byte stores
        const int4 o = make_int4(run, run + v[0], run + v[0] + v[1], run + v[0] + v[1] + v[2]);
        *reinterpret_cast<int4*>(start + c0) = o;
        *reinterpret_cast<int4*>(cursor + c0) = o;
        *reinterpret_cast<int4*>(cnt + c0) = make_int4(0, 0, 0, 0);
        return;  // (the terminal entry start[ncell] belongs to a partial quad)
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int c = c0 + k;
        if (c <= ncell) {
            start[c] = run;
            if (c < ncell) {
                cursor[c] = run;
                cnt[c] = 0;
            }
        }
        run += v[k];
    }
}

// Counting-sort scatter; also zeroes the cell counts for the next count pass
// (ncell_zero cells; 0 when the counts were cleared otherwise).
// QV (svel != nullptr): the sorted record carries q24(v) as int32 bits in z, w
// (the stencil's candidates) and svel the float velocity (the agent's own update).
// cell_of == nullptr: the cell is recomputed from the state (which the pass
// reads anyway) instead of read -- 8 B/agent less traffic between the passes.
__global__ void boids_scatter_kernel(const float4* __restrict__ st, const int32_t* __restrict__ ids, int64_t n,
                                     const int* __restrict__ cell_of, int* __restrict__ cursor, float4* __restrict__ sorted,
                                     int32_t* __restrict__ sorted_ids, int* __restrict__ cnt, int ncell_zero,
                                     float2* __restrict__ svel, BoidsArgs a)
{
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = tid; c < ncell_zero; c += nt) cnt[c] = 0;
    const int64_t rounds = (n + nt - 1) / nt;
    for (int64_t r = 0; r < rounds; ++r) {  // uniform trip count: the lanes cooperate
        const int64_t p = r * nt + tid;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        int32_t id = 0;
        int c = -1;
        if (p < n) {
            v = st[p];
            id = ids[p];  // issued with the record, not after the cursor claim
            c = cell_of ? cell_of[p] : cell_coord(v.y, a) * a.ncx + cell_x(v.x, a);
        }
        int head, rank, len;
        lane_runs(c, head, rank, len);
        int q = 0;
        if (c >= 0 && rank == 0) q = atomicAdd(cursor + c, len);  // one cursor claim per run
        q = __shfl_sync(0xffffffffu, q, head) + rank;
        if (c >= 0) {
            AMBER_DCHECK(q >= 0 && q < n, "Boids scatter: sorted slot out of range");
            if (svel) {
                sorted[q] = make_float4(v.x, v.y, __int_as_float(__float2int_rn(__fmul_rn(v.z, kFix))),
                                        __int_as_float(__float2int_rn(__fmul_rn(v.w, kFix))));
                svel[q] = make_float2(v.z, v.w);
            } else {
                sorted[q] = v;
            }
            sorted_ids[q] = id;
        }
    }
}

// Small grids (<= kScanSmemCells cells): the cell scan folded into the scatter
// pass.  Every block (1024 threads, one per SM) scans the whole count array
// itself -- 16 counts per thread by 16-byte loads, one block scan, the starts
// kept in shared memory -- instead of a one-CTA scan launch before the scatter
// (C3: 10^4 cells, a 40 KB read per block from L2); block 0 also writes the
// global starts the stencil reads.  Counts and placement counters are
// double-buffered by step parity (row stride cs, a multiple of 16, padding
// zero): this pass reads cnt and claims slots in fill (zero), and zeroes the
// other parity's cnt (counted by the next stencil) and fill (the next step's
// placement).
constexpr int kScanSmemCells = 12000;  // ss: 48 KB static shared memory

__global__ void __launch_bounds__(1024) boids_scatter_scan_kernel(
    const float4* __restrict__ st, const int32_t* __restrict__ ids, int64_t n, const int* __restrict__ cnt,
    int* __restrict__ cnt_zero, int* __restrict__ fill, int* __restrict__ fill_zero, int ncell, int cs,
    int* __restrict__ start, float4* __restrict__ sorted, int32_t* __restrict__ sorted_ids,
    float2* __restrict__ svel, BoidsArgs a)
{
    __shared__ __align__(16) int ss[(kScanSmemCells + 16) & ~15];
    __shared__ int wsum[32];
    pdl_wait();  // launched with launch_pdl: the previous step's stencil must be complete
    pdl_trigger();
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int total = ncell + 1;  // cnt[ncell] = 0, so start[ncell] = n
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + tid, nt = (int64_t)gridDim.x * blockDim.x;
    // the first round's agent loads are issued before the scan (C3: one round)
    float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f);
    int32_t id0 = 0;
    if (gt < n) {
        x0 = st[gt];
        id0 = ids[gt];
    }
    const int c0 = tid * 16;
    int v[16];
    if (c0 < total) {  // cs >= c0 + 16: the padded row
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int4 q = __ldcg(reinterpret_cast<const int4*>(cnt + c0) + k);
            v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = 0;
    }
    int sum = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) sum += v[k];
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int x = wsum[lane];
        int xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += u;
        }
        wsum[lane] = xi - x;
    }
    __syncthreads();
    if (c0 < total) {
        int run = wsum[w] + incl - sum;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            int4 o;
            o.x = run; run += v[4 * k];
            o.y = run; run += v[4 * k + 1];
            o.z = run; run += v[4 * k + 2];
            o.w = run; run += v[4 * k + 3];
            reinterpret_cast<int4*>(ss + c0)[k] = o;  // c0 + 16 <= 12016
            if (blockIdx.x == 0) {
                if (c0 + 4 * k + 4 <= total) {
                    reinterpret_cast<int4*>(start + c0)[k] = o;
                } else {
                    const int e[4] = {o.x, o.y, o.z, o.w};
                    for (int j = 0; j < 4 && c0 + 4 * k + j < total; ++j) start[c0 + 4 * k + j] = e[j];
                }
            }
        }
    }
    for (int64_t c = gt; c < cs / 4; c += nt) {
        reinterpret_cast<int4*>(cnt_zero)[c] = make_int4(0, 0, 0, 0);
        reinterpret_cast<int4*>(fill_zero)[c] = make_int4(0, 0, 0, 0);
    }
    __syncthreads();
    const int64_t rounds = (n + nt - 1) / nt;
    for (int64_t r = 0; r < rounds; ++r) {  // uniform trip count: the lanes cooperate
        const int64_t p = r * nt + gt;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        int c = -1;
        if (p < n) {
            x = r == 0 ? x0 : st[p];
            c = cell_coord(x.y, a) * a.ncx + cell_x(x.x, a);
        }
        int head, rank, len;
        lane_runs(c, head, rank, len);
        int q = 0;
        if (c >= 0 && rank == 0) q = ss[c] + atomicAdd(fill + c, len);  // one slot claim per run
        q = __shfl_sync(0xffffffffu, q, head) + rank;
        if (c >= 0) {
            AMBER_DCHECK(q >= 0 && q < n, "Boids scatter: sorted slot out of range");
            if (svel) {
                sorted[q] = make_float4(x.x, x.y, __int_as_float(__float2int_rn(__fmul_rn(x.z, kFix))),
                                        __int_as_float(__float2int_rn(__fmul_rn(x.w, kFix))));
                svel[q] = make_float2(x.z, x.w);
            } else {
                sorted[q] = x;
            }
            sorted_ids[q] = r == 0 ? id0 : ids[p];
        }
    }
}

struct Acc {
    long long n, sdx, sdy, svx, svy, ssx, ssy;
};

__device__ __forceinline__ long long q24(float f) { return __float2ll_rn(__fmul_rn(f, kFix)); }

__device__ __forceinline__ float min_image(float d, float L, float halfL)
{
    if (d > halfL) return __fsub_rn(d, L);
    if (d < -halfL) return __fadd_rn(d, L);
    return d;
}


// WRAP = false: the caller guarantees |o - me| <= L/2 per coordinate (both
// agents in interior cells), where the minimum image is the identity.
// QV: the candidate record carries its velocity pre-quantised (o.z, o.w hold
// q24(v) as int32 bits, written once per agent by the scatter pass), and the
// displacement converts with a 32-bit F2I: |dx| <= R < 100 so |q24(dx)| < 2^31.
// Same integers as the float path (B3), two F2I.S64 fewer per neighbour
// (tools/alu_ceiling.cu: the stencil's ALU ceiling 7.9e11 -> 9.3e11 candidate
// visits/s, profiles/r02_alu_ceiling.txt).
template <bool WRAP = true, bool QV = false>
__device__ __forceinline__ void boid_accumulate(const float4 o, const float4 me, float L, float halfL, float R2,
                                                float rs2, Acc& acc)
{
    float dx = __fsub_rn(o.x, me.x), dy = __fsub_rn(o.y, me.y);
    if constexpr (WRAP) {
        const float dxm = __fsub_rn(dx, L), dxp = __fadd_rn(dx, L), dym = __fsub_rn(dy, L), dyp = __fadd_rn(dy, L);
        dx = dx > halfL ? dxm : (dx < -halfL ? dxp : dx);
        dy = dy > halfL ? dym : (dy < -halfL ? dyp : dy);
    }
    const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
    if (d2 <= R2) {
        if constexpr (QV) {
            const int qx = __float2int_rn(__fmul_rn(dx, kFix)), qy = __float2int_rn(__fmul_rn(dy, kFix));
            acc.n += 1;
            acc.sdx += qx;
            acc.sdy += qy;
            acc.svx += __float_as_int(o.z);
            acc.svy += __float_as_int(o.w);
            if (d2 <= rs2) {
                acc.ssx += qx;
                acc.ssy += qy;
            }
        } else {
            const long long qx = q24(dx), qy = q24(dy);
            acc.n += 1;
            acc.sdx += qx;
            acc.sdy += qy;
            acc.svx += q24(o.z);
            acc.svy += q24(o.w);
            if (d2 <= rs2) {
                acc.ssx += qx;
                acc.ssy += qy;
            }
        }
    }
}

// B8 per-agent terms (speed, unit velocity) summed in double.  The terms are
// float32 from one approximate reciprocal square root (MUFU, ~2 ulp): their
// error (< 3e-7 relative) is four orders below the B8 tolerances (mean speed
// 1e-3 relative, polarisation 1e-3 absolute), and one lane's eight
// instructions replace three lanes' double sqrt + division sequences (r02 ncu:
// 7.6% of the V3 stencil's instructions).
__device__ __forceinline__ void boid_observe(float vx, float vy, double& sp, double& ux, double& uy)
{
    const float s2 = __fadd_rn(__fmul_rn(vx, vx), __fmul_rn(vy, vy));
    if (s2 > 0.0f) {
        const float r = rsqrtf(s2);
        sp += static_cast<double>(__fmul_rn(s2, r));
        ux += static_cast<double>(__fmul_rn(vx, r));
        uy += static_cast<double>(__fmul_rn(vy, r));
    }
}

// B4-B6 given the four neighbour means (computed by the caller) and the sums.
__device__ __forceinline__ float4 boid_update_means(const float4 me, const Acc& acc, float cohx, float cohy, float avx,
                                                    float avy, const BoidsArgs& a)
{
    const float L = a.L;
    float ux = me.z, uy = me.w;
    if (acc.n > 0) {
        const float sepx = __double2float_rn(__dmul_rn(static_cast<double>(acc.ssx), 1.0 / 16777216.0));
        const float sepy = __double2float_rn(__dmul_rn(static_cast<double>(acc.ssy), 1.0 / 16777216.0));
        ux = __fsub_rn(__fadd_rn(__fadd_rn(me.z, __fmul_rn(a.wc, cohx)), __fmul_rn(a.wa, __fsub_rn(avx, me.z))),
                       __fmul_rn(a.ws, sepx));
        uy = __fsub_rn(__fadd_rn(__fadd_rn(me.w, __fmul_rn(a.wc, cohy)), __fmul_rn(a.wa, __fsub_rn(avy, me.w))),
                       __fmul_rn(a.ws, sepy));
    }
    const float s2 = __fadd_rn(__fmul_rn(ux, ux), __fmul_rn(uy, uy));
    if (s2 > __fmul_rn(a.vmax, a.vmax)) {
        const float f = __fdiv_rn(a.vmax, __fsqrt_rn(s2));
        ux = __fmul_rn(ux, f);
        uy = __fmul_rn(uy, f);
    }
    float x = __fadd_rn(me.x, __fmul_rn(ux, a.dt));
    float y = __fadd_rn(me.y, __fmul_rn(uy, a.dt));
    if (x < 0.0f) x = __fadd_rn(x, L);
    if (x >= L) x = __fsub_rn(x, L);
    if (y < 0.0f) y = __fadd_rn(y, L);
    if (y >= L) y = __fsub_rn(y, L);
    return make_float4(x, y, ux, uy);
}

// ---------------------------------------------------------------- grouped step
// G lanes per agent: the lanes of a group stride over the candidates of the
// agent's 3x3 stencil (cell runs of the sorted array, L1-resident), then the
// seven int64 fixed-point sums are combined with xor-shuffles inside the group
// (exact integer adds, so the result equals the one-lane definition bit for
// bit).  G times more threads than agents hide the L1 latency of the candidate
// loop that bounds the one-lane kernel once flocks cluster (r01 ncu: 15K
// instructions per agent at step 90, 30% warp occupancy).
template <int G, bool QV>
__device__ __forceinline__ void boids_group_body(const float4* __restrict__ sorted, const int32_t* __restrict__ sids,
                                                 const int* __restrict__ start, int64_t n, const BoidsArgs& a,
                                                 float4* __restrict__ out, int32_t* __restrict__ out_ids, BoidsSlot* slot,
                                                 int digest, int* __restrict__ next_cnt,
                                                 int* __restrict__ next_cell, const float2* __restrict__ svel)
{
    static_assert(G >= 4, "the update spreads four divisions over the group's lanes");
    const float L = a.L, halfL = a.halfL, R2 = a.R2, rs2 = a.rs2;
    const int sub = threadIdx.x & (G - 1);
    // each block owns one contiguous range of the cell-sorted agents (blockDim/G
    // agents per round): consecutive rounds slide along the same cell rows, so
    // the stencil's rows stay in this SM's L1 instead of being fetched by a
    // different SM every round
    // (large populations only: at C3's 1e5 agents -- two rounds per block -- the
    // grid-strided order measured faster, 54 vs 58 us; dealing the warps' chunks
    // to the blocks round-robin, so each block samples the whole box, 57 vs 44 us
    // in r02: the block's warps share L1 lines only when they are neighbours)
    const int64_t apb = blockDim.x / G;  // agents per block per round
    const int64_t ng = apb * gridDim.x;
    const int64_t rounds = (n + ng - 1) / ng;  // uniform: every lane runs every round (shuffles)
    const bool contig = n > (1ll << 22);
    const int64_t base = contig ? static_cast<int64_t>(blockIdx.x) * rounds * apb + threadIdx.x / G
                                : static_cast<int64_t>(blockIdx.x) * apb + threadIdx.x / G;
    const int64_t rstride = contig ? apb : ng;
    double sp_sum = 0.0, ux_sum = 0.0, uy_sum = 0.0;
    unsigned long long dig = 0;
    for (int64_t r = 0; r < rounds; ++r) {
        const int64_t p = base + r * rstride;
        const bool active = p < n;
        Acc acc{0, 0, 0, 0, 0, 0, 0};
        float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
        int qself_x = 0, qself_y = 0;  // QV: the agent's own quantised velocity
        if (active) {
            me = sorted[p];
            if constexpr (QV) {
                qself_x = __float_as_int(me.z);
                qself_y = __float_as_int(me.w);
                const float2 v = svel[p];
                me.z = v.x;
                me.w = v.y;
            }
            auto run = [&](int b, int e) {
                AMBER_DCHECK(b >= 0 && b <= e && e <= n, "Boids stencil: cell run out of range");
                for (int q = b + sub; q < e; q += G)
                    boid_accumulate<true, QV>(sorted[q], me, L, halfL, R2, rs2, acc);
            };
            // interior agents (stencil inside the box, so every candidate is within
            // two cells < L/2 per coordinate): no minimum image, rows as runs
            auto run_in = [&](int b, int e) {
                AMBER_DCHECK(b >= 0 && b <= e && e <= n, "Boids stencil: cell run out of range");
                int q = b + sub;
#if AMBER_BOIDS_INFLIGHT == 4
                for (; q + 3 * G < e; q += 4 * G) {  // four candidate loads in flight per lane
                    const float4 o0 = sorted[q], o1 = sorted[q + G], o2 = sorted[q + 2 * G], o3 = sorted[q + 3 * G];
                    boid_accumulate<false, QV>(o0, me, L, halfL, R2, rs2, acc);
                    boid_accumulate<false, QV>(o1, me, L, halfL, R2, rs2, acc);
                    boid_accumulate<false, QV>(o2, me, L, halfL, R2, rs2, acc);
                    boid_accumulate<false, QV>(o3, me, L, halfL, R2, rs2, acc);
                }
#endif
                for (; q + G < e; q += 2 * G) {  // two candidate loads in flight per lane
                    const float4 o0 = sorted[q], o1 = sorted[q + G];
                    boid_accumulate<false, QV>(o0, me, L, halfL, R2, rs2, acc);
                    boid_accumulate<false, QV>(o1, me, L, halfL, R2, rs2, acc);
                }
                if (q < e) boid_accumulate<false, QV>(sorted[q], me, L, halfL, R2, rs2, acc);
            };
            const int sx = a.sx, ncx = a.ncx;
            const int cx0 = a.nc >= 3 ? cell_x(me.x, a) : 0, cy0 = a.nc >= 3 ? cell_coord(me.y, a) : 0;
            // interior: the whole stencil inside the box and within 2 cells < L/2 (nc >= 5)
            if (a.nc >= 5 && cx0 >= sx && cx0 + sx < ncx && cy0 >= 1 && cy0 + 1 < a.nc) {
#pragma unroll 1
                for (int dyc = -1; dyc <= 1; ++dyc) {
                    const int row = (cy0 + dyc) * ncx;
                    run_in(start[row + cx0 - sx], start[row + cx0 + sx + 1]);
                }
            } else if (a.nc >= 3) {
                const int cx = cx0, cy = cy0;
#pragma unroll 1
                for (int dyc = -1; dyc <= 1; ++dyc) {
                    int yy = cy + dyc;
                    yy = yy < 0 ? yy + a.nc : (yy >= a.nc ? yy - a.nc : yy);
                    const int row = yy * ncx;
                    if (cx >= sx && cx + sx < ncx) {
                        // columns cx-sx .. cx+sx of a row are contiguous in the sorted array
                        run(start[row + cx - sx], start[row + cx + sx + 1]);
                    } else {
#pragma unroll 1
                        for (int dxc = -sx; dxc <= sx; ++dxc) {
                            int xx = cx + dxc;
                            xx = xx < 0 ? xx + ncx : (xx >= ncx ? xx - ncx : xx);
                            run(start[row + xx], start[row + xx + 1]);
                        }
                    }
                }
            } else {
                run(start[0], start[1]);  // one cell holding every agent
            }
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
        if (active) {  // the agent itself was accumulated once (d = 0, inside both radii): take it out
            acc.n -= 1;
            acc.svx -= QV ? static_cast<long long>(qself_x) : q24(me.z);
            acc.svy -= QV ? static_cast<long long>(qself_y) : q24(me.w);
        }
        // B4's four mean divisions in parallel on lanes 0..3 of the group
        // (x / 2^24 is exact, so it is a multiplication), gathered by shuffles
        float mv = 0.0f;
        if (acc.n > 0 && sub < 4) {
            const long long sv = sub == 0 ? acc.sdx : (sub == 1 ? acc.sdy : (sub == 2 ? acc.svx : acc.svy));
            mv = __double2float_rn(__ddiv_rn(__dmul_rn(static_cast<double>(sv), 1.0 / 16777216.0),
                                             static_cast<double>(acc.n)));
        }
        const float cohx = __shfl_sync(0xffffffffu, mv, 0, G), cohy = __shfl_sync(0xffffffffu, mv, 1, G);
        const float avx = __shfl_sync(0xffffffffu, mv, 2, G), avy = __shfl_sync(0xffffffffu, mv, 3, G);
        int ncell_of = -1;  // the agent's cell in the next step's binning (next_cnt)
        if (active) {
            const float4 nx = boid_update_means(me, acc, cohx, cohy, avx, avy, a);
            if (sub == 0) {
                out[p] = nx;
                const int32_t id = sids[p];
                out_ids[p] = id;
                if (digest) dig += digest_term(static_cast<unsigned long long>(id), __float_as_uint(nx.x));
                if (next_cnt) {
                    ncell_of = cell_coord(nx.y, a) * a.ncx + cell_x(nx.x, a);
                    if (next_cell) next_cell[p] = ncell_of;
                }
            }
            if (sub == 0) boid_observe(nx.z, nx.w, sp_sum, ux_sum, uy_sum);
        }
        if (next_cnt) {
            // the next step's cell counts (fused count pass): the warp's agents
            // (lanes 0, G, 2G, ...) are consecutive in cell order and mostly stay
            // in their cell, so a run of equal cells is one atomic by its head
            const int lane = threadIdx.x & 31;
            const int prev = __shfl_up_sync(0xffffffffu, ncell_of, G);
            int run = 1;
            bool more = true;
#pragma unroll
            for (int k = 1; k < 32 / G; ++k) {
                const int nx = __shfl_down_sync(0xffffffffu, ncell_of, k * G);
                more = more && lane + k * G < 32 && nx == ncell_of;
                run += more ? 1 : 0;
            }
            if (ncell_of >= 0 && (lane < G || prev != ncell_of)) atomicAdd(next_cnt + ncell_of, run);
        }
    }
    __shared__ double red[3][8];
    __shared__ unsigned long long dred[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    sp_sum = warp_sum_f64(sp_sum);
    ux_sum = warp_sum_f64(ux_sum);
    uy_sum = warp_sum_f64(uy_sum);
    dig = warp_sum_u64(dig);
    if (lane == 0) {
        red[0][wid] = sp_sum;
        red[1][wid] = ux_sum;
        red[2][wid] = uy_sum;
        dred[wid] = dig;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0, s1 = 0, s2v = 0;
        unsigned long long d = 0;
        for (int w = 0; w < nw; ++w) {
            s0 += red[0][w];
            s1 += red[1][w];
            s2v += red[2][w];
            d += dred[w];
        }
        atomicAdd(&slot->mean_speed, s0);
        atomicAdd(&slot->polar_x, s1);
        atomicAdd(&slot->polar_y, s2v);
        if (digest) atomicAdd(&slot->digest, d);
    }
    __syncthreads();
}

template <int G, bool QV, int MINB = AMBER_BOIDS_MINB>
__global__ void __launch_bounds__(256, MINB) boids_group_kernel(const float4* __restrict__ sorted, const int32_t* __restrict__ sids,
                                                          const int* __restrict__ start, int64_t n, BoidsArgs a,
                                                          float4* __restrict__ out, int32_t* __restrict__ out_ids,
                                                          BoidsSlot* slot, int digest, int* __restrict__ next_cnt,
                                                          int* __restrict__ next_cell, const float2* __restrict__ svel)
{
    pdl_wait();  // launched with launch_pdl: the binning pass must be complete
    pdl_trigger();
    boids_group_body<G, QV>(sorted, sids, start, n, a, out, out_ids, slot, digest, next_cnt, next_cell, svel);
}

// Candidate visits of one stencil pass over the current binning (the 3x3 cell
// neighbourhood's agent count, summed over the agents; the roofline's unit of
// work): sum over cells c of count(c) * sum of the counts of c's 3x3 stencil.
__global__ void boids_candidates_kernel(const int* __restrict__ start, int nc, int ncx, int sx,
                                        unsigned long long* out)
{
    unsigned long long s = 0;
    const int64_t ncell = static_cast<int64_t>(nc) * ncx;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell; c += (int64_t)gridDim.x * blockDim.x) {
        const int cx = static_cast<int>(c % ncx), cy = static_cast<int>(c / ncx);
        const long long own = start[c + 1] - start[c];
        if (!own) continue;
        long long nb = 0;
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -sx; dx <= sx; ++dx) {
                const int x = (cx + dx + ncx) % ncx, y = (cy + dy + nc) % nc;
                const int64_t k = static_cast<int64_t>(y) * ncx + x;
                nb += start[k + 1] - start[k];
            }
        s += static_cast<unsigned long long>(own * nb);
    }
    if (s) atomicAdd(out, s);
}

// 1 in *big if any |velocity| >= 127 or is not finite (the QV stencil's int32 range)
__global__ void boids_big_velocity_kernel(const float4* __restrict__ st, int64_t n, unsigned int* big)
{
    bool b = false;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const float4 s = st[p];
        b |= !(fabsf(s.z) < 127.0f) || !(fabsf(s.w) < 127.0f);
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(big, 1u);
}

// Un-permute: column k of the state (0 x, 1 y, 2 vx, 3 vy) into id order.
__global__ void boids_gather_column(const float4* __restrict__ st, const int32_t* __restrict__ ids, int64_t n, int k,
                                    float* __restrict__ out)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const float4 s = st[p];
        out[ids[p]] = k == 0 ? s.x : (k == 1 ? s.y : (k == 2 ? s.z : s.w));
    }
}

__global__ void boids_put_column(float4* __restrict__ st, const int32_t* __restrict__ ids, int64_t n, int k,
                                 const float* __restrict__ in)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const float v = in[ids[p]];
        float4 s = st[p];
        if (k == 0) s.x = v;
        else if (k == 1) s.y = v;
        else if (k == 2) s.z = v;
        else s.w = v;
        st[p] = s;
    }
}

__global__ void boids_zero_slots(BoidsSlot* ring, int64_t cap, int64_t s0, int64_t count)
{
    for (int64_t k = threadIdx.x; k < count && k < cap; k += blockDim.x) ring[(s0 + k) % cap] = BoidsSlot{0.0, 0.0, 0.0, 0ull};
}


// ---------------------------------------------------------------- sharded Boids (NEXT-3)
// x-slabs of whole cell columns: rank r owns columns [col0[r], col0[r+1]).  An
// agent belongs to the rank whose slab holds its cell column (same cell_coord
// as the binning, so ownership and stencil always agree).  Per step: migrate
// agents whose column left the slab, send the first / last own column to the
// left / right neighbour as halos, bin own + halo agents on a local
// column-major grid of (w + 2) x nc cells (halo columns 0 and w + 1), and step
// the own agents (a contiguous range of the sorted array).  Sums are exact
// fixed point, so the result equals the unsharded step bit for bit.
struct __align__(16) BoidAgent {
    float4 s;
    int32_t id;
    int32_t role;  // halo: 0 = left halo column of the receiver, 1 = right
    int32_t pad0, pad1;
};

struct SlabArgs {
    BoidsArgs a;
    const int* col0;  // [world + 1] first cell column of each slab
    int world, me, c_lo, c_hi;  // my slab [c_lo, c_hi)
    uint64_t cap;               // send block capacity (agents per destination)
};

__device__ __forceinline__ int slab_of(int cx, const SlabArgs& g)
{
    int lo = 0, hi = g.world - 1;  // largest r with col0[r] <= cx
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (g.col0[mid] <= cx) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Warp-aggregated append to the send block of destination d.
__device__ __forceinline__ void slab_send(BoidAgent* send, uint32_t* counts, uint64_t cap, int d, const BoidAgent& v)
{
    const unsigned peers = __match_any_sync(__activemask(), d);
    const int leader = __ffs(peers) - 1;
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counts + d, static_cast<uint32_t>(__popc(peers)));
    base = __shfl_sync(peers, base, leader);
    const uint32_t pos = base + __popc(peers & ((1u << lane) - 1u));
    if (pos < cap) send[static_cast<uint64_t>(d) * cap + pos] = v;
}

// Migration: own agents whose cell column left the slab go to the owner.
// Kept agents are compacted with one cursor atomic per 256-agent block tile
// (per-agent, then per-warp returning atomics on the one counter serialised:
// r02 ncu at G = 8, 2.5e6 agents per rank, 70% of the stall samples on it).
__global__ void __launch_bounds__(256) slab_route_kernel(const float4* __restrict__ st, const int32_t* __restrict__ ids,
                                                         int64_t n_own, SlabArgs g, float4* __restrict__ keep,
                                                         int32_t* __restrict__ keep_ids, uint32_t* keep_n,
                                                         BoidAgent* send, uint32_t* counts)
{
    __shared__ uint32_t wcnt[8], tbase;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x; t0 < n_own;
         t0 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t p = t0 + threadIdx.x;
        const bool in = p < n_own;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        int d = g.me;
        if (in) {
            x = st[p];
            const int cx = cell_coord(x.x, g.a);
            // the own slab first: most agents stay (slab_of searches the column table)
            d = cx >= g.c_lo && cx < g.c_hi ? g.me : slab_of(cx, g);
        }
        const bool kept = in && d == g.me;
        const unsigned km = __ballot_sync(0xffffffffu, kept);
        if (lane == 0) wcnt[wid] = __popc(km);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
                const uint32_t c = wcnt[w];
                wcnt[w] = tot;
                tot += c;
            }
            tbase = tot ? atomicAdd(keep_n, tot) : 0u;
        }
        __syncthreads();
        if (kept) {
            const uint32_t q = tbase + wcnt[wid] + __popc(km & ((1u << lane) - 1u));
            keep[q] = x;
            keep_ids[q] = ids[p];
        } else if (in) {
            slab_send(send, counts, g.cap, d, BoidAgent{x, ids[p], 0, 0, 0});
        }
        __syncthreads();  // wcnt / tbase are rewritten by the next tile
    }
}

__global__ void slab_unpack_kernel(const BoidAgent* __restrict__ in, uint64_t cnt, float4* __restrict__ st,
                                   int32_t* __restrict__ ids, uint64_t off)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < static_cast<int64_t>(cnt);
         k += (int64_t)gridDim.x * blockDim.x) {
        st[off + k] = in[k].s;
        ids[off + k] = in[k].id;
    }
}

// Halos: the first own column goes to the left neighbour (its right halo), the
// last to the right neighbour (its left halo); a one-column slab sends both.
__global__ void slab_halo_kernel(const float4* __restrict__ st, const int32_t* __restrict__ ids, int64_t n_own,
                                 SlabArgs g, BoidAgent* send, uint32_t* counts)
{
    const int left = (g.me + g.world - 1) % g.world, right = (g.me + 1) % g.world;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_own; p += (int64_t)gridDim.x * blockDim.x) {
        const float4 x = st[p];
        const int cx = cell_coord(x.x, g.a);
        if (cx == g.c_lo) slab_send(send, counts, g.cap, left, BoidAgent{x, ids[p], 1, 0, 0});
        if (cx == g.c_hi - 1) slab_send(send, counts, g.cap, right, BoidAgent{x, ids[p], 0, 0, 0});
    }
}

// Local column-major cell of an own agent (local column 1..w) or a halo agent (0 / w + 1).
// The slab grid is column-major with each cell column split into sub-rows of
// height cs / sy in y (BoidsArgs sx / ncx / inv_csx carry sy / ny / ny / L here,
// cell_x of the y coordinate): a stencil run spans (2 + 1 / sy) cs in y
// instead of 3 cs -- the y counterpart of the one-GPU grid's x-subdivision.
__device__ __forceinline__ int slab_cell(float4 x, int lcol, const BoidsArgs& a)
{
    return lcol * a.ncx + cell_x(x.y, a);
}

__global__ void slab_count_kernel(const float4* __restrict__ st, int64_t n_own, const BoidAgent* __restrict__ halo,
                                  int64_t n_halo, SlabArgs g, int* __restrict__ cnt, int* __restrict__ cell_of)
{
    const int w = g.c_hi - g.c_lo;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_own + n_halo;
         p += (int64_t)gridDim.x * blockDim.x) {
        int c;
        if (p < n_own) {
            const float4 x = st[p];
            c = slab_cell(x, cell_coord(x.x, g.a) - g.c_lo + 1, g.a);
        } else {
            const BoidAgent h = halo[p - n_own];
            c = slab_cell(h.s, h.role ? w + 1 : 0, g.a);
        }
        cell_of[p] = c;
        atomicAdd(cnt + c, 1);
    }
}

__global__ void slab_scatter_kernel(const float4* __restrict__ st, const int32_t* __restrict__ ids, int64_t n_own,
                                    const BoidAgent* __restrict__ halo, int64_t n_halo, const int* __restrict__ cell_of,
                                    int* __restrict__ cursor, float4* __restrict__ sorted, int32_t* __restrict__ sids)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_own + n_halo;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int q = atomicAdd(cursor + cell_of[p], 1);
        if (p < n_own) {
            sorted[q] = st[p];
            sids[q] = ids[p];
        } else {
            sorted[q] = halo[p - n_own].s;
            sids[q] = halo[p - n_own].id;
        }
    }
}

// The step for the own agents sorted[own0, own1): G lanes per agent over the
// 3 x 3 stencil of the local grid (three column runs of three cells; y wraps),
// minimum image in both coordinates (halos may come across the periodic x edge).
template <int G>
__global__ void __launch_bounds__(256, 4) slab_step_kernel(const float4* __restrict__ sorted, const int32_t* __restrict__ sids,
                                                           const int* __restrict__ start, int64_t own0, int64_t own1,
                                                           SlabArgs g, float4* __restrict__ out,
                                                           int32_t* __restrict__ out_ids, BoidsSlot* slot, int digest)
{
    const BoidsArgs& a = g.a;
    const float L = a.L, halfL = a.halfL, R2 = a.R2, rs2 = a.rs2;
    const int sub = threadIdx.x & (G - 1);
    const int64_t gid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    const int64_t ng = (static_cast<int64_t>(gridDim.x) * blockDim.x) / G;
    const int64_t n = own1 - own0;
    const int64_t rounds = (n + ng - 1) / ng;
    double sp_sum = 0.0, ux_sum = 0.0, uy_sum = 0.0;
    unsigned long long dig = 0;
    for (int64_t r = 0; r < rounds; ++r) {
        const int64_t k = r * ng + gid;
        const int64_t p = own0 + k;
        const bool active = k < n;
        Acc acc{0, 0, 0, 0, 0, 0, 0};
        float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
        if (active) {
            me = sorted[p];
            auto run = [&](int b, int e) {
                for (int q = b + sub; q < e; q += G) boid_accumulate<true>(sorted[q], me, L, halfL, R2, rs2, acc);
            };
            // no minimum image where no candidate can lie across a periodic edge
            // (as in the one-GPU stencil's interior path, with two candidate
            // loads in flight): rows away from the y edges, and columns whose
            // stencil does not reach a halo taken across the x edge
            auto run_in = [&](int b, int e) {
                int q = b + sub;
                for (; q + G < e; q += 2 * G) {
                    const float4 o0 = sorted[q], o1 = sorted[q + G];
                    boid_accumulate<false>(o0, me, L, halfL, R2, rs2, acc);
                    boid_accumulate<false>(o1, me, L, halfL, R2, rs2, acc);
                }
                if (q < e) boid_accumulate<false>(sorted[q], me, L, halfL, R2, rs2, acc);
            };
            const int lc = cell_coord(me.x, a) - g.c_lo + 1;
            const int sy = a.sx, ny = a.ncx, hy = cell_x(me.y, a);  // y sub-row (slab_cell)
            const int w = g.c_hi - g.c_lo;
            const bool xwrap = (g.c_lo == 0 && lc <= 1) || (g.c_hi == a.nc && lc >= w);
            const bool yin = hy >= sy && hy + sy < ny;
            const bool inner = a.nc >= 5 && !xwrap && yin;
#pragma unroll 1
            for (int dc = -1; dc <= 1; ++dc) {
                const int colb = (lc + dc) * ny;
                if (inner) {
                    run_in(start[colb + hy - sy], start[colb + hy + sy + 1]);
                } else if (yin) {
                    run(start[colb + hy - sy], start[colb + hy + sy + 1]);
                } else {
#pragma unroll 1
                    for (int dy = -sy; dy <= sy; ++dy) {
                        int yy = hy + dy;
                        yy = yy < 0 ? yy + ny : (yy >= ny ? yy - ny : yy);
                        run(start[colb + yy], start[colb + yy + 1]);
                    }
                }
            }
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
        if (active) {  // the agent itself was accumulated once: take it out
            acc.n -= 1;
            acc.svx -= q24(me.z);
            acc.svy -= q24(me.w);
        }
        float mv = 0.0f;
        if (acc.n > 0 && sub < 4) {
            const long long sv = sub == 0 ? acc.sdx : (sub == 1 ? acc.sdy : (sub == 2 ? acc.svx : acc.svy));
            mv = __double2float_rn(__ddiv_rn(__dmul_rn(static_cast<double>(sv), 1.0 / 16777216.0),
                                             static_cast<double>(acc.n)));
        }
        const float cohx = __shfl_sync(0xffffffffu, mv, 0, G), cohy = __shfl_sync(0xffffffffu, mv, 1, G);
        const float avx = __shfl_sync(0xffffffffu, mv, 2, G), avy = __shfl_sync(0xffffffffu, mv, 3, G);
        if (active) {
            const float4 nx = boid_update_means(me, acc, cohx, cohy, avx, avy, a);
            if (sub == 0) {
                out[k] = nx;
                const int32_t id = sids[p];
                out_ids[k] = id;
                if (digest) dig += digest_term(static_cast<unsigned long long>(id), __float_as_uint(nx.x));
            }
            if (sub == 0) boid_observe(nx.z, nx.w, sp_sum, ux_sum, uy_sum);
        }
    }
    __shared__ double red[3][8];
    __shared__ unsigned long long dred[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    sp_sum = warp_sum_f64(sp_sum);
    ux_sum = warp_sum_f64(ux_sum);
    uy_sum = warp_sum_f64(uy_sum);
    dig = warp_sum_u64(dig);
    if (lane == 0) {
        red[0][wid] = sp_sum;
        red[1][wid] = ux_sum;
        red[2][wid] = uy_sum;
        dred[wid] = dig;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0, s1 = 0, s2v = 0;
        unsigned long long d = 0;
        for (int w = 0; w < nw; ++w) {
            s0 += red[0][w];
            s1 += red[1][w];
            s2v += red[2][w];
            d += dred[w];
        }
        atomicAdd(&slot->mean_speed, s0);
        atomicAdd(&slot->polar_x, s1);
        atomicAdd(&slot->polar_y, s2v);
        if (digest) atomicAdd(&slot->digest, d);
    }
}

// Id-ordered column (bit patterns) of the own agents, zero elsewhere: summed over
// the ranks it is the global column (each id is owned by exactly one rank).
__global__ void slab_column_kernel(const float4* __restrict__ st, const int32_t* __restrict__ ids, int64_t n_own, int k,
                                   unsigned long long* __restrict__ out)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_own; p += (int64_t)gridDim.x * blockDim.x) {
        const float4 s = st[p];
        const float v = k == 0 ? s.x : (k == 1 ? s.y : (k == 2 ? s.z : s.w));
        out[ids[p]] = __float_as_uint(v);
    }
}

__global__ void u64_to_f32_kernel(const unsigned long long* __restrict__ in, int64_t n, float* __restrict__ out)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        out[p] = __uint_as_float(static_cast<uint32_t>(in[p]));
}

// Own agents of a freshly initialised (or rewritten) full population.
__global__ void slab_pick_kernel(const float4* __restrict__ st, const int32_t* __restrict__ ids, int64_t n, SlabArgs g,
                                 float4* __restrict__ own, int32_t* __restrict__ own_ids, uint32_t* n_own)
{
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const float4 x = st[p];
        if (slab_of(cell_coord(x.x, g.a), g) == g.me) {
            const uint32_t q = atomicAdd(n_own, 1u);
            own[q] = x;
            own_ids[q] = ids[p];
        }
    }
}

}  // namespace

class BoidsModel final : public Model {
public:
    int64_t n = 0;
    amber_boids_params p{};
    uint64_t seed = 0;
    BoidsArgs ba{};
    DevBuf<float4> st, sorted;
    DevBuf<int32_t> ids, sids;
    DevBuf<int> cnt, start, cursor, cell_of, block_sums;
    DevBuf<float> col_tmp;
    DevBuf<int> chunk_sums;  // large-grid scan: one total per kScanChunk cells
    DevBuf<float2> svel;     // QV: float velocities in cell-sorted order
    bool vel_small = true;   // every |velocity| < 127 (true at init; re-checked on velocity writes)
    DevBuf<BoidsSlot> ring;
    int64_t m_first = 0;
    int ncell = 0;
    // lanes per agent in the stencil scan (1 = one-lane kernel; 4, 8, 16): 4 measured
    // best for both the clustered C3 (54 vs 58 us at 8) and the uniform V3 (22.6
    // vs 32.7 ms): two shuffle levels for the seven int64 sums instead of three,
    // and eight agents per warp (tools/boids_lanes_probe.py)
    int64_t lanes = 4;
    bool counted = false;  // cnt / cell_of hold the cell counts of the current state (from the last group step)
    // small grids: counts and placement counters double-buffered by step parity
    // (boids_scatter_scan_kernel); spar flips every step, independent of t
    bool fused_scan = false;
    int spar = 0;
    DevBuf<int> fill;
    int cs = 0;  // count row stride (fused_scan: a multiple of 16)
    int* cnt_of(int par) { return cnt.p + static_cast<int64_t>(par) * cs; }
    // populations up to this size count the next step's cells inside the stencil
    // kernel (one launch less); larger ones run the streaming count pass
    int64_t fused_count_max = [] {
        const char* v = getenv("AMBER_BOIDS_FUSED_COUNT_MAX");
        return v && *v ? std::atoll(v) : (1ll << 22);
    }();

    BoidsModel(int64_t n_, const amber_boids_params& p_, uint64_t seed_, const amber_runtime* r)
    {
        rt.init(r);
        n = n_;
        p = p_;
        seed = seed_;
        AMBER_REQUIRE(n >= 1 && n < (1ll << 31), "Boids needs 1 <= n_agents < 2^31");
        AMBER_REQUIRE(p.L > 0 && p.R > 0 && p.rs >= 0 && p.rs <= p.R && p.vmax > 0 && p.dt >= 0,
                      "Boids params out of range (need L, R, vmax > 0, 0 <= rs <= R, dt >= 0)");
        AMBER_REQUIRE(p.R < 0.5f * p.L && p.vmax * p.dt < 0.5f * p.L, "Boids needs R < L/2 and vmax*dt < L/2");
        ba = BoidsArgs{p.L, p.R, p.rs, p.wc, p.wa, p.ws, p.vmax, p.dt, 0, 0.f, 1};
        // Cells of side >= R*(1+1e-3) with a 3x3 stencil.  The margin means float
        // rounding of the cell index can never hide a neighbour outside the
        // stencil.  The stencil needs >= 3 distinct cells per side; boxes with
        // fewer use one cell holding every agent (each agent then scans all
        // others, i.e. the brute-force definition).  Any covering stencil gives
        // the same result (exact fixed-point sums, B3).  (A 5x5 stencil of R/2
        // cells has ~30% fewer candidates but five short row runs per agent:
        // measured slower, C3 99 vs 83 us, V3 34.9 vs 32.1 ms; not shipped.)
        const double nc1 = std::min(std::floor(static_cast<double>(p.L) / (static_cast<double>(p.R) * 1.001)), 4096.0);
        ba.nc = static_cast<int>(nc1 >= 3 ? nc1 : 1);
        ba.span = 1;
        ba.inv_cs = static_cast<float>(ba.nc / static_cast<double>(p.L));
        // x columns of width cs / sx (AMBER_BOIDS_SX): the stencil row runs shrink
        // from 3 cs to (2 + 1/sx) cs -- 25% fewer candidates at sx 4
        // (measured, tools/boids_qv_probe.py: V3 stencil 17.3 -> 15.4 ms at sx 4; C3,
        // whose small grid is L1-resident, gains nothing and keeps sx 1)
        const char* sxe = getenv("AMBER_BOIDS_SX");
        const int sx_default = n > (1ll << 22) ? 4 : 1;
        ba.sx = ba.nc >= 3 ? std::max(1, std::min(16, sxe && *sxe ? std::atoi(sxe) : sx_default)) : 1;
        while (ba.sx > 1 && static_cast<int64_t>(ba.nc) * ba.nc * ba.sx > (1ll << 30)) --ba.sx;
        ba.ncx = ba.nc * ba.sx;
        ba.inv_csx = static_cast<float>(ba.ncx / static_cast<double>(p.L));
        boids_derived(ba);
        ncell = ba.nc * ba.ncx;
        st.allocate(&rt, n);
        sorted.allocate(&rt, n);
        ids.allocate(&rt, n);
        sids.allocate(&rt, n);
        fused_scan = ba.nc > 1 && ncell <= kScanSmemCells;
        cs = fused_scan ? (ncell + 16) & ~15 : 0;
        cnt.allocate(&rt, fused_scan ? 2 * static_cast<int64_t>(cs) : ncell + 1);
        cnt.zero_async(rt.stream);
        if (fused_scan) {
            fill.allocate(&rt, 2 * static_cast<int64_t>(cs));
            fill.zero_async(rt.stream);
        }
        start.allocate(&rt, ncell + 1);
        cursor.allocate(&rt, ncell + 1);
        cell_of.allocate(&rt, n);
        chunk_sums.allocate(&rt, ceil_div(ncell + 1, kScanChunk));
        svel.allocate(&rt, n);
        ring.allocate(&rt, metrics_cap);
        ring.zero_async(rt.stream);
        boids_init_kernel<<<rt.num_sms * 8, 256, 0, rt.stream>>>(philox_key(seed), n, p.L, st.p, ids.p);
        check_launch("boids_init_kernel");
        rt.sync();
    }

    ~BoidsModel() override
    {
        if (rt.stream) cudaStreamSynchronize(rt.stream);
        st.reset(); sorted.reset(); ids.reset(); sids.reset(); cnt.reset(); start.reset(); cursor.reset(); fill.reset();
        cell_of.reset(); col_tmp.reset(); ring.reset(); block_sums.reset(); chunk_sums.reset(); svel.reset();
        rt.destroy();
    }

    // The pre-quantised-velocity stencil (QV) needs |q24(dx)| and |q24(v)| to fit
    // int32: R < 100, vmax < 64 (so every stepped velocity is small) and the
    // current velocities small (false after a write of a large velocity, until
    // the next step has clamped them); the degenerate one-cell box copies the
    // state without the scatter pass and keeps the float records.
    bool qv_ok() const { return p.R < 100.0f && p.vmax < 64.0f && ba.nc > 1; }
    bool qv_now() const { return qv_ok() && vel_small && !no_qv; }
    int64_t no_qv = 0;  // option "qv" = 0: force the float-velocity stencil (tests)

    int grid_for(int threads) const
    {
        if (grid) return static_cast<int>(grid);
        return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), rt.num_sms * 16)));
    }

    void step(int64_t nsteps) override
    {
        AMBER_REQUIRE(nsteps >= 0, "n_steps must be >= 0");
        const int threads = block ? static_cast<int>(std::min<int64_t>(block, 256)) : 256;
        for (int64_t k = 0; k < nsteps; ++k) {
            if (k % metrics_cap == 0) {  // this call's records, a ring's worth at a time
                boids_zero_slots<<<1, 256, 0, rt.stream>>>(ring.p, metrics_cap, t, std::min(nsteps - k, metrics_cap));
                check_launch("boids_zero_slots");
            }
            if (ba.nc == 1) {
                // degenerate small box: one cell holding every agent (the stencil
                // visits it once); count = n, start = {0, n}
                const int h[2] = {0, static_cast<int>(n)};
                AMBER_CUDA(cudaMemcpyAsync(start.p, h, sizeof(h), cudaMemcpyHostToDevice, rt.stream));
                AMBER_CUDA(cudaMemcpyAsync(sorted.p, st.p, n * sizeof(float4), cudaMemcpyDeviceToDevice, rt.stream));
                AMBER_CUDA(cudaMemcpyAsync(sids.p, ids.p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, rt.stream));
            } else {
                // the cell counts: from the previous group step (fused), else a count pass
                if (!counted) {
                    prof.launch(rt.stream, "boids_bin", [&] {
                        boids_count_kernel<<<grid_for(threads), threads, 0, rt.stream>>>(st.p, n, ba, cnt_of(spar),
                                                                                         nullptr, nullptr);
                    });
                    check_launch("boids_count_kernel");
                }
                counted = false;
                // exclusive scan of the ncell + 1 counts (cnt[ncell] = 0, so start[ncell] = n),
                // cursors = starts, counts re-zeroed for the next step: one CTA for small
                // grids, a device-wide scan for large ones (the one-CTA scan took 20 ms at
                // V3's 10^7 cells, r01)
                if (fused_scan) {
                    prof.launch(rt.stream, "boids_scatter", [&] {
                        const int gs = grid ? static_cast<int>(grid)
                                            : static_cast<int>(std::max<int64_t>(
                                                  1, std::min<int64_t>(ceil_div(n, 1024), rt.num_sms)));
                        launch_pdl(boids_scatter_scan_kernel, gs, 1024, 0, rt.stream, st.p, ids.p, n, cnt_of(spar),
                                   cnt_of(spar ^ 1), fill.p + spar * cs, fill.p + (spar ^ 1) * cs, ncell, cs,
                                   start.p, sorted.p, sids.p, qv_now() ? svel.p : nullptr, ba);
                    });
                    check_launch("boids_scatter_scan_kernel");
                } else {
                prof.launch(rt.stream, "boids_scan", [&] {
                    if (ncell <= (1 << 16)) {  // one launch: scan, cursors, re-zeroed counts
                        boids_scan_reg_kernel<<<1, 1024, 0, rt.stream>>>(cnt.p, start.p, cursor.p, ncell);
                    } else {
                        const int nch = static_cast<int>(ceil_div(ncell + 1, kScanChunk));
                        boids_chunk_sums_kernel<<<nch, 1024, 0, rt.stream>>>(cnt.p, ncell + 1, chunk_sums.p);
                        check_launch("boids_chunk_sums_kernel");
                        boids_chunk_offsets_kernel<<<1, 1024, 0, rt.stream>>>(chunk_sums.p, nch);
                        check_launch("boids_chunk_offsets_kernel");
                        boids_chunk_scan_kernel<<<nch, 1024, 0, rt.stream>>>(cnt.p, chunk_sums.p, ncell, start.p,
                                                                              cursor.p);
                    }
                });
                check_launch("boids_scan");
                prof.launch(rt.stream, "boids_scatter", [&] {
                    boids_scatter_kernel<<<grid_for(threads), threads, 0, rt.stream>>>(
                        st.p, ids.p, n, nullptr, cursor.p, sorted.p, sids.p, cnt.p,
                        ncell <= (1 << 16) ? ncell : 0,
                        qv_now() ? svel.p : nullptr, ba);
                });
                check_launch("boids_scatter_kernel");
                }
            }
            const BoidsArgs a = ba;
            {
                // each block steps a contiguous range of the sorted agents: at least
                // 8 blocks per SM, and at most 64 rounds per block for large N (many
                // short ranges keep the blocks balanced once flocks cluster)
                const int64_t apb = threads / lanes;
                const int g = grid ? static_cast<int>(grid)
                                   : static_cast<int>(std::max<int64_t>(
                                         {1, std::min<int64_t>(ceil_div(n * lanes, threads), rt.num_sms * 8),
                                          ceil_div(n, apb * 64)}));
                BoidsSlot* sl = ring.p + (t % metrics_cap);
                const int dg = digest_on ? 1 : 0;
                prof.launch(rt.stream, "boids_step", [&] {
                    // small populations: the group step also counts the next step's
                    // cells (one launch less per step: C3 83 -> 75 us); large ones keep
                    // the streaming count pass (the stencil kernel is issue-bound there:
                    // fused, V3 32.8 -> 33.7 ms)
                    int* nc_cnt = ba.nc > 1 && n <= fused_count_max ? cnt_of(spar ^ 1) : nullptr;
                    const bool qv = qv_now();
#define AMBER_BOIDS_GROUP(G_, QV_, MB_)                                                                          \
    launch_pdl(boids_group_kernel<G_, QV_, MB_>, g, threads, 0, rt.stream, sorted.p, sids.p, start.p, n, a, st.p, \
               ids.p, sl, dg, nc_cnt, static_cast<int*>(nullptr), svel.p)
#define AMBER_BOIDS_GROUP4(QV_)                                                  \
    if (n > (1ll << 22)) AMBER_BOIDS_GROUP(4, QV_, AMBER_BOIDS_MINB_LARGE); \
    else AMBER_BOIDS_GROUP(4, QV_, AMBER_BOIDS_MINB)
                    if (lanes == 4) {
                        if (qv) { AMBER_BOIDS_GROUP4(true); } else { AMBER_BOIDS_GROUP4(false); }
                    } else if (lanes == 16) {
                        if (qv) AMBER_BOIDS_GROUP(16, true, AMBER_BOIDS_MINB); else AMBER_BOIDS_GROUP(16, false, AMBER_BOIDS_MINB);
                    } else {
                        if (qv) AMBER_BOIDS_GROUP(8, true, AMBER_BOIDS_MINB); else AMBER_BOIDS_GROUP(8, false, AMBER_BOIDS_MINB);
                    }
#undef AMBER_BOIDS_GROUP4
#undef AMBER_BOIDS_GROUP
                });
                check_launch("boids_group_kernel");
                counted = ba.nc > 1 && n <= fused_count_max;
            }
            if (fused_scan) spar ^= 1;
            ++t;
            if (p.vmax < 64.0f) vel_small = true;  // the step clamped every velocity to vmax < 64
        }
    }

    int col_index(const std::string& k) const
    {
        if (k == "pos_x") return 0;
        if (k == "pos_y") return 1;
        if (k == "vel_x") return 2;
        if (k == "vel_y") return 3;
        return -1;
    }

    bool column_info(const char* name, amber_dtype* dt, int64_t* glen, int64_t* off, int64_t* len) override
    {
        if (col_index(name) < 0) return false;
        if (dt) *dt = AMBER_F32;
        if (glen) *glen = n;
        if (off) *off = 0;
        if (len) *len = n;
        return true;
    }

    void read_column(const char* name, void* dst, size_t bytes, bool on_dev) override
    {
        const int k = col_index(name);
        if (k < 0) fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        if (bytes < static_cast<size_t>(n) * 4) fail(AMBER_E_BUFFER_TOO_SMALL, "dst too small");
        if (!col_tmp.p) col_tmp.allocate(&rt, n);
        boids_gather_column<<<grid_for(256), 256, 0, rt.stream>>>(st.p, ids.p, n, k, col_tmp.p);
        check_launch("boids_gather_column");
        copy_out(rt, dst, col_tmp.p, n * 4, on_dev);
    }

    void write_column(const char* name, const void* src, size_t bytes, bool on_dev) override
    {
        const int k = col_index(name);
        if (k < 0) fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        if (bytes < static_cast<size_t>(n) * 4) fail(AMBER_E_BUFFER_TOO_SMALL, "src too small");
        if (!col_tmp.p) col_tmp.allocate(&rt, n);
        copy_in(rt, col_tmp.p, src, n * 4, on_dev);
        boids_put_column<<<grid_for(256), 256, 0, rt.stream>>>(st.p, ids.p, n, k, col_tmp.p);
        check_launch("boids_put_column");
        if (k >= 2) {  // a velocity column: are all velocities still small enough for the QV stencil?
            DevBuf<unsigned int> big;
            big.allocate(&rt, 1);
            big.zero_async(rt.stream);
            boids_big_velocity_kernel<<<grid_for(256), 256, 0, rt.stream>>>(st.p, n, big.p);
            check_launch("boids_big_velocity_kernel");
            unsigned int h = 0;
            AMBER_CUDA(cudaMemcpyAsync(&h, big.p, 4, cudaMemcpyDeviceToHost, rt.stream));
            rt.sync();
            vel_small = h == 0;
        }
        // positions changed: drop the counts the last group step left (the next
        // step counts again from zero)
        if (counted) AMBER_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), rt.stream));
        rt.sync();
        counted = false;
    }

    void read_metrics(const char* name, void* dst, size_t bytes, int64_t* n_out) override
    {
        std::string k(name);
        if (k != "mean_speed" && k != "polarisation" && !(k == "digest" && digest_on))
            fail(AMBER_E_UNKNOWN_NAME, "no metric " + k);
        std::vector<BoidsSlot> h(metrics_cap);
        AMBER_CUDA(cudaMemcpyAsync(h.data(), ring.p, metrics_cap * sizeof(BoidsSlot), cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        const int64_t first = std::max(m_first, t - metrics_cap + 1);
        const int64_t cnt_ = std::max<int64_t>(t - first, 0);
        if (bytes < static_cast<size_t>(cnt_) * 8) fail(AMBER_E_BUFFER_TOO_SMALL, "metrics dst too small");
        for (int64_t s = first; s < t; ++s) {
            const BoidsSlot& x = h[s % metrics_cap];
            if (k == "mean_speed") static_cast<double*>(dst)[s - first] = x.mean_speed / static_cast<double>(n);
            else if (k == "polarisation")
                static_cast<double*>(dst)[s - first] = std::sqrt(x.polar_x * x.polar_x + x.polar_y * x.polar_y) / static_cast<double>(n);
            else static_cast<unsigned long long*>(dst)[s - first] = x.digest;
        }
        if (n_out) *n_out = cnt_;
    }

    void reset_metrics() override
    {
        rt.sync();
        m_first = t;
    }

    uint64_t digest(const char* name) override
    {
        const int k = col_index(name);
        if (k < 0) fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        if (!col_tmp.p) col_tmp.allocate(&rt, n);
        boids_gather_column<<<grid_for(256), 256, 0, rt.stream>>>(st.p, ids.p, n, k, col_tmp.p);
        check_launch("boids_gather_column");
        return device_digest_u32(rt, reinterpret_cast<const uint32_t*>(col_tmp.p), n, 0);
    }

    void set_step(int64_t s) override
    {
        AMBER_REQUIRE(s >= 0, "step out of range");
        rt.sync();
        t = s;
        m_first = s;
    }

    bool set_option(const char* key, int64_t v) override
    {
        std::string k(key);
        if (k == "metrics_capacity") {
            AMBER_REQUIRE(v >= 16, "metrics_capacity must be >= 16");
            rt.sync();
            metrics_cap = v;
            ring.allocate(&rt, metrics_cap);
            ring.zero_async(rt.stream);
            m_first = t;
            return true;
        }
        if (k == "block") AMBER_REQUIRE(v <= 256, "Boids kernels are built for <= 256 threads per block");
        if (k == "qv") {
            no_qv = v ? 0 : 1;
            return true;
        }
        if (k == "lanes") {
            AMBER_REQUIRE(v == 4 || v == 8 || v == 16, "lanes must be 4, 8 or 16");
            lanes = v;
            return true;
        }
        return Model::set_option(key, v);
    }

    bool get_option(const char* key, int64_t* v) override
    {
        if (std::string(key) == "cells_per_side") {
            *v = ba.nc;
            return true;
        }
        if (std::string(key) == "x_subdivision") {  // columns per cell width in x
            *v = ba.sx;
            return true;
        }
        if (std::string(key) == "lanes") {
            *v = lanes;
            return true;
        }
        if (std::string(key) == "stencil_candidates") {  // candidate visits of the last step's stencil pass
            AMBER_REQUIRE(ba.nc >= 3, "stencil_candidates needs >= 3 cells per side");
            DevBuf<unsigned long long> d;
            d.allocate(&rt, 1);
            d.zero_async(rt.stream);
            boids_candidates_kernel<<<rt.num_sms * 8, 256, 0, rt.stream>>>(start.p, ba.nc, ba.ncx, ba.sx, d.p);
            check_launch("boids_candidates_kernel");
            unsigned long long h = 0;
            AMBER_CUDA(cudaMemcpyAsync(&h, d.p, 8, cudaMemcpyDeviceToHost, rt.stream));
            rt.sync();
            *v = static_cast<int64_t>(h);
            return true;
        }
        if (std::string(key) == "qv") {  // 1: the next step runs the pre-quantised-velocity stencil
            *v = qv_now() ? 1 : 0;
            return true;
        }
        return Model::get_option(key, v);
    }
};

// Sharded Boids (NEXT-3): see the slab kernels above.  Columns and digests
// are global (collective reads); metrics are summed over the ranks.
class BoidsShardModel final : public Model {
public:
    int64_t n = 0;
    amber_boids_params p{};
    BoidsArgs ba{};
    ShardComm* sc = nullptr;
    std::vector<int> col0;      // [world + 1]
    DevBuf<int> d_col0;
    int c_lo = 0, c_hi = 0, w = 0;
    int64_t n_own = 0, cap = 0;
    DevBuf<float4> st, st2, sorted;
    DevBuf<int32_t> ids, ids2, sids, cell_of;
    DevBuf<BoidAgent> send, recv;
    DevBuf<uint32_t> counts, keep_n;
    DevBuf<int> cnt, start, cursor;
    DevBuf<int> chunk_sums;  // hand-written chunked scan (kScanChunk cells per total)
    int ncell_loc = 0;
    DevBuf<BoidsSlot> ring;
    int64_t m_first = 0;

    BoidsShardModel(int64_t n_, const amber_boids_params& p_, uint64_t seed, const amber_runtime* r)
    {
        rt.init(r);
        n = n_;
        p = p_;
        AMBER_REQUIRE(n >= 1 && n < (1ll << 31), "Boids needs 1 <= n_agents < 2^31");
        AMBER_REQUIRE(p.L > 0 && p.R > 0 && p.rs >= 0 && p.rs <= p.R && p.vmax > 0 && p.dt >= 0,
                      "Boids params out of range (need L, R, vmax > 0, 0 <= rs <= R, dt >= 0)");
        AMBER_REQUIRE(p.R < 0.5f * p.L && p.vmax * p.dt < 0.5f * p.L, "Boids needs R < L/2 and vmax*dt < L/2");
        ba = BoidsArgs{p.L, p.R, p.rs, p.wc, p.wa, p.ws, p.vmax, p.dt, 0, 0.f, 1};  // 3x3 stencil, halo 1 column
        double nc = std::floor(static_cast<double>(p.L) / (static_cast<double>(p.R) * 1.001));
        nc = std::min(nc, 4096.0);
        AMBER_REQUIRE(nc >= 3 && nc >= rt.world, "sharded Boids needs >= 3 cells per side and >= 1 cell column per rank");
        ba.nc = static_cast<int>(nc);
        ba.inv_cs = static_cast<float>(ba.nc / static_cast<double>(p.L));
        // sub-rows in y (slab_cell): sy = AMBER_BOIDS_SX, default 4 above 2^22
        // agents (as the one-GPU grid's x columns), 1 below
        const char* sye = getenv("AMBER_BOIDS_SX");
        int sy = n > (1ll << 22) ? 4 : 1;
        if (sye && *sye) sy = std::max(1, std::min(16, std::atoi(sye)));
        ba.sx = sy;
        ba.ncx = ba.nc * sy;
        ba.inv_csx = static_cast<float>(ba.ncx / static_cast<double>(p.L));
        boids_derived(ba);
        col0.resize(rt.world + 1);
        for (int q = 0; q <= rt.world; ++q) col0[q] = static_cast<int>(static_cast<int64_t>(q) * ba.nc / rt.world);
        c_lo = col0[rt.rank];
        c_hi = col0[rt.rank + 1];
        w = c_hi - c_lo;
        ncell_loc = (w + 2) * ba.ncx;
        d_col0.allocate(&rt, rt.world + 1);
        AMBER_CUDA(cudaMemcpyAsync(d_col0.p, col0.data(), col0.size() * sizeof(int), cudaMemcpyHostToDevice, rt.stream));
        cap = n;  // per-destination send capacity: any distribution of the agents fits
        for (auto* b : {&st, &st2}) b->allocate(&rt, n);
        for (auto* b : {&ids, &ids2}) b->allocate(&rt, n);
        sorted.allocate(&rt, 2 * n);
        sids.allocate(&rt, 2 * n);
        cell_of.allocate(&rt, 2 * n);
        send.allocate(&rt, static_cast<size_t>(rt.world) * cap);
        recv.allocate(&rt, n);
        counts.allocate(&rt, rt.world);
        keep_n.allocate(&rt, 1);
        cnt.allocate(&rt, ncell_loc + 1);
        cnt.zero_async(rt.stream);
        start.allocate(&rt, ncell_loc + 1);
        cursor.allocate(&rt, ncell_loc + 1);
        chunk_sums.allocate(&rt, ceil_div(ncell_loc + 1, kScanChunk));
        ring.allocate(&rt, metrics_cap);
        ring.zero_async(rt.stream);
        // every rank draws the full seeded population (B1) and keeps its slab
        boids_init_kernel<<<rt.num_sms * 8, 256, 0, rt.stream>>>(philox_key(seed), n, p.L, st2.p, ids2.p);
        check_launch("boids_init_kernel");
        pick(st2.p, ids2.p);
        sc = make_shard_comm(rt, r);
        rt.sync();
    }

    ~BoidsShardModel() override
    {
        if (rt.stream) cudaStreamSynchronize(rt.stream);
        for (auto* b : {&st, &st2, &sorted}) b->reset();
        for (auto* b : {&ids, &ids2, &sids, &cell_of}) b->reset();
        send.reset(); recv.reset(); counts.reset(); keep_n.reset(); cnt.reset(); start.reset(); cursor.reset();
        chunk_sums.reset(); ring.reset(); d_col0.reset();
        if (sc) destroy_shard_comm(sc);
        rt.destroy();
    }

    SlabArgs args() const { return SlabArgs{ba, d_col0.p, rt.world, rt.rank, c_lo, c_hi, static_cast<uint64_t>(cap)}; }
    int grid_for(int64_t items) const
    {
        return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, 256), rt.num_sms * 16)));
    }

    // own agents of a full id-ordered population (st_full, ids_full)
    void pick(const float4* st_full, const int32_t* ids_full)
    {
        keep_n.zero_async(rt.stream);
        slab_pick_kernel<<<grid_for(n), 256, 0, rt.stream>>>(st_full, ids_full, n, args(), st.p, ids.p, keep_n.p);
        check_launch("slab_pick_kernel");
        uint32_t h = 0;
        AMBER_CUDA(cudaMemcpyAsync(&h, keep_n.p, 4, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        n_own = h;
    }

    void step(int64_t nsteps) override
    {
        AMBER_REQUIRE(nsteps >= 0, "n_steps must be >= 0");
        const SlabArgs g = args();
        for (int64_t k = 0; k < nsteps; ++k) {
            boids_zero_slots<<<1, 32, 0, rt.stream>>>(ring.p, metrics_cap, t, 1);
            check_launch("boids_zero_slots");
            // 1) migration
            counts.zero_async(rt.stream);
            keep_n.zero_async(rt.stream);
            prof.launch(rt.stream, "boids_slab_route", [&] {
                slab_route_kernel<<<grid_for(n_own), 256, 0, rt.stream>>>(st.p, ids.p, n_own, g, st2.p, ids2.p,
                                                                           keep_n.p, send.p, counts.p);
            });
            check_launch("slab_route_kernel");
            const uint64_t got = shard_alltoallv(sc, rt, send.p, counts.p, cap, sizeof(BoidAgent), recv.p, n);
            uint32_t kept = 0;
            AMBER_CUDA(cudaMemcpyAsync(&kept, keep_n.p, 4, cudaMemcpyDeviceToHost, rt.stream));
            rt.sync();
            if (got)
                slab_unpack_kernel<<<grid_for(got), 256, 0, rt.stream>>>(recv.p, got, st2.p, ids2.p, kept);
            check_launch("slab_unpack_kernel");
            n_own = kept + static_cast<int64_t>(got);
            std::swap(st.p, st2.p);
            std::swap(ids.p, ids2.p);
            // 2) halos
            counts.zero_async(rt.stream);
            prof.launch(rt.stream, "boids_slab_halo", [&] {
                slab_halo_kernel<<<grid_for(n_own), 256, 0, rt.stream>>>(st.p, ids.p, n_own, g, send.p, counts.p);
            });
            check_launch("slab_halo_kernel");
            const int64_t n_halo = static_cast<int64_t>(
                shard_alltoallv(sc, rt, send.p, counts.p, cap, sizeof(BoidAgent), recv.p, n));
            // 3) local binning (column-major, halo columns 0 and w + 1)
            const int64_t tot = n_own + n_halo;
            prof.launch(rt.stream, "boids_slab_bin", [&] {
                slab_count_kernel<<<grid_for(tot), 256, 0, rt.stream>>>(st.p, n_own, recv.p, n_halo, g, cnt.p,
                                                                         cell_of.p);
                check_launch("slab_count_kernel");
                const int nch = static_cast<int>(ceil_div(ncell_loc + 1, kScanChunk));
                boids_chunk_sums_kernel<<<nch, 1024, 0, rt.stream>>>(cnt.p, static_cast<int>(ncell_loc + 1),
                                                                      chunk_sums.p);
                check_launch("boids_chunk_sums_kernel");
                boids_chunk_offsets_kernel<<<1, 1024, 0, rt.stream>>>(chunk_sums.p, nch);
                check_launch("boids_chunk_offsets_kernel");
                boids_chunk_scan_kernel<<<nch, 1024, 0, rt.stream>>>(cnt.p, chunk_sums.p, static_cast<int>(ncell_loc),
                                                                      start.p, cursor.p);
                check_launch("boids_chunk_scan_kernel");
                slab_scatter_kernel<<<grid_for(tot), 256, 0, rt.stream>>>(st.p, ids.p, n_own, recv.p, n_halo,
                                                                           cell_of.p, cursor.p, sorted.p, sids.p);
            });
            check_launch("slab_scatter_kernel");
            // 4) the step of the own agents: sorted[start[nc], start[(w + 1) nc])
            int own_rng[2] = {0, 0};
            AMBER_CUDA(cudaMemcpyAsync(&own_rng[0], start.p + ba.ncx, 4, cudaMemcpyDeviceToHost, rt.stream));
            AMBER_CUDA(cudaMemcpyAsync(&own_rng[1], start.p + (w + 1) * ba.ncx, 4, cudaMemcpyDeviceToHost, rt.stream));
            rt.sync();
            AMBER_REQUIRE(own_rng[1] - own_rng[0] == n_own, "sharded Boids: own agents outside the slab columns");
            const int gsteps = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_own * 4, 256),
                                                                                        rt.num_sms * 8)));
            BoidsSlot* sl = ring.p + (t % metrics_cap);
            const int dg = digest_on ? 1 : 0;
            prof.launch(rt.stream, "boids_slab_step", [&] {
                slab_step_kernel<4><<<gsteps, 256, 0, rt.stream>>>(sorted.p, sids.p, start.p, own_rng[0], own_rng[1], g,
                                                                    st.p, ids.p, sl, dg);
            });
            check_launch("slab_step_kernel");
            ++t;
        }
    }

    int col_index(const std::string& k) const
    {
        if (k == "pos_x") return 0;
        if (k == "pos_y") return 1;
        if (k == "vel_x") return 2;
        if (k == "vel_y") return 3;
        return -1;
    }

    bool column_info(const char* name, amber_dtype* dt, int64_t* glen, int64_t* off, int64_t* len) override
    {
        if (col_index(name) < 0) return false;
        if (dt) *dt = AMBER_F32;
        if (glen) *glen = n;
        if (off) *off = 0;
        if (len) *len = n;  // reads are collective and return the whole id-ordered column
        return true;
    }

    // Global id-ordered column on every rank (collective): own values by id, zero
    // elsewhere, summed over the ranks as bit patterns.
    void gather_column(int k, unsigned long long* dcol)
    {
        AMBER_CUDA(cudaMemsetAsync(dcol, 0, n * 8, rt.stream));
        slab_column_kernel<<<grid_for(n_own), 256, 0, rt.stream>>>(st.p, ids.p, n_own, k, dcol);
        check_launch("slab_column_kernel");
        shard_allreduce_u64(sc, rt, dcol, static_cast<size_t>(n));
    }

    void read_column(const char* name, void* dst, size_t bytes, bool on_dev) override
    {
        const int k = col_index(name);
        if (k < 0) fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        if (bytes < static_cast<size_t>(n) * 4) fail(AMBER_E_BUFFER_TOO_SMALL, "dst too small");
        DevBuf<unsigned long long> col;
        col.allocate(&rt, n);
        DevBuf<float> f;
        f.allocate(&rt, n);
        gather_column(k, col.p);
        u64_to_f32_kernel<<<grid_for(n), 256, 0, rt.stream>>>(col.p, n, f.p);
        check_launch("u64_to_f32_kernel");
        copy_out(rt, dst, f.p, n * 4, on_dev);
    }

    // Collective: every rank passes the same whole id-ordered column; agents whose
    // position changes slabs migrate at the next step.
    void write_column(const char* name, const void* src, size_t bytes, bool on_dev) override
    {
        const int k = col_index(name);
        if (k < 0) fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        if (bytes < static_cast<size_t>(n) * 4) fail(AMBER_E_BUFFER_TOO_SMALL, "src too small");
        DevBuf<float> f;
        f.allocate(&rt, n);
        copy_in(rt, f.p, src, n * 4, on_dev);
        boids_put_column<<<grid_for(n_own), 256, 0, rt.stream>>>(st.p, ids.p, n_own, k, f.p);
        check_launch("boids_put_column");
        rt.sync();
    }

    void read_metrics(const char* name, void* dst, size_t bytes, int64_t* n_out) override
    {
        std::string k(name);
        if (k != "mean_speed" && k != "polarisation" && !(k == "digest" && digest_on))
            fail(AMBER_E_UNKNOWN_NAME, "no metric " + k);
        std::vector<BoidsSlot> h(metrics_cap);
        AMBER_CUDA(cudaMemcpyAsync(h.data(), ring.p, metrics_cap * sizeof(BoidsSlot), cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        const int64_t first = std::max(m_first, t - metrics_cap + 1);
        const int64_t cnt_ = std::max<int64_t>(t - first, 0);
        if (bytes < static_cast<size_t>(cnt_) * 8) fail(AMBER_E_BUFFER_TOO_SMALL, "metrics dst too small");
        // sum the per-rank slots (doubles as bit patterns would not add: gather them instead)
        std::vector<unsigned long long> mine(4 * cnt_);
        for (int64_t s = first; s < t; ++s) {
            const BoidsSlot& x = h[s % metrics_cap];
            std::memcpy(&mine[4 * (s - first)], &x, sizeof(BoidsSlot));
        }
        std::vector<double> all;
        if (cnt_) {
            DevBuf<unsigned long long> d;
            d.allocate(&rt, 4 * cnt_ * rt.world);
            DevBuf<unsigned long long> m;
            m.allocate(&rt, 4 * cnt_);
            AMBER_CUDA(cudaMemcpyAsync(m.p, mine.data(), mine.size() * 8, cudaMemcpyHostToDevice, rt.stream));
            shard_allgather_u32(sc, rt, reinterpret_cast<const uint32_t*>(m.p), reinterpret_cast<uint32_t*>(d.p),
                                8 * cnt_);
            all.resize(4 * cnt_ * rt.world);
            AMBER_CUDA(cudaMemcpyAsync(all.data(), d.p, all.size() * 8, cudaMemcpyDeviceToHost, rt.stream));
            rt.sync();
        }
        for (int64_t s = 0; s < cnt_; ++s) {
            double sp = 0, px = 0, py = 0;
            unsigned long long dg = 0;
            for (int q = 0; q < rt.world; ++q) {
                const double* v = all.data() + (static_cast<size_t>(q) * cnt_ + s) * 4;
                sp += v[0];
                px += v[1];
                py += v[2];
                unsigned long long u;
                std::memcpy(&u, v + 3, 8);
                dg += u;
            }
            if (k == "mean_speed") static_cast<double*>(dst)[s] = sp / static_cast<double>(n);
            else if (k == "polarisation") static_cast<double*>(dst)[s] = std::sqrt(px * px + py * py) / static_cast<double>(n);
            else static_cast<unsigned long long*>(dst)[s] = dg;
        }
        if (n_out) *n_out = cnt_;
    }

    void reset_metrics() override
    {
        rt.sync();
        m_first = t;
    }

    uint64_t digest(const char* name) override
    {
        const int k = col_index(name);
        if (k < 0) fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        DevBuf<unsigned long long> col;
        col.allocate(&rt, n);
        gather_column(k, col.p);
        DevBuf<uint32_t> c32;
        c32.allocate(&rt, n);
        u64_to_f32_kernel<<<grid_for(n), 256, 0, rt.stream>>>(col.p, n, reinterpret_cast<float*>(c32.p));
        check_launch("u64_to_f32_kernel");
        return device_digest_u32(rt, c32.p, n, 0);
    }

    void set_step(int64_t s) override
    {
        AMBER_REQUIRE(s >= 0, "step out of range");
        rt.sync();
        t = s;
        m_first = s;
    }

    bool set_option(const char* key, int64_t v) override
    {
        std::string k(key);
        if (k == "metrics_capacity") {
            AMBER_REQUIRE(v >= 16, "metrics_capacity must be >= 16");
            rt.sync();
            metrics_cap = v;
            ring.allocate(&rt, metrics_cap);
            ring.zero_async(rt.stream);
            m_first = t;
            return true;
        }
        return Model::set_option(key, v);
    }

    bool get_option(const char* key, int64_t* v) override
    {
        std::string k(key);
        if (k == "cells_per_side") { *v = ba.nc; return true; }
        if (k == "own_agents") { *v = n_own; return true; }
        if (k == "slab_columns") { *v = w; return true; }
        return Model::get_option(key, v);
    }
};

Model* make_boids(int64_t n, const amber_boids_params& p, uint64_t seed, const amber_runtime* rt)
{
    // AMBER_TEST_FORCE_EXCHANGE=1 with a unique id: the sharded path with one rank
    const char* force = getenv("AMBER_TEST_FORCE_EXCHANGE");
    if ((rt && rt->world > 1) || (force && force[0] == '1' && rt && rt->nccl_unique_id))
        return new BoidsShardModel(n, p, seed, rt);
    return new BoidsModel(n, p, seed, rt);
}

}  // namespace amber
