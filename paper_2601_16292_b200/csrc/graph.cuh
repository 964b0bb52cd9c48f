// graph.cuh -- batched Erdos-Renyi CSR built on the device (sir.cu), shared by
// the SIR model and the replicate sweep (sweep.cu).
#pragma once

#include <vector>

#include "internal.cuh"

namespace amber {

// R independent G(n, M) graphs as one CSR over R*n vertices (vertex r*n + v);
// row_ptr holds global offsets, col holds replicate-local neighbour ids.
struct Graphs {
    int64_t R = 0, n = 0, m = 0, arcs = 0;
    DevBuf<int32_t> row_ptr;  // R*n + 1
    DevBuf<int32_t> col;      // arcs (+ padding)
};

// G1-G3 for every seed in `seeds` (M endpoint draws each).
void build_graphs(Runtime& rt, const std::vector<unsigned long long>& seeds, int64_t n, int64_t m, Graphs& g);

// S1: initial states (row stride n_pad; padding entries = 3) for every seed.
void build_init_state(Runtime& rt, const std::vector<unsigned long long>& seeds, int64_t n, int64_t n_pad,
                      int64_t k_inf, uint8_t* state, uint32_t tag = 0x12u);

// Warp-cooperative walk over the concatenated CSR rows of the lanes in `own`
// (lane L owns row [rb_L, re_L); col_at(e) returns the neighbour of arc e).
// Position q of the concatenation -> owner lane by a 5-step shuffle search
// over the inclusive prefix of the row lengths (SIR step, sir.cu, and the
// replicate sweep, sweep.cu).  kU batches of 32 arcs are in flight per iteration: all their
// column loads are issued, then all the neighbour tests, so each warp keeps
// kU x 32 independent gathers outstanding (the walk is latency-bound on the
// col -> bitmap chain at large N).  test(j, e, owner) returns true for an arc
// that sets the owner's bit; owners whose bit is set skip their remaining arcs
// (early exit).  Returns the mask of owners with a set bit.  All 32 lanes call it.
struct NoProbe {
    __device__ __forceinline__ uint32_t operator()(uint32_t) const { return 1u; }
};

// probe(j) (optional) is the arc's neighbour lookup: it runs for all kU
// batches before any test, so their kU x 32 loads are in flight together (a
// load inside test() is ordered after the previous batch's branch on its own
// load); test() then sees only arcs whose probe returned non-zero.
template <int kU, bool kPay, bool kFast, class C, class P, class T>
__device__ __forceinline__ uint32_t walk_rows_core(C&& col_at, uint32_t own, int32_t rb, int32_t re, uint32_t pay,
                                                   P&& probe, T&& test)
{
    const int lane = threadIdx.x & 31;
    const int32_t len = ((own >> lane) & 1u) ? re - rb : 0;
    int32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const int32_t start = rb - (incl - len);  // arc index of concatenation position q is start_L + q
    // kFast: owner lookup by row-end bits when the non-empty rows are lanes 0 .. k-1 (owners
    // compacted to a prefix, no empty row among them -- the common case): the
    // prefix ends incl_L are then strictly increasing, so the owner of position
    // q = (#lanes with incl <= q0 - 1) + (#row ends in [q0, q]) -- one OR-reduce
    // of the row-end bits of the 32-position window and a popc per batch,
    // instead of the 5-step shuffle search.  Measured (r02): V2 1.354 -> 1.335
    // ms/step, C5 24.09 -> 23.90 ms, SIR in space (rows compacted to a lane
    // prefix first) 0.171 -> 0.166 ms; C2 4.94 -> 5.04 us slower (short walks at
    // one agent per lane: the ballot and check cost more than they save), so
    // the small-population SIR walk keeps the search.  Also measured and not kept:
    // compacting the arcs whose probe passed before the draws (full-warp
    // Philox instead of SIMT utilisation = hit rate): faster only below ~35%
    // susceptible neighbours in push steps (V2 steps 15-19, which pull), slower
    // above (compaction cost > saved draws); and drawing every live arc of the
    // kU batches branch-free before the tests, so the kU Philox chains overlap
    // (V2 1.296 vs 1.274 ms: the four live draws cost registers at the 48 cap).
    const uint32_t ne = kFast ? __ballot_sync(0xffffffffu, len > 0) : 0u;
    const bool fast = kFast && (ne & (ne + 1u)) == 0u;
    const uint32_t le = 0xffffffffu >> (31 - lane);  // lanes 0 .. lane
    int base = 0;  // fast: #lanes with incl <= q0 - 1
    uint32_t hit = 0;
    for (int32_t q0 = 0; q0 < total; q0 += 32 * kU) {
        int Ls[kU];
        int32_t es[kU];
        uint32_t ps[kU];
        bool live[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            live[u] = false;
            Ls[u] = 0;
            es[u] = 0;
            ps[u] = 0;
            if (q0 + 32 * u >= total) continue;  // warp-uniform: no dead batches
            const int32_t q = q0 + 32 * u + lane;
            int L = 0;  // number of lanes with incl <= q = the owner of position q
            if (fast) {
                const uint32_t d = static_cast<uint32_t>(incl - (q0 + 32 * u));
                const uint32_t m = __reduce_or_sync(0xffffffffu, d < 32u ? 1u << (d & 31u) : 0u);
                L = base + __popc(m & le);
                base += __popc(m);
            } else {
#pragma unroll
                for (int st = 16; st > 0; st >>= 1) {
                    const int32_t v = __shfl_sync(0xffffffffu, incl, (L + st - 1) & 31);
                    if (v <= q) L += st;
                }
            }
            L &= 31;
            Ls[u] = L;
            es[u] = __shfl_sync(0xffffffffu, start, L) + q;
            if constexpr (kPay) ps[u] = __shfl_sync(0xffffffffu, pay, L);
            live[u] = q < total && !((hit >> L) & 1u);
        }
        uint32_t js[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) js[u] = live[u] ? col_at(es[u]) : 0u;
        uint32_t pb[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) pb[u] = live[u] ? probe(js[u]) : 0u;
        uint32_t add = 0;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            bool h = false;
            if constexpr (kPay) h = pb[u] && test(js[u], es[u], Ls[u], ps[u]);
            else h = pb[u] && test(js[u], es[u], Ls[u]);
            if (h) add |= 1u << Ls[u];
        }
        hit |= __reduce_or_sync(0xffffffffu, add);
        if ((hit & own) == own) break;  // every owner decided
    }
    return hit;
}

template <int kU, class C, class T>
__device__ __forceinline__ uint32_t walk_rows(C&& col_at, uint32_t own, int32_t rb, int32_t re, T&& test)
{
    return walk_rows_core<kU, false, false>(col_at, own, rb, re, 0u, NoProbe{}, test);
}

// walk_rows with a neighbour probe (see walk_rows_core): test(j, e, owner)
// runs only where probe(j) != 0.
template <int kU, bool kFast = false, class C, class P, class T>
__device__ __forceinline__ uint32_t walk_rows_probe(C&& col_at, uint32_t own, int32_t rb, int32_t re, P&& probe,
                                                    T&& test)
{
    return walk_rows_core<kU, false, kFast>(col_at, own, rb, re, 0u, probe, test);
}

// walk_rows with a per-owner payload: test(j, e, owner, pay_of_owner).  Used
// when the owner lanes were compacted from several warp chunks (the owner's
// agent id is no longer chunk base + lane).
template <int kU, bool kFast = false, class C, class P, class T>
__device__ __forceinline__ uint32_t walk_rows_pay(C&& col_at, uint32_t own, int32_t rb, int32_t re, uint32_t pay,
                                                  P&& probe, T&& test)
{
    return walk_rows_core<kU, true, kFast>(col_at, own, rb, re, pay, probe, test);
}

// Appends the agents a0 + b for the set bits b of `mask` to the warp's owner
// queue (lane k holds the k-th queued agent in qid; qc = queued count), and
// walks 32 of them as soon as 32 are queued (sweep.cu, sirs.cu).  All 32 lanes
// call it.
template <class W>
__device__ __forceinline__ void enqueue(uint32_t mask, uint32_t a0, uint32_t& qid, uint32_t& qc, W&& walk)
{
    const uint32_t lane = threadIdx.x & 31, k = __popc(mask);
    if (!k) return;
    if (lane >= qc && lane < qc + k) qid = a0 + __fns(mask, 0, static_cast<int>(lane - qc + 1));
    if (qc + k < 32) {
        qc += k;
        return;
    }
    walk(32u);
    const uint32_t rem = qc + k - 32;
    if (lane < rem) qid = a0 + __fns(mask, 0, static_cast<int>(32 - qc + lane + 1));
    qc = rem;
}

}  // namespace amber
