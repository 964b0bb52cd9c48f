// wealth.cuh -- pieces of the wealth model shared by its two scatter
// implementations (wealth.cu: packed-counter L2 atomics, also the exact replay
// path; wealth_bins.cu: range-partitioned scatter, the default on one GPU).
#pragma once

#include "internal.cuh"
#include "philox.cuh"

namespace amber {

// Per-step record (ring slot); all 64-bit for atomics.
struct WealthSlot {
    unsigned long long total, active, digest, sent, got;
};

// Range-partitioned scatter: receivers are bucketed by 2^16-agent range.
constexpr int kBinShift = 16;
constexpr int64_t kBinRange = 1ll << kBinShift;

struct BinPlan {
    int K = 0;                  // global ranges (bins) = ceil(N / 2^16)
    int k0 = 0, k_loc = 0;      // this rank's first range and range count
    uint32_t cap = 0;           // entry capacity per bin
    int tile = 0;               // agents per production tile (shared-memory staging)
    size_t prod_smem = 0, apply_smem = 0;
    int prod_grid = 0, apply_grid = 0, apply_threads = 512;
};

struct BinBuffers {
    DevBuf<uint16_t> data[2];   // [parity][K][cap] receiver offsets within the range
    DevBuf<uint32_t> cnt[2];    // [parity][K] entries produced (cursor)
    DevBuf<int> queue;          // [2] work-queue counters (production tiles, apply ranges)
};

// Plan + allocate; returns false if the range count does not fit the shared-memory staging.
bool bins_plan(Runtime& rt, int64_t n, int64_t lo, int64_t n_pad, BinPlan& plan);
void bins_allocate(Runtime& rt, const BinPlan& plan, BinBuffers& b);

struct WealthStepCfg {
    PhiloxKey key;
    int64_t n_loc, n_pad;
    unsigned long long lo, n_glob;
    int32_t amount, exclude_self;
    int digest;
};

// Step t: produce (bucket step t's receivers from w) then apply (w -> w_out).
void bins_step(Runtime& rt, Profiler& prof, const BinPlan& plan, BinBuffers& b, const WealthStepCfg& c,
               uint32_t t, const int32_t* w, int32_t* w_out, WealthSlot* slot_t, WealthSlot* slot_next);

// Fused range-binned step (wealth_fb.cu): bins written as 16-byte chunks from
// per-CTA shared-memory write-combining buffers, consumed by a per-range
// shared-memory histogram in the next launch.
struct FbPlan {
    int K = 0, k0 = 0, k_loc = 0, S = 0, grid = 0;
    uint32_t cap_lo = 0, cap_hi = 0;
    size_t smem_apply = 0, smem_prod = 0;
};

struct FbBuffers {
    DevBuf<uint16_t> data[2];  // [parity][K][cap_lo + cap_hi]
    DevBuf<uint32_t> lo[2];    // full-chunk entries per range
    DevBuf<uint32_t> hi[2];    // tail entries per range
    DevBuf<int> queue;         // [2] work-queue counters, alternated by launch
};

// Segmented-bin step (wealth_seg.cu): ranges of R agents (R a multiple of
// 8192, <= 344064, about two ranges per SM), a 4-bit shared-memory histogram
// per range, and per-(destination, producer) bin segments written from a
// per-chunk shared-memory staging area, so no global atomic per transfer.
struct SegPlan {
    int64_t R = 0;              // agents per range
    int K = 0;                  // ranges (= bins)
    int S = 0;                  // staging slots per destination per chunk
    int NT = 1024;              // threads per CTA (1024: one CTA per SM; 512: two)
    int grid = 0;               // persistent CTAs
    uint32_t cap = 0;           // entries per (destination, producer) segment
    uint32_t tcap = 0;          // overflow ("tail") entries per destination
    unsigned long long magic = 0;  // d = umulhi(r, magic) >> msh == r / R for r < 2^31
    int msh = 0;
    size_t smem = 0;
};

struct SegBuffers {
    DevBuf<uint32_t> data[2];   // [parity][K dest][K producer][cap]
    DevBuf<uint32_t> cnt[2];    // [parity][K dest][K producer] entries produced
    DevBuf<uint32_t> tail[2];   // [parity][K dest][tcap]
    DevBuf<uint32_t> tcnt[2];   // [parity][K dest]
};

bool seg_plan(Runtime& rt, int64_t n, int64_t n_loc, SegPlan& plan);
void seg_allocate(Runtime& rt, const SegPlan& plan, SegBuffers& b);
void seg_reset(Runtime& rt, SegBuffers& b);
// apply == false: produce step t_prod's bins from w_in only ("prime").
void seg_launch(Runtime& rt, Profiler& prof, const SegPlan& plan, SegBuffers& b, const WealthStepCfg& c, bool apply,
                uint32_t t_apply, uint32_t t_prod, const int32_t* w_in, int32_t* w_out, WealthSlot* slot_apply,
                WealthSlot* slot_prod, WealthSlot* slot_zero);

bool fb_plan(Runtime& rt, int64_t n, int64_t lo, int64_t n_pad, FbPlan& plan);
void fb_allocate(Runtime& rt, const FbPlan& plan, FbBuffers& b);
void fb_launch(Runtime& rt, Profiler& prof, const FbPlan& plan, FbBuffers& b, const WealthStepCfg& c, bool apply,
               uint32_t t_apply, uint32_t t_prod, const int32_t* w_in, int32_t* w_out, WealthSlot* slot_apply,
               WealthSlot* slot_prod, WealthSlot* slot_zero, int launch_parity);

}  // namespace amber
