// wealth.cuh -- the wealth model's per-step record (ring slot), shared by its
// kernels (wealth.cu) and the experimental scatters kept out of the library
// (tools/experiments/).
#pragma once

#include "internal.cuh"
#include "philox.cuh"

namespace amber {

// Per-step record (ring slot); all 64-bit for atomics.
struct WealthSlot {
    unsigned long long total, active, digest, sent, got;
};

}  // namespace amber
