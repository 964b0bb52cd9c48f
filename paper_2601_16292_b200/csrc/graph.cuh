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

}  // namespace amber
