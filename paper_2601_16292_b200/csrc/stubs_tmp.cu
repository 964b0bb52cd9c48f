#include "internal.cuh"
namespace amber {
Model* make_sir(int64_t, const amber_sir_params&, uint64_t, const amber_runtime*) { fail(AMBER_E_UNSUPPORTED, "sir: not built yet"); }
Model* make_boids(int64_t, const amber_boids_params&, uint64_t, const amber_runtime*) { fail(AMBER_E_UNSUPPORTED, "boids: not built yet"); }
void run_sweep(int64_t, const amber_sir_params&, const amber_replicate*, int64_t, int64_t, const amber_runtime*, double*, amber_sweep_stats*) { fail(AMBER_E_UNSUPPORTED, "sweep: not built yet"); }
}
