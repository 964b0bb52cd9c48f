// Test pin (R1): cuRAND's own Philox4x32-10 block function, compiled for the
// HOST from the CUDA toolkit header (its NV_IS_HOST branch), exported with a
// C ABI so tests can compare the oracle's Philox against a library routine.
// Nothing here is used by the product or by the oracle.
#define QUALIFIERS static inline
#include <vector_types.h>
#include <curand_philox4x32_x.h>
extern "C" void curand_host_philox(const unsigned* ctr, const unsigned* key, unsigned* out, long n) {
  for (long i = 0; i < n; ++i) {
    uint4 c = {ctr[4*i], ctr[4*i+1], ctr[4*i+2], ctr[4*i+3]};
    uint2 k = {key[2*i], key[2*i+1]};
    uint4 r = curand_Philox4x32_10(c, k);
    out[4*i] = r.x; out[4*i+1] = r.y; out[4*i+2] = r.z; out[4*i+3] = r.w;
  }
}
