// solve.cu — the readout gather kernel of the step path. The time
// stepping itself (rhs, PCG, recovery) is the persistent kernel in pcg.cu.

#include "common.cuh"
#include "device.h"

namespace tcg {

// glued readout: out[e] = a_loc[src[e]] (lowest-id owner copy)
__global__ void k_gather_glued(double* out, const double* __restrict__ a_loc, const int64_t* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a_loc[src[i]];
}

}  // namespace tcg
