// Device-side synthetic input generator (matrix.py:192-284 on the GPU).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "solver.cuh"

namespace bsel {

using BtaDevView = BtaDev;

// Fill `m` with generate_dd_bta(n, b, a, seed, dominance).
cudaError_t generate_dd_bta_device(const BtaDevView& m, uint64_t seed, double dominance, cudaStream_t s);
// m <- (m + m^H)/2 on the pattern, in place.
cudaError_t hermitianize_device(const BtaDevView& m, cudaStream_t s);

}  // namespace bsel
