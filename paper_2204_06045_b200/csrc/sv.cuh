// Launch interface of the QAOA state-vector oracle (sv.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace qtng {

// Device scratch bytes sv_run needs for m edges: the edge bit pairs (int2,
// first), the m per-edge results (double), then per-CTA partial sums.
size_t sv_scratch_bytes(int m);

// run_ansatz + the per-edge <Z_u Z_v> of expectation_cost on `amps` (2^n
// complex128 in HBM).  phase_bits_dev: per edge (n-1-u, n-1-v); per layer k:
// w[k] = exp(-i gamma_k), c[k] = (cos beta_k, 0), ms[k] = (0, -sin beta_k);
// amp0 = 1/sqrt(2^n).  zz_dev receives the m expectations.
cudaError_t sv_run(cudaStream_t s, double2* amps, int n, int m, const int2* phase_bits_dev,
                   int p, const double2* w, const double2* c, const double2* ms, double amp0,
                   void* scratch, double* zz_dev);

}  // namespace qtng
