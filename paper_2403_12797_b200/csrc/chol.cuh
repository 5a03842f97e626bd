// Persistent cooperative Cholesky (chol.cu).
#pragma once

#include "common.cuh"

namespace fagp {
namespace la {

// scratch doubles: diag (m) | panel buffer (32 * round_up(m, 32)) | L11^{-1} x 2 | flag
__host__ __device__ inline int64_t chol_scratch_len(int64_t m) { return m + 32 * ((m + 31) / 32 * 32) + 2 * 32 * 32 + 2; }

// Lower Cholesky in place (upper triangle zeroed), LAPACK 1-based *info on breakdown.
// FAGP_EUNSUPPORTED when the device cannot co-schedule the grid (the caller falls back).
int potrf_persistent(double* A, int64_t m, int64_t lda, int* info, double* scratch, cudaStream_t s);

}  // namespace la
}  // namespace fagp
