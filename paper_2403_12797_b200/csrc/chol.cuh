// Persistent cooperative Cholesky (chol.cu).
#pragma once

#include "common.cuh"

namespace fagp {
namespace la {

// scratch doubles: diag (m) | panel buffer (32 * round_up(m, 32)) | L11^{-1} x 2 | flag
__host__ __device__ inline int64_t chol_scratch_len(int64_t m) { return m + 32 * ((m + 31) / 32 * 32) + 2 * 32 * 32 + 2; }

// Lower Cholesky in place (upper triangle zeroed), LAPACK 1-based *info on breakdown.
// FAGP_EUNSUPPORTED when the device cannot co-schedule the grid (the caller falls back).
// info_off is added to the reported breakdown column (a diagonal block of a larger matrix); the
// launch returns at once when *info is already set.
int potrf_persistent(double* A, int64_t m, int64_t lda, int* info, double* scratch, cudaStream_t s,
                     int info_off = 0);

// scratch doubles: L_kk^{-1} x 2 | panels (T blocks) | flag
// [2 L^{-1} blocks | T panels | flag + 2 barrier counters (2 doubles, zeroed per launch) |
//  SM id per CTA (kCholInvSmTab ints)]
constexpr int64_t kCholInvSmTab = 1024;
__host__ __device__ inline int64_t cholinv_scratch_len(int64_t m) {
  return int64_t(2 + (m + 31) / 32) * 32 * 32 + 2 + kCholInvSmTab / 2;
}

// Dout (ld ldd, full symmetric) = A^{-1} of the SPD m x m matrix A (overwritten) by one
// persistent kernel (Cholesky, triangular inverse into X (m x m scratch), X^T X); *info
// (device) = dpotrf's 1-based breakdown column, 0 on success (Dout untouched otherwise).
int chol_inverse_persistent(double* A, int64_t m, int64_t lda, int* info, double* scratch, double* X, double* Dout,
                            int64_t ldd, cudaStream_t s);

}  // namespace la
}  // namespace fagp
