// Shared device helpers for libfagp_b200 (sm_100a).
//
// FP64 tensor-core path on B200: tcgen05 has no f64 kind, so the FP64 MMA is the
// warp-level mma.sync.m8n8k4.f64, which lowers to SASS DMMA.8x8x4 (256 FMA/instr).
// Measured on the pool's B200s: 37.06 TF/s register-only (profiles/fp64_peak_r01.json),
// i.e. one DMMA per 16 clocks per SM sub-partition at 1965 MHz.
#pragma once

#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>

#include "../../include/fagp_b200.h"

// FAGP_DEBUG=1 in the environment prints the CUDA error behind an FAGP_ECUDA status.
#define FAGP_CUDA_TRY(expr)                                    \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::fagp::cuda_fail(_e, __FILE__, __LINE__); \
  } while (0)

#define FAGP_LAUNCH_CHECK()                                    \
  do {                                                         \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return ::fagp::cuda_fail(_e, __FILE__, __LINE__); \
  } while (0)

namespace fagp {

__host__ inline int cuda_fail(cudaError_t e, const char* file, int line) {
  const char* dbg = getenv("FAGP_DEBUG");
  if (dbg && dbg[0] == '1') fprintf(stderr, "[fagp] %s:%d: %s\n", file, line, cudaGetErrorString(e));
  return FAGP_ECUDA;
}

constexpr int kNumSMs = 148;  // B200; only used as a grid-sizing hint (queried at run time)

constexpr int kMaxDevices = 64;  // per-device caches of device properties / occupancies

__host__ inline int num_sms() {
  static int cached[kMaxDevices];  // per device (a device property; 0 = not read yet)
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return kNumSMs;
  if (dev < kMaxDevices && cached[dev] > 0) return cached[dev];
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = kNumSMs;
  if (dev < kMaxDevices) cached[dev] = n;
  return n;
}

// D += A(8x4) * B(4x8) on the FP64 tensor pipe.  Fragment layout (lane = 0..31):
//   a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
//   d0,d1 = D[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Integer test for Inf/NaN (exponent all ones); keeps the FP64 pipe free.
__device__ __forceinline__ bool not_finite(double v) {
  return ((__double2hiint(v) >> 20) & 0x7ff) == 0x7ff;
}

__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Basis table accessors (layout documented in include/fagp_b200.h).
struct BasisView {
  int p, M;
  int64_t m;
  const double* table;
  __host__ __device__ const double* rho_beta() const { return table; }
  __host__ __device__ const double* neg_delta2() const { return table + p; }
  __host__ __device__ const double* sqrt_beta() const { return table + 2 * p; }
  __host__ __device__ const double* lam1d() const { return table + 3 * p; }
  // modal linearisation coefficients V[pi][k] (P x L, pair pi = (a <= b) a-major):
  // h_a(z) h_b(z) = sum_k V[pi][k] h_k(sqrt2 z)  (see modal.cu)
  __host__ __device__ const double* modal() const { return table + 3 * p + p * M; }
};

inline int check_basis(const fagp_basis* b) {
  if (b == nullptr || b->table == nullptr) return FAGP_EINVAL;
  if (b->p < 1 || b->M < 1) return FAGP_EINVAL;
  if (b->p > FAGP_MAX_P) return FAGP_EUNSUPPORTED;
  int64_t m = 1;
  for (int d = 0; d < b->p; ++d) {
    m *= b->M;
    if (m > (int64_t(1) << 31)) return FAGP_EUNSUPPORTED;
  }
  if (m != b->m) return FAGP_EINVAL;
  return FAGP_OK;
}

inline BasisView view(const fagp_basis* b) { return BasisView{b->p, b->M, b->m, b->table}; }

template <class T>
__host__ __device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }
template <class T>
__host__ __device__ __forceinline__ T tmax(T a, T b) { return a < b ? b : a; }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// The modal (Hermite-linearised) path runs for 2 <= p <= 8 while the pair-indexed
// intermediates (P^p entries, P = M(M+1)/2) fit 31-bit indices; p = 1 uses the direct SYRK.
__host__ __device__ inline bool modal_on(int p, int M) {
  if (p < 2 || p > 8 || M < 1) return false;
  const int64_t P = int64_t(M) * (M + 1) / 2;
  int64_t h = 1;
  for (int d = 0; d < p; ++d) h *= P;
  return h < (int64_t(1) << 31);
}
__host__ __device__ __forceinline__ int modal_L(int M) { return 2 * M - 1; }

// Table row layout (fagp_basis_eval), every section 16-byte aligned for cp.async:
//   [phi_{d,i} (d < p, i < M) | r | 1.0 | 0.0 | pad]                 width table_gbase = round_up(pM + 3, 2)
//   [g_{d,k} (d < p, k < L = 2M-1) | 1.0 | 0.0 | pad]                 modal path only, width round_up(pL + 2, 2)
// g_{d,k}(x) = beta_d exp(-2 delta2_d x^2) h_k(sqrt2 rho_d beta_d x) spans every product
// phi_{d,a} phi_{d,b} (modal.cu).
__host__ __device__ __forceinline__ int table_gbase(int p, int M) { return (p * M + 3 + 1) & ~1; }
__host__ __device__ __forceinline__ int table_gsec(int p, int M) { return (p * modal_L(M) + 2 + 1) & ~1; }
__host__ __device__ __forceinline__ int table_width(int p, int M) {
  return table_gbase(p, M) + (modal_on(p, M) ? table_gsec(p, M) : 0);
}
__host__ __device__ __forceinline__ int table_col_r(int pM) { return pM; }
__host__ __device__ __forceinline__ int table_col_one(int pM) { return pM + 1; }
__host__ __device__ __forceinline__ int table_col_zero(int pM) { return pM + 2; }

__device__ __forceinline__ void raise_flag(uint32_t* flags, uint32_t bit) {
  if (flags) atomicOr(flags, bit);
}

}  // namespace fagp
