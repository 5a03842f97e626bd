// The reference's cross-check route, method="literal" (posterior.py:236-244, 256-260):
// LamBar = diag(1/lam_f) + G / sigma2 is factorized directly and the mean goes through
// t1..t5 with two Phi^T products and one Phi product over the training rows
// (fagp_phi_tmatvec / fagp_phi_matvec).  This file holds the small elementwise pieces of
// that route, each rounding exactly like the numpy expression it restates:
//   fagp_vec_op            t1 = r / sigma2, t5 = t1 - t4 / sigma2, w = lam_f * u, ...
//   fagp_lambda_bar        LamBar = 0.5 (B + B^T), B = diag(1 / lam_f) + G / sigma2
//   fagp_literal_inner     inner = sym(diag(lam_f) - lam_f[:, None] * mid * lam_f[None, :])
//   fagp_inner_operand     pair-folded predict operand from an explicit inner matrix
//   fagp_rowdot            var_i = sum_j A[i, j] B[i, j] (direct-form variance of Phi* inner Phi*^T)
#include "common.cuh"
#include "modal.cuh"

namespace fagp {
namespace lit {

__global__ void vec_op_kernel(int op, int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                              double alpha, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double v;
    switch (op) {
      case FAGP_VEC_DIV: v = __ddiv_rn(x[i], alpha); break;
      case FAGP_VEC_SUB_DIV: v = __dsub_rn(x[i], __ddiv_rn(y[i], alpha)); break;
      case FAGP_VEC_MUL: v = __dmul_rn(x[i], y[i]); break;
      case FAGP_VEC_SUB: v = __dsub_rn(x[i], y[i]); break;
      default: v = __dsub_rn(x[i], alpha); break;  // FAGP_VEC_SUB_SCALAR
    }
    out[i] = v;
  }
}

__global__ void lambda_bar_kernel(const double* __restrict__ G, const double* __restrict__ lam_f, int64_t m,
                                  double sigma2, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m * m; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / m, j = e - (e / m) * m;
    // np.diag(1 / lam) + G / sigma2, then 0.5 * (B + B^T)
    const double bij = __dadd_rn(i == j ? __ddiv_rn(1.0, lam_f[i]) : 0.0, __ddiv_rn(G[i * m + j], sigma2));
    const double bji = __dadd_rn(i == j ? __ddiv_rn(1.0, lam_f[i]) : 0.0, __ddiv_rn(G[j * m + i], sigma2));
    out[e] = __dmul_rn(0.5, __dadd_rn(bij, bji));
  }
}

__global__ void literal_inner_kernel(const double* __restrict__ mid, const double* __restrict__ lam_f, int64_t m,
                                     double* __restrict__ out) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m * m; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / m, j = e - (e / m) * m;
    const double aij = __dsub_rn(i == j ? lam_f[i] : 0.0, __dmul_rn(__dmul_rn(lam_f[i], mid[i * m + j]), lam_f[j]));
    const double aji = __dsub_rn(i == j ? lam_f[i] : 0.0, __dmul_rn(__dmul_rn(lam_f[j], mid[j * m + i]), lam_f[i]));
    out[e] = __dmul_rn(0.5, __dadd_rn(aij, aji));
  }
}

// one warp per row, fixed-order lane partials + xor tree
__global__ void rowdot_kernel(const double* __restrict__ A, const double* __restrict__ B, int64_t n, int64_t k,
                              double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x / 32;
  for (int64_t r = blockIdx.x * wpb + threadIdx.x / 32; r < n; r += int64_t(gridDim.x) * wpb) {
    double acc = 0.0;
    for (int64_t j = lane; j < k; j += 32) acc = fma(A[r * k + j], B[r * k + j], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = acc;
  }
}

inline unsigned grid_for(int64_t n) { return unsigned(tmax<int64_t>(1, tmin<int64_t>(ceil_div(n, 256), 8 * num_sms()))); }

}  // namespace lit
}  // namespace fagp

using namespace fagp;

extern "C" {

int fagp_vec_op(int32_t op, int64_t n, const double* x, const double* y, double alpha, double* out, void* stream) {
  if (op < FAGP_VEC_DIV || op > FAGP_VEC_SUB_SCALAR || n < 0) return FAGP_EINVAL;
  const bool needs_y = op == FAGP_VEC_SUB_DIV || op == FAGP_VEC_MUL || op == FAGP_VEC_SUB;
  if (n > 0 && (x == nullptr || out == nullptr || (needs_y && y == nullptr))) return FAGP_EINVAL;
  if (n == 0) return FAGP_OK;
  lit::vec_op_kernel<<<lit::grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(op, n, x, y, alpha, out);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

int fagp_lambda_bar(const double* G, const double* lam_f, int64_t m, double sigma2, double* out, void* stream) {
  if (m < 0 || (m > 0 && (G == nullptr || lam_f == nullptr || out == nullptr)) || G == out) return FAGP_EINVAL;
  if (!(sigma2 > 0.0)) return FAGP_EINVAL;
  if (m == 0) return FAGP_OK;
  lit::lambda_bar_kernel<<<lit::grid_for(m * m), 256, 0, static_cast<cudaStream_t>(stream)>>>(G, lam_f, m, sigma2,
                                                                                               out);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

int fagp_literal_inner(const double* mid, const double* lam_f, int64_t m, double* inner, void* stream) {
  if (m < 0 || (m > 0 && (mid == nullptr || lam_f == nullptr || inner == nullptr)) || mid == inner)
    return FAGP_EINVAL;
  if (m == 0) return FAGP_OK;
  lit::literal_inner_kernel<<<lit::grid_for(m * m), 256, 0, static_cast<cudaStream_t>(stream)>>>(mid, lam_f, m,
                                                                                                  inner);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

size_t fagp_inner_operand_workspace_size(const fagp_basis* basis) {
  if (check_basis(basis) != FAGP_OK || !modal::enabled(basis->p, basis->M)) return 0;
  return size_t(modal::scratch_len(basis)) * sizeof(double);
}

int fagp_inner_operand(const double* inner, const double* w, const fagp_basis* basis, double* predict_op,
                       void* workspace, size_t workspace_bytes, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (!modal::enabled(basis->p, basis->M)) return FAGP_EUNSUPPORTED;  // checked first: callers probe the form
  if (inner == nullptr || w == nullptr || predict_op == nullptr) return FAGP_EINVAL;
  if (workspace == nullptr || workspace_bytes < fagp_inner_operand_workspace_size(basis)) return FAGP_EWORKSPACE;
  double* S0 = static_cast<double*>(workspace);
  double* S1 = S0 + modal::scratch_len(basis) / 2;
  return modal::build_predict_op(inner, nullptr, w, basis, predict_op, S0, S1, static_cast<cudaStream_t>(stream));
}

int fagp_rowdot(const double* A, const double* B, int64_t n, int64_t k, double* out, void* stream) {
  if (n < 0 || k < 0 || (n > 0 && (A == nullptr || B == nullptr || out == nullptr))) return FAGP_EINVAL;
  if (n == 0) return FAGP_OK;
  lit::rowdot_kernel<<<unsigned(tmax<int64_t>(1, tmin<int64_t>(ceil_div(n, 8), 16 * num_sms()))), 256, 0,
                       static_cast<cudaStream_t>(stream)>>>(A, B, n, k, out);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // extern "C"
