// The exact dense GP on the device: the reference validates the fast
// route against exact_posterior (posterior.py:107-144), which needs the SE kernel matrix
//   K[i, j] = exp(-sum_d (eps_d (a_id - b_jd))^2)          (kernels.py:119-145 gram_matrix)
// and then a dense SPD factorisation of C = K + sigma2 I, which reuses the repo's Cholesky
// (fagp_potrf, jitter schedule on the host), cho_solve (fagp_potrs) and DMMA GEMM (fagp_dgemm).
// The accumulation over dimensions keeps the reference's order and roundings
// (t = eps * (a - b); acc += t * t), so K differs from numpy only where CUDA's exp rounds
// differently (<= 1 ulp); K(A, A) has an exactly unit diagonal as in the reference.
#include "common.cuh"

namespace fagp {
namespace exact {

constexpr int kMaxDims = 64;
struct Eps {
  double v[kMaxDims];
};

// One thread per entry, 32 x 8 threads per 32 x 32 tile (B rows staged in shared memory).
__global__ void __launch_bounds__(256) se_gram_kernel(const double* __restrict__ A, int64_t na,
                                                      const double* __restrict__ B, int64_t nb, int p, const Eps eps,
                                                      double* __restrict__ K, int64_t ldk, double diag_add) {
  const int64_t j = blockIdx.x * 32 + threadIdx.x;
  for (int64_t i = blockIdx.y * 32 + threadIdx.y; i < na && i < (int64_t(blockIdx.y) + 1) * 32; i += 8) {
    if (j >= nb) continue;
    double acc = 0.0;
    for (int d = 0; d < p; ++d) {
      const double t = __dmul_rn(eps.v[d], __dsub_rn(A[i * p + d], B[j * p + d]));
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
    double k = exp(-acc);
    if (diag_add != 0.0 && i == j) k = __dadd_rn(k, diag_add);  // K + sigma2 * np.eye(N)
    K[i * ldk + j] = k;
  }
}

}  // namespace exact
}  // namespace fagp

using namespace fagp;

extern "C" int fagp_se_gram(const double* A, int64_t na, const double* B, int64_t nb, int32_t p,
                            const double* eps_host, double diag_add, double* K, int64_t ldk, void* stream) {
  if (na < 0 || nb < 0 || p < 1 || p > exact::kMaxDims || eps_host == nullptr || ldk < nb) return FAGP_EINVAL;
  if (na == 0 || nb == 0) return FAGP_OK;
  if (A == nullptr || B == nullptr || K == nullptr) return FAGP_EINVAL;
  if (ceil_div(na, 32) > 65535) return FAGP_EUNSUPPORTED;
  exact::Eps e{};
  for (int d = 0; d < p; ++d) e.v[d] = eps_host[d];
  const dim3 grid(unsigned(ceil_div(nb, 32)), unsigned(ceil_div(na, 32)));
  exact::se_gram_kernel<<<grid, dim3(32, 8), 0, static_cast<cudaStream_t>(stream)>>>(A, na, B, nb, p, e, K, ldk,
                                                                                      diag_add);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}
