// Stage (1) of the path: SE Mercer eigenvalues and 1-D Hermite eigenfunctions.
//
// Follows /root/reference/pkg/src/fagp/mercer.py:
//   normalized_hermite   mercer.py:122-143   (three-term recurrence, kept in registers)
//   _phi_1d              mercer.py:276-281   (sqrt(beta) * exp((-delta2*x)*x) * h(rho*beta*x))
//   eigensystem lam      mercer.py:350-353   (tensor products, first dimension slowest)
//   lam_floored          mercer.py:259-266
//   multi_indices        mercer.py:195-216
//   _assemble_phi        mercer.py:284-292   (materialised Phi, test/API use only)
// Every multiply/subtract is issued as an explicit round-to-nearest op (__dmul_rn,
// __dsub_rn) so nvcc cannot contract it into an FMA: the result then matches numpy's
// evaluation order bit for bit except for exp(), whose CUDA and numpy-SIMD versions differ
// by at most a couple of ulps on a small fraction of arguments.
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "eigfun.cuh"

namespace fagp {

__global__ void hermite_kernel(const double* __restrict__ z, int64_t n, int count,
                               double* __restrict__ out) {
  extern __shared__ double coef[];  // [count] c1, [count] c2
  for (int k = threadIdx.x; k < count; k += blockDim.x) {
    coef[k] = herm_c1(k);
    coef[count + k] = herm_c2(k);
  }
  __syncthreads();
  const double sqrt2 = kSqrt2;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const double zr = z[r];
    double* o = out + r * count;
    double hm1 = 1.0;
    o[0] = 1.0;
    if (count > 1) {
      double h = __dmul_rn(zr, sqrt2);
      o[1] = h;
      for (int k = 1; k < count - 1; ++k) {
        // (z * c1[k]) * h_k - c2[k] * h_{k-1}
        double hn = __dsub_rn(__dmul_rn(__dmul_rn(zr, coef[k]), h), __dmul_rn(coef[count + k], hm1));
        o[k + 1] = hn;
        hm1 = h;
        h = hn;
      }
    }
  }
}

// T[r, d*M + i] = phi_{i+1}(X[r, d]) for every row r and dimension d, followed by the
// residual r = y - c (0 without y), 1.0 and 0.0 (see table_width in common.cuh).
// One thread per (row, dim); rows are staged through shared memory so the table rows
// are written to HBM with coalesced 8-byte stores.
// Modal path (2 <= p <= 8): the g-section g_{d,k} = beta_d exp(-2 delta2_d x^2) h_k(sqrt2 z),
// k < L = 2M - 1, then 1.0 and 0.0 (modal.cu).
__global__ void basis_eval_kernel(const double* __restrict__ X, int64_t N, BasisView b,
                                  const double* __restrict__ y, double mean_const,
                                  double* __restrict__ T, uint32_t* flags, int rows_per_cta) {
  extern __shared__ double sm[];
  const int M = b.M, p = b.p, pM = p * M, W = table_width(p, M);
  const bool modal = modal_on(p, M);
  const int L = modal_L(M), G0 = table_gbase(p, M), KC = modal ? L : M;
  double* c1 = sm;              // [KC]
  double* c2 = sm + KC;         // [KC]
  double* stage = sm + 2 * KC;  // [rows_per_cta * W]
  for (int k = threadIdx.x; k < KC; k += blockDim.x) {
    c1[k] = herm_c1(k);
    c2[k] = herm_c2(k);
  }
  const int64_t row0 = int64_t(blockIdx.x) * rows_per_cta;
  const int nrows = int(tmin<int64_t>(rows_per_cta, N - row0));
  __syncthreads();
  bool bad_x = false;
  for (int task = threadIdx.x; task < nrows * p; task += blockDim.x) {
    const int rl = task / p, d = task - rl * p;
    const double x = X[(row0 + rl) * p + d];
    bad_x |= not_finite(x);
    eval_phi_dim(x, b, d, c1, c2, stage + rl * W + d * M);
    if (modal) eval_g_dim(x, b, d, c1, c2, stage + rl * W + G0 + d * L);
  }
  for (int rl = threadIdx.x; rl < nrows; rl += blockDim.x) {
    double* o = stage + rl * W;
    o[table_col_r(pM)] = y ? __dsub_rn(y[row0 + rl], mean_const) : 0.0;  // r = y - c (posterior.py:229)
    o[table_col_one(pM)] = 1.0;
    o[table_col_zero(pM)] = 0.0;
    for (int c = pM + 3; c < G0; ++c) o[c] = 0.0;
    if (modal) {
      o[G0 + p * L] = 1.0;
      o[G0 + p * L + 1] = 0.0;
      for (int c = G0 + p * L + 2; c < W; ++c) o[c] = 0.0;
    }
  }
  __syncthreads();
  double* dst = T + row0 * W;
  for (int i = threadIdx.x; i < nrows * W; i += blockDim.x) dst[i] = stage[i];
  if (bad_x) raise_flag(flags, FAGP_FLAG_X_NONFINITE);
}

__global__ void set_residual_kernel(double* __restrict__ T, int64_t N, int pM, int W, const double* __restrict__ y,
                                    double mean_const) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < N; r += int64_t(gridDim.x) * blockDim.x)
    T[r * W + table_col_r(pM)] = y ? __dsub_rn(y[r], mean_const) : 0.0;
}

// Phi[r, j] = ((T[r, i_0] * T[r, M + i_1]) * T[r, 2M + i_2]) * ...  with j's mixed-radix
// digits i_d (first dimension slowest), matching _assemble_phi's broadcast order.
__global__ void features_kernel(const double* __restrict__ T, int64_t N, BasisView b,
                                double* __restrict__ phi, uint32_t* flags) {
  const int64_t m = b.m;
  const int M = b.M, p = b.p, W = table_width(p, M);
  bool bad = false;
  const int64_t total = N * m;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / m;
    int64_t j = e - r * m;
    const double* Tr = T + r * W;
    // digits from the last (fastest) dimension up
    int dig[FAGP_MAX_P];
    for (int d = p - 1; d >= 0; --d) {
      dig[d] = int(j % M);
      j /= M;
    }
    double v = Tr[dig[0]];
    for (int d = 1; d < p; ++d) v = __dmul_rn(v, Tr[d * M + dig[d]]);
    bad |= not_finite(v);
    phi[e] = v;
  }
  if (bad) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
}

// Smallest linear index r*m + j with a non-finite Phi[r, j]; int64 max when none.
__global__ void find_nonfinite_kernel(const double* __restrict__ T, int64_t N, BasisView b,
                                      unsigned long long* first) {
  const int64_t m = b.m;
  const int M = b.M, p = b.p, W = table_width(p, M);
  const int64_t total = N * m;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / m;
    int64_t j = e - r * m;
    const double* Tr = T + r * W;
    int dig[FAGP_MAX_P];
    for (int d = p - 1; d >= 0; --d) {
      dig[d] = int(j % M);
      j /= M;
    }
    double v = Tr[dig[0]];
    for (int d = 1; d < p; ++d) v = __dmul_rn(v, Tr[d * M + dig[d]]);
    if (not_finite(v)) atomicMin(first, (unsigned long long)e);
  }
}

__global__ void finish_first_kernel(int64_t* first) {
  if (*reinterpret_cast<unsigned long long*>(first) == ~0ull) *first = -1;
}

// lam_j = ((1*lam1[i_0]) * lam2[i_1]) * ...; floored = max(lam, max(lam) * floor_rel);
// s = sqrt(floored).  One CTA: m is at most a few 1e4 and this runs once per fit.
__global__ void eigenvalues_kernel(BasisView b, double floor_rel, double* lam, double* lam_floored,
                                   double* sqrt_lam) {
  __shared__ double red[1024];
  const int64_t m = b.m;
  const int M = b.M, p = b.p;
  const double* l1 = b.lam1d();
  double mx = -1.0;
  bool nan_seen = false;
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    int64_t q = j;
    int dig[FAGP_MAX_P];
    for (int d = p - 1; d >= 0; --d) {
      dig[d] = int(q % M);
      q /= M;
    }
    double v = __dmul_rn(1.0, l1[dig[0]]);
    for (int d = 1; d < p; ++d) v = __dmul_rn(v, l1[d * M + dig[d]]);
    if (lam) lam[j] = v;
    if (v != v) nan_seen = true;
    mx = v > mx ? v : mx;
  }
  red[threadIdx.x] = nan_seen ? __longlong_as_double(0x7ff8000000000000LL) : mx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      double a = red[threadIdx.x], c = red[threadIdx.x + s];
      red[threadIdx.x] = (a != a || c != c) ? (a != a ? a : c) : (a > c ? a : c);
    }
    __syncthreads();
  }
  const double floor_v = __dmul_rn(red[0], floor_rel);  // lam.max() * floor_rel
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    int64_t q = j;
    int dig[FAGP_MAX_P];
    for (int d = p - 1; d >= 0; --d) {
      dig[d] = int(q % M);
      q /= M;
    }
    double v = __dmul_rn(1.0, l1[dig[0]]);
    for (int d = 1; d < p; ++d) v = __dmul_rn(v, l1[d * M + dig[d]]);
    // np.maximum propagates NaN from either side
    double f = (v != v || floor_v != floor_v) ? (v != v ? v : floor_v) : (v > floor_v ? v : floor_v);
    if (lam_floored) lam_floored[j] = f;
    if (sqrt_lam) sqrt_lam[j] = __dsqrt_rn(f);
  }
}

}  // namespace fagp

using namespace fagp;

extern "C" {

int fagp_abi_version(void) { return FAGP_ABI_VERSION; }

const char* fagp_strerror(int status) {
  switch (status) {
    case FAGP_OK: return "ok";
    case FAGP_EINVAL: return "invalid argument";
    case FAGP_EBUDGET: return "size exceeds the configured budget";
    case FAGP_ENOTPD: return "matrix is not positive definite";
    case FAGP_ENONFINITE: return "non-finite feature value";
    case FAGP_ECUDA: return "CUDA runtime error";
    case FAGP_EWORKSPACE: return "workspace too small";
    case FAGP_EUNSUPPORTED: return "shape not supported by the kernels";
    default: return "unknown status";
  }
}

int64_t fagp_basis_table_len(int32_t p, int32_t M) {
  if (p < 1 || M < 1) return -1;
  return int64_t(3) * p + int64_t(p) * M + int64_t(M) * (M + 1) / 2 * (2 * int64_t(M) - 1);
}

// V[pi][k] with h_a(z) h_b(z) = sum_k V[pi][k] h_k(sqrt2 z) for every pair pi = (a <= b)
// (a-major), h = the reference's normalised Hermite polynomials (mercer.py:122-143).
// Built from the three-term recurrence lifted to coefficient space, in long double:
//   z h_k(sqrt2 z) = (sqrt(k+1) h_{k+1}(sqrt2 z) + sqrt(k) h_{k-1}(sqrt2 z)) / 2
//   h_{a+1}(z) h_b(z) = sqrt(2/(a+1)) z h_a(z) h_b(z) - sqrt(a/(a+1)) h_{a-1}(z) h_b(z)
// |V| <= 1 (an orthonormal expansion of a product of orthonormal Hermite functions).
int fagp_modal_coeffs(int32_t M, double* out) {
  if (M < 1 || out == nullptr) return FAGP_EINVAL;
  const int L = 2 * M - 1;
  std::vector<long double> V(size_t(M) * M * L, 0.0L), z(L);
  auto at = [&](int a, int b) { return V.data() + (size_t(a) * M + b) * L; };
  auto times_z = [&](const long double* v, long double* o) {
    for (int k = 0; k < L; ++k) o[k] = 0.0L;
    for (int k = 0; k < L; ++k) {
      if (v[k] == 0.0L) continue;
      if (k + 1 < L) o[k + 1] += v[k] * sqrtl((long double)(k + 1)) / 2.0L;
      if (k > 0) o[k - 1] += v[k] * sqrtl((long double)k) / 2.0L;
    }
  };
  at(0, 0)[0] = 1.0L;
  for (int b = 0; b + 1 < M; ++b) {
    times_z(at(0, b), z.data());
    const long double c1 = sqrtl(2.0L / (b + 1)), c2 = sqrtl((long double)b / (b + 1));
    for (int k = 0; k < L; ++k) at(0, b + 1)[k] = c1 * z[k] - (b > 0 ? c2 * at(0, b - 1)[k] : 0.0L);
  }
  for (int a = 0; a + 1 < M; ++a) {
    const long double c1 = sqrtl(2.0L / (a + 1)), c2 = sqrtl((long double)a / (a + 1));
    for (int b = 0; b < M; ++b) {
      times_z(at(a, b), z.data());
      for (int k = 0; k < L; ++k) at(a + 1, b)[k] = c1 * z[k] - (a > 0 ? c2 * at(a - 1, b)[k] : 0.0L);
    }
  }
  int64_t pi = 0;
  for (int a = 0; a < M; ++a)
    for (int b = a; b < M; ++b, ++pi)
      for (int k = 0; k < L; ++k) out[pi * L + k] = double(at(a, b)[k]);
  return FAGP_OK;
}

int fagp_multi_indices(int32_t M, int32_t p, int64_t* out) {
  if (M < 1 || p < 1 || out == nullptr) return FAGP_EINVAL;
  int64_t m = 1;
  for (int d = 0; d < p; ++d) {
    m *= M;
    if (m > (int64_t(1) << 40)) return FAGP_EUNSUPPORTED;
  }
  for (int64_t j = 0; j < m; ++j) {
    int64_t q = j;
    for (int d = p - 1; d >= 0; --d) {
      out[j * p + d] = 1 + q % M;
      q /= M;
    }
  }
  return FAGP_OK;
}

int fagp_read_flags(uint32_t* flags_dev, uint32_t* flags_host, void* stream) {
  if (flags_dev == nullptr || flags_host == nullptr) return FAGP_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FAGP_CUDA_TRY(cudaMemcpyAsync(flags_host, flags_dev, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  FAGP_CUDA_TRY(cudaStreamSynchronize(s));
  FAGP_CUDA_TRY(cudaMemsetAsync(flags_dev, 0, sizeof(uint32_t), s));
  return FAGP_OK;
}

int fagp_find_nonfinite(const double* T, int64_t N, const fagp_basis* basis, int64_t* first_dev,
                        void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (first_dev == nullptr || N < 0 || (N > 0 && T == nullptr)) return FAGP_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FAGP_CUDA_TRY(cudaMemsetAsync(first_dev, 0xff, sizeof(int64_t), s));
  if (N > 0) {
    int64_t total = N * basis->m;
    int grid = int(tmin<int64_t>(ceil_div(total, 256), 16 * num_sms()));
    find_nonfinite_kernel<<<grid, 256, 0, s>>>(T, N, view(basis), reinterpret_cast<unsigned long long*>(first_dev));
    FAGP_LAUNCH_CHECK();
  }
  finish_first_kernel<<<1, 1, 0, s>>>(first_dev);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

int fagp_eigenvalues(const fagp_basis* basis, double floor_rel, double* lam, double* lam_floored,
                     double* sqrt_lam, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  eigenvalues_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(view(basis), floor_rel, lam,
                                                                        lam_floored, sqrt_lam);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

int fagp_hermite(const double* z, int64_t n, int32_t count, double* out, void* stream) {
  if (count < 1 || n < 0 || (n > 0 && (z == nullptr || out == nullptr))) return FAGP_EINVAL;
  if (n == 0) return FAGP_OK;
  size_t smem = size_t(2) * count * sizeof(double);
  if (smem > 200 * 1024) return FAGP_EUNSUPPORTED;
  if (smem > 48 * 1024)
    FAGP_CUDA_TRY(cudaFuncSetAttribute(hermite_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int grid = int(tmin<int64_t>(ceil_div(n, 256), 4 * num_sms()));
  hermite_kernel<<<grid, 256, smem, static_cast<cudaStream_t>(stream)>>>(z, n, count, out);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

int32_t fagp_table_width(int32_t p, int32_t M) { return (p < 1 || M < 1) ? -1 : table_width(p, M); }

int fagp_set_residual(double* T, int64_t N, const fagp_basis* basis, const double* y, double mean_const,
                      void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || (N > 0 && T == nullptr)) return FAGP_EINVAL;
  if (N == 0) return FAGP_OK;
  const int pM = basis->p * basis->M;
  int grid = int(tmin<int64_t>(ceil_div(N, 256), 8 * num_sms()));
  set_residual_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(T, N, pM, table_width(basis->p, basis->M),
                                                                          y, mean_const);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

int fagp_basis_eval(const double* X, int64_t N, const fagp_basis* basis, const double* y, double mean_const,
                    double* T, uint32_t* flags, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || (N > 0 && (X == nullptr || T == nullptr))) return FAGP_EINVAL;
  if (N == 0) return FAGP_OK;
  const int64_t W = table_width(basis->p, basis->M);
  const int rows = int(tmax<int64_t>(1, tmin<int64_t>(64, (96 * 1024) / (W * 8))));
  const int KC = modal_on(basis->p, basis->M) ? modal_L(basis->M) : basis->M;
  size_t smem = (size_t(2) * KC + size_t(rows) * W) * sizeof(double);
  if (smem > 200 * 1024) return FAGP_EUNSUPPORTED;
  FAGP_CUDA_TRY(cudaFuncSetAttribute(basis_eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int64_t grid = ceil_div(N, rows);
  basis_eval_kernel<<<unsigned(grid), 256, smem, static_cast<cudaStream_t>(stream)>>>(X, N, view(basis), y,
                                                                                     mean_const, T, flags, rows);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

int fagp_features(const double* T, int64_t N, const fagp_basis* basis, double* phi, uint32_t* flags,
                  void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || (N > 0 && (T == nullptr || phi == nullptr))) return FAGP_EINVAL;
  if (N == 0) return FAGP_OK;
  int64_t total = N * basis->m;
  int grid = int(tmin<int64_t>(ceil_div(total, 256), 16 * num_sms()));
  features_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(T, N, view(basis), phi, flags);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // extern "C"
