// Stage (4) of the path: predictive mean and variance for N* test rows.
//   mean_i = c + phi*_i . w                        posterior.py:247
//   var_i  = sigma2 * || V phi*_i ||^2             diag of posterior.py:249-263 (cli.py:222)
// with V = L^{-1} diag(s) lower triangular, so Z = Phi* V^T touches only the upper
// triangle of V^T; the operand P = [V^T | w] (fagp_factor) puts w in column m so the
// mean falls out of the same contraction.
//
// K5 (predict_kernel_fast<P>): one CTA per 128 test rows, whose table rows are staged in
// shared memory once.  The CTA walks the flattened sequence of (output column tile c,
// K chunk) steps -- column tile c only needs K rows j < min(m, 128 (c+1)), the triangle --
// and for every step it prefetches the next step's P chunk [32 x 128] with cp.async and
// generates the next step's Phi* chunk [128 x 32] (product of p table entries, reference
// order, branch-free: columns j >= m gather the table's 0.0 entry) interleaved with its
// own DMMA k-loop (8 warps, 64x32 warp tiles).  Tile epilogues fold squares of Z into
// per-row registers; the final lane/warp reduction is in a fixed order (deterministic,
// no atomics) and each row's mean and var are single coalesced 8-byte stores.  A
// non-finite phi*_i shows up as a non-finite mean_i / var_i and raises the flag.
#include "common.cuh"

namespace fagp {
namespace pred {

constexpr int BM = 128, BN = 128, BK = 32, NT = 256;
constexpr int ASP = BK + 4;  // 36 % 16 == 4
constexpr int BSP = BN + 4;  // 132 % 16 == 4
constexpr int WM = 64, WN = 32, FM = WM / 8, FN = WN / 8;
constexpr int A_STAGE = BM * ASP, B_STAGE = BK * BSP;
constexpr int OP_COL_ALIGN = 128;
constexpr size_t BASE_SMEM = size_t(2) * (A_STAGE + B_STAGE) * sizeof(double) + size_t(4) * BM * sizeof(double);
constexpr size_t kMaxSmem = 227 * 1024;
inline size_t fast_smem_bytes(int W) { return BASE_SMEM + size_t(BM) * W * sizeof(double); }

// Digit offsets of K column j for factor d (feature), or the zero entry for j >= m.
__device__ __forceinline__ int kcol_offset(int64_t j, int64_t m, int M, int pM, int d, int p) {
  if (j < m) {
    int64_t q = j;
    for (int e = p - 1; e > d; --e) q /= M;
    return d * M + int(q % M);
  }
  return d == 0 ? table_col_zero(pM) : table_col_one(pM);
}

// fold column tile c0 of the accumulators into the per-row sums / mean registers
__device__ __forceinline__ void fold_tile(const double (&acc)[FM][FN][2], double (&vsum)[FM], double (&mval)[FM],
                                          int64_t c0, int64_t m, int wj, int lane) {
#pragma unroll
  for (int t = 0; t < FN; ++t) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t k = c0 + wj * WN + t * 8 + 2 * (lane & 3) + e;
      if (k < m) {
#pragma unroll
        for (int s = 0; s < FM; ++s) vsum[s] = fma(acc[s][t][e], acc[s][t][e], vsum[s]);
      } else if (k == m) {
#pragma unroll
        for (int s = 0; s < FM; ++s) mval[s] = acc[s][t][e];
      }
    }
  }
}

// Final fixed-order reduction: lanes sharing a row, then the 4 warp columns.
__device__ __forceinline__ void finish_rows(double (&vsum)[FM], const double (&mval)[FM], double* red, double* mbuf,
                                            int64_t m, int wi, int wj, int lane, int tid, int64_t row0, int64_t Ns,
                                            double sigma2, double mean_const, double* mean, double* var,
                                            uint32_t* flags) {
  const int mwarp = int((m % BN) / WN);
  const int mlane = int((m % WN) % 8) / 2;
#pragma unroll
  for (int s = 0; s < FM; ++s) {
    double v = vsum[s];
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    vsum[s] = v;
  }
  if ((lane & 3) == 0) {
#pragma unroll
    for (int s = 0; s < FM; ++s) red[wj * BM + wi * WM + s * 8 + (lane >> 2)] = vsum[s];
  }
  if (wj == mwarp && (lane & 3) == mlane) {
#pragma unroll
    for (int s = 0; s < FM; ++s) mbuf[wi * WM + s * 8 + (lane >> 2)] = mval[s];
  }
  __syncthreads();
  if (tid < BM) {
    const int64_t row = row0 + tid;
    if (row < Ns) {
      const double tot = ((red[tid] + red[BM + tid]) + red[2 * BM + tid]) + red[3 * BM + tid];
      const double vv = sigma2 * tot, mm = mean_const + mbuf[tid];
      if (var) var[row] = vv;
      mean[row] = mm;
      if (not_finite(vv) || not_finite(mm)) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
    }
  }
}

template <int P>
__global__ void __launch_bounds__(NT, 1)
predict_kernel_fast(const double* __restrict__ Ts, int64_t Ns, BasisView b, const double* __restrict__ Pop,
                    int64_t pc, double sigma2, double mean_const, double* __restrict__ mean,
                    double* __restrict__ var, uint32_t* flags) {
  extern __shared__ double sm[];
  double* As = sm;                             // [2][BM][ASP]
  double* Bs = sm + 2 * A_STAGE;               // [2][BK][BSP]
  double* red = sm + 2 * (A_STAGE + B_STAGE);  // [4][BM]
  const int M = b.M, pM = P * M, W = table_width(P, M);
  double* tsm = red + 4 * BM;  // [BM][W]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = warp / 4, wj = warp % 4;
  const int64_t row0 = int64_t(blockIdx.x) * BM;
  const int64_t m = b.m;
  const int Tn = int(ceil_div(m + 1, BN));
  {
    const int nd = int(tmin<int64_t>(BM, Ns - row0)) * W;
    const double* src = Ts + row0 * W;
    for (int i = tid; i < nd / 2; i += NT) cp_async_16(tsm + 2 * i, src + 2 * i);
    for (int i = nd + tid; i < BM * W; i += NT) tsm[i] = 0.0;  // rows past N*
    cp_async_commit();
  }
  const int gk = tid % BK, gr0 = tid / BK;  // generator: K column gk, rows gr0 + 8 q, q < 16

  auto nk_of = [&](int c) { return int(round_up(tmin<int64_t>(m, int64_t(c) * BN + BN), BK) / BK); };
  auto offsets = [&](int64_t j0, int (&off)[P]) {
#pragma unroll
    for (int d = 0; d < P; ++d) off[d] = kcol_offset(j0 + gk, m, M, pM, d, P);
  };
  auto gen_rows = [&](int stage, const int (&off)[P], int q0) {
    double* dst = As + stage * A_STAGE + gk;
#pragma unroll
    for (int qi = 0; qi < 2; ++qi) {
      const int r = gr0 + 8 * (q0 + qi);
      const double* Tr = tsm + r * W;
      double v = Tr[off[0]];
#pragma unroll
      for (int d = 1; d < P; ++d) v = __dmul_rn(v, Tr[off[d]]);
      dst[r * ASP] = v;
    }
  };
  auto load_b = [&](int stage, int64_t j0, int64_t c0) {
    double* dst = Bs + stage * B_STAGE;
#pragma unroll
    for (int q = 0; q < (BK * BN / 2) / NT; ++q) {
      const int e = tid + q * NT;
      const int k = e / (BN / 2), n2 = e % (BN / 2);
      cp_async_16(dst + k * BSP + 2 * n2, Pop + (j0 + k) * pc + c0 + 2 * n2);
    }
    cp_async_commit();
  };

  double vsum[FM], mval[FM];
#pragma unroll
  for (int s = 0; s < FM; ++s) vsum[s] = mval[s] = 0.0;
  double acc[FM][FN][2];
#pragma unroll
  for (int s = 0; s < FM; ++s)
#pragma unroll
    for (int t = 0; t < FN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;

  cp_async_wait<0>();
  __syncthreads();
  load_b(0, 0, 0);
  {
    int off[P];
    offsets(0, off);
#pragma unroll
    for (int q0 = 0; q0 < 16; q0 += 2) gen_rows(0, off, q0);
  }
  cp_async_wait<0>();
  __syncthreads();

  int c = 0, n = 0, nk = nk_of(0), buf = 0;
  while (true) {
    int c2 = c, n2 = n + 1;
    if (n2 == nk) {
      c2 = c + 1;
      n2 = 0;
    }
    const bool has_next = c2 < Tn;
    if (has_next) load_b(buf ^ 1, int64_t(n2) * BK, int64_t(c2) * BN);
    int off[P];
    offsets(int64_t(n2) * BK, off);  // past the last step: harmless garbage into the spare buffer
    const double* Ab = As + buf * A_STAGE + (wi * WM + (lane >> 2)) * ASP + (lane & 3);
    const double* Bb = Bs + buf * B_STAGE + (lane & 3) * BSP + wj * WN + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[FM], bb[FN];
#pragma unroll
      for (int s = 0; s < FM; ++s) a[s] = Ab[s * 8 * ASP + kk * 4];
#pragma unroll
      for (int t = 0; t < FN; ++t) bb[t] = Bb[kk * 4 * BSP + t * 8];
#pragma unroll
      for (int s = 0; s < FM; ++s)
#pragma unroll
        for (int t = 0; t < FN; ++t) dmma_8x8x4(acc[s][t][0], acc[s][t][1], a[s], bb[t]);
      gen_rows(buf ^ 1, off, kk * 2);
    }
    cp_async_wait<0>();
    __syncthreads();
    if (n2 == 0 || !has_next) {
      fold_tile(acc, vsum, mval, int64_t(c) * BN, m, wj, lane);
#pragma unroll
      for (int s = 0; s < FM; ++s)
#pragma unroll
        for (int t = 0; t < FN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;
    }
    if (!has_next) break;
    c = c2;
    n = n2;
    nk = nk_of(c);
    buf ^= 1;
  }
  finish_rows(vsum, mval, red, As, m, wi, wj, lane, tid, row0, Ns, sigma2, mean_const, mean, var, flags);
}

// Generic K5 (p > 8 or table rows too wide to stage): runtime p, table through L1, one
// barrier-separated generation phase per step.
__global__ void __launch_bounds__(NT, 1)
predict_kernel_generic(const double* __restrict__ Ts, int64_t Ns, BasisView b, const double* __restrict__ Pop,
                       int64_t pc, double sigma2, double mean_const, double* __restrict__ mean,
                       double* __restrict__ var, uint32_t* flags) {
  extern __shared__ double sm[];
  double* As = sm;
  double* Bs = sm + A_STAGE;
  double* red = sm + 2 * (A_STAGE + B_STAGE);
  const int M = b.M, p = b.p, pM = p * M, W = table_width(p, M);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = warp / 4, wj = warp % 4;
  const int64_t row0 = int64_t(blockIdx.x) * BM;
  const int64_t m = b.m;
  const int Tn = int(ceil_div(m + 1, BN));
  const int gk = tid % BK, gr0 = tid / BK;
  double vsum[FM], mval[FM];
#pragma unroll
  for (int s = 0; s < FM; ++s) vsum[s] = mval[s] = 0.0;
  for (int c = 0; c < Tn; ++c) {
    const int64_t c0 = int64_t(c) * BN;
    const int nk = int(round_up(tmin<int64_t>(m, c0 + BN), BK) / BK);
    double acc[FM][FN][2];
#pragma unroll
    for (int s = 0; s < FM; ++s)
#pragma unroll
      for (int t = 0; t < FN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;
    for (int n = 0; n < nk; ++n) {
      const int64_t j0 = int64_t(n) * BK;
      for (int q = 0; q < (BK * BN / 2) / NT; ++q) {
        const int e = tid + q * NT;
        const int k = e / (BN / 2), n2 = e % (BN / 2);
        cp_async_16(Bs + k * BSP + 2 * n2, Pop + (j0 + k) * pc + c0 + 2 * n2);
      }
      cp_async_commit();
      int off[FAGP_MAX_P];
      for (int d = 0; d < p; ++d) off[d] = kcol_offset(j0 + gk, m, M, pM, d, p);
      for (int r = gr0; r < BM; r += NT / BK) {
        const int64_t row = row0 + r;
        double v = 0.0;
        if (row < Ns) {
          const double* Tr = Ts + row * W;
          v = __ldg(Tr + off[0]);
          for (int d = 1; d < p; ++d) v = __dmul_rn(v, __ldg(Tr + off[d]));
        }
        As[r * ASP + gk] = v;
      }
      cp_async_wait<0>();
      __syncthreads();
      const double* Ab = As + (wi * WM + (lane >> 2)) * ASP + (lane & 3);
      const double* Bb = Bs + (lane & 3) * BSP + wj * WN + (lane >> 2);
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        double a[FM], bb[FN];
#pragma unroll
        for (int s = 0; s < FM; ++s) a[s] = Ab[s * 8 * ASP + kk * 4];
#pragma unroll
        for (int t = 0; t < FN; ++t) bb[t] = Bb[kk * 4 * BSP + t * 8];
#pragma unroll
        for (int s = 0; s < FM; ++s)
#pragma unroll
          for (int t = 0; t < FN; ++t) dmma_8x8x4(acc[s][t][0], acc[s][t][1], a[s], bb[t]);
      }
      __syncthreads();
    }
    fold_tile(acc, vsum, mval, c0, m, wj, lane);
  }
  finish_rows(vsum, mval, red, As, m, wi, wj, lane, tid, row0, Ns, sigma2, mean_const, mean, var, flags);
}

}  // namespace pred
}  // namespace fagp

using namespace fagp;

extern "C" {

int fagp_predict(const double* Ts, int64_t Ns, const fagp_basis* basis, const double* predict_op, double sigma2,
                 double mean_const, double* mean, double* var, uint32_t* flags, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (Ns < 0 || predict_op == nullptr || (Ns > 0 && (Ts == nullptr || mean == nullptr))) return FAGP_EINVAL;
  if (Ns == 0) return FAGP_OK;
  const int64_t pc = round_up(basis->m + 1, pred::OP_COL_ALIGN);
  const int W = table_width(basis->p, basis->M);
  const int64_t grid = ceil_div(Ns, pred::BM);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t fsmem = pred::fast_smem_bytes(W);
  if (basis->p <= 8 && fsmem <= pred::kMaxSmem) {
    auto launch = [&](auto kern) -> int {
      FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(fsmem)));
      kern<<<unsigned(grid), pred::NT, fsmem, s>>>(Ts, Ns, view(basis), predict_op, pc, sigma2, mean_const, mean,
                                                   var, flags);
      return FAGP_OK;
    };
    int rc;
    switch (basis->p) {
      case 1: rc = launch(pred::predict_kernel_fast<1>); break;
      case 2: rc = launch(pred::predict_kernel_fast<2>); break;
      case 3: rc = launch(pred::predict_kernel_fast<3>); break;
      case 4: rc = launch(pred::predict_kernel_fast<4>); break;
      case 5: rc = launch(pred::predict_kernel_fast<5>); break;
      case 6: rc = launch(pred::predict_kernel_fast<6>); break;
      case 7: rc = launch(pred::predict_kernel_fast<7>); break;
      default: rc = launch(pred::predict_kernel_fast<8>); break;
    }
    if (rc) return rc;
  } else {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(pred::predict_kernel_generic, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(pred::BASE_SMEM)));
    pred::predict_kernel_generic<<<unsigned(grid), pred::NT, pred::BASE_SMEM, s>>>(
        Ts, Ns, view(basis), predict_op, pc, sigma2, mean_const, mean, var, flags);
  }
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // extern "C"
