// Stage (4) of the path: predictive mean and variance for N* test rows.
//   mean_i = c + phi*_i . w                        posterior.py:247
//   var_i  = sigma2 * || V phi*_i ||^2             diag of posterior.py:249-263 (cli.py:222)
// with V = L^{-1} diag(s) lower triangular, so Z = Phi* V^T touches only the upper
// triangle of V^T; the operand P = [V^T | w] (fagp_factor) puts w in column m so the
// mean falls out of the same contraction.
//
// K5 (predict_kernel): one CTA per 128 test rows, persistent over the output column
// tiles.  For column tile c it contracts rows j < min(m, 128 (c+1)) (the triangle):
// Phi* chunks [128 x 32] are generated into shared memory from the 1-D table Ts
// (product of p entries, reference order) while the matching P chunk [32 x 128] arrives
// by cp.async; 8 warps issue mma.m8n8k4.f64 on 64x32 warp tiles.  The epilogue squares
// and sums each row's Z entries in registers across all column tiles, then reduces over
// lanes and warps in a fixed order: deterministic, no atomics, one 8-byte store per row
// per output (coalesced).
#include "common.cuh"

namespace fagp {
namespace pred {

constexpr int BM = 128, BN = 128, BK = 32, NT = 256;
constexpr int ASP = BK + 4;  // 36 % 16 == 4
constexpr int BSP = BN + 4;  // 132 % 16 == 4
constexpr int WM = 64, WN = 32, FM = WM / 8, FN = WN / 8;
constexpr int A_STAGE = BM * ASP, B_STAGE = BK * BSP;
constexpr int OP_COL_ALIGN = 128;
constexpr size_t SMEM = size_t(2) * (A_STAGE + B_STAGE) * sizeof(double) + size_t(4) * BM * sizeof(double);

__global__ void __launch_bounds__(NT, 1)
predict_kernel(const double* __restrict__ Ts, int64_t Ns, BasisView b, const double* __restrict__ P, int64_t pc,
               double sigma2, double mean_const, double* __restrict__ mean, double* __restrict__ var,
               uint32_t* flags) {
  extern __shared__ double sm[];
  double* As = sm;                         // [2][BM][ASP]
  double* Bs = sm + 2 * A_STAGE;           // [2][BK][BSP]
  double* red = sm + 2 * (A_STAGE + B_STAGE);  // [4][BM] cross-warp partial sums
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = warp / 4, wj = warp % 4;
  const int64_t row0 = int64_t(blockIdx.x) * BM;
  const int64_t m = b.m;
  const int M = b.M, p = b.p, pM = p * M;
  const int Tn = int(ceil_div(m + 1, BN));

  // generator role: column kc = tid % 32 of the chunk, rows tid/32 + 8q
  const int gk = tid % BK, gr0 = tid / BK;
  bool bad = false;

  auto gen_a = [&](int stage, int64_t j0) {
    const int64_t j = j0 + gk;
    int off[FAGP_MAX_P];
    const bool feat = j < m;
    if (feat) {
      int64_t q = j;
      for (int d = p - 1; d >= 0; --d) {
        off[d] = d * M + int(q % M);
        q /= M;
      }
    }
    double* dst = As + stage * A_STAGE + gk;
#pragma unroll 4
    for (int r = gr0; r < BM; r += NT / BK) {
      const int64_t row = row0 + r;
      double v = 0.0;
      if (feat && row < Ns) {
        const double* Tr = Ts + row * pM;
        v = __ldg(Tr + off[0]);
        for (int d = 1; d < p; ++d) v = __dmul_rn(v, __ldg(Tr + off[d]));
        bad |= not_finite(v);
      }
      dst[r * ASP] = v;
    }
  };
  auto load_b = [&](int stage, int64_t j0, int64_t c0) {
    double* dst = Bs + stage * B_STAGE;
    // BK x BN doubles = 2048 16-byte copies, 8 per thread
#pragma unroll
    for (int q = 0; q < (BK * BN / 2) / NT; ++q) {
      const int e = tid + q * NT;
      const int k = e / (BN / 2), n2 = e % (BN / 2);
      cp_async_16(dst + k * BSP + 2 * n2, P + (j0 + k) * pc + c0 + 2 * n2);
    }
    cp_async_commit();
  };

  double vsum[FM];
#pragma unroll
  for (int s = 0; s < FM; ++s) vsum[s] = 0.0;
  double mval[FM];
#pragma unroll
  for (int s = 0; s < FM; ++s) mval[s] = 0.0;

  for (int c = 0; c < Tn; ++c) {
    const int64_t c0 = int64_t(c) * BN;
    const int64_t kend = round_up(tmin<int64_t>(m, c0 + BN), BK);
    const int nk = int(kend / BK);
    double acc[FM][FN][2];
#pragma unroll
    for (int s = 0; s < FM; ++s)
#pragma unroll
      for (int t = 0; t < FN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;

    load_b(0, 0, c0);
    gen_a(0, 0);
    cp_async_wait<0>();
    __syncthreads();
    for (int n = 0; n < nk; ++n) {
      const int cur = n & 1;
      if (n + 1 < nk) {
        load_b(cur ^ 1, int64_t(n + 1) * BK, c0);
        gen_a(cur ^ 1, int64_t(n + 1) * BK);
      }
      const double* Ab = As + cur * A_STAGE + (wi * WM + (lane >> 2)) * ASP + (lane & 3);
      const double* Bb = Bs + cur * B_STAGE + (lane & 3) * BSP + wj * WN + (lane >> 2);
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
      cp_async_wait<0>();
      __syncthreads();
    }
    // epilogue for this column tile: squares of Z[:, k < m], mean from column m
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

  // ---- reduce the per-thread row partials: lanes sharing a row, then the 4 warp columns
  const int mwarp = int((m % BN) / WN);      // warp column holding column m of the last tile
  const int mlane = int((m % WN) % 8) / 2;   // lane & 3 holding it
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
  __syncthreads();
  double* mbuf = As;  // reuse: mean values per row
  if (wj == mwarp && (lane & 3) == mlane) {
#pragma unroll
    for (int s = 0; s < FM; ++s) mbuf[wi * WM + s * 8 + (lane >> 2)] = mval[s];
  }
  __syncthreads();
  if (tid < BM) {
    const int64_t row = row0 + tid;
    if (row < Ns) {
      const double tot = ((red[tid] + red[BM + tid]) + red[2 * BM + tid]) + red[3 * BM + tid];
      if (var) var[row] = sigma2 * tot;
      mean[row] = mean_const + mbuf[tid];
    }
  }
  if (bad) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
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
  FAGP_CUDA_TRY(cudaFuncSetAttribute(pred::predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(pred::SMEM)));
  const int64_t grid = ceil_div(Ns, pred::BM);
  pred::predict_kernel<<<unsigned(grid), pred::NT, pred::SMEM, static_cast<cudaStream_t>(stream)>>>(
      Ts, Ns, view(basis), predict_op, pc, sigma2, mean_const, mean, var, flags);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // extern "C"
