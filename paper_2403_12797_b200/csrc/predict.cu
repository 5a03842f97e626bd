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
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "modal.cuh"

namespace fagp {
namespace pred {

constexpr int BK = 32;  // K rows per step (the predict operand's rows are padded to 32)
constexpr int OP_COL_ALIGN = 128;
constexpr size_t kMaxSmem = 227 * 1024;

// Tile configuration: BM test rows x BN output columns per step, warp grid WGM x WGN.
template <int BM_, int BN_, int WGM_, int WGN_, int MINB_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, WGM = WGM_, WGN = WGN_, MINB = MINB_;
  static constexpr int NT = 32 * WGM * WGN;
  static constexpr int ASP = BK + 4;  // 36 % 16 == 4
  static constexpr int BSP = BN + 4;  // % 16 == 4
  static constexpr int WM = BM / WGM, WN = BN / WGN, FM = WM / 8, FN = WN / 8;
  static constexpr int A_STAGE = BM * ASP, B_STAGE = BK * BSP;
  static constexpr int GROWS = NT / BK;             // generator row groups
  static constexpr int GPER = BM * BK / NT;         // generated elements per thread per step
  static constexpr int GPERKK = GPER / (BK / 4);    // ... per DMMA k-step
  static constexpr size_t BASE_SMEM = size_t(2) * (A_STAGE + B_STAGE) * sizeof(double) + size_t(WGN) * BM * sizeof(double);
  static_assert(BSP % 16 == 4 && ASP % 16 == 4, "fragment bank mapping");
  static_assert(GPERKK * (BK / 4) == GPER, "generation split");
};
using CfgSmall = Cfg<64, 64, 2, 2, 2>;     // 4 warps of 32x32, 2 CTAs/SM (default)
using CfgLarge = Cfg<128, 128, 2, 4, 1>;   // 8 warps of 64x32, 1 CTA/SM

template <class C>
inline size_t fast_smem_bytes(int W) { return C::BASE_SMEM + size_t(C::BM) * W * sizeof(double); }

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
template <class C>
__device__ __forceinline__ void fold_tile(const double (&acc)[C::FM][C::FN][2], double (&vsum)[C::FM],
                                          double (&mval)[C::FM], int64_t c0, int64_t m, int wj, int lane) {
#pragma unroll
  for (int t = 0; t < C::FN; ++t) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t k = c0 + wj * C::WN + t * 8 + 2 * (lane & 3) + e;
      if (k < m) {
#pragma unroll
        for (int s = 0; s < C::FM; ++s) vsum[s] = fma(acc[s][t][e], acc[s][t][e], vsum[s]);
      } else if (k == m) {
#pragma unroll
        for (int s = 0; s < C::FM; ++s) mval[s] = acc[s][t][e];
      }
    }
  }
}

// Final fixed-order reduction: lanes sharing a row, then the WGN warp columns.
template <class C>
__device__ __forceinline__ void finish_rows(double (&vsum)[C::FM], const double (&mval)[C::FM], double* red,
                                            double* mbuf, int64_t m, int wi, int wj, int lane, int tid, int64_t row0,
                                            int64_t Ns, double sigma2, double mean_const, double* mean, double* var,
                                            uint32_t* flags) {
  const int mwarp = int((m % C::BN) / C::WN);
  const int mlane = int((m % C::WN) % 8) / 2;
#pragma unroll
  for (int s = 0; s < C::FM; ++s) {
    double v = vsum[s];
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    vsum[s] = v;
  }
  if ((lane & 3) == 0) {
#pragma unroll
    for (int s = 0; s < C::FM; ++s) red[wj * C::BM + wi * C::WM + s * 8 + (lane >> 2)] = vsum[s];
  }
  if (wj == mwarp && (lane & 3) == mlane) {
#pragma unroll
    for (int s = 0; s < C::FM; ++s) mbuf[wi * C::WM + s * 8 + (lane >> 2)] = mval[s];
  }
  __syncthreads();
  for (int r = tid; r < C::BM; r += C::NT) {
    const int64_t row = row0 + r;
    if (row < Ns) {
      double tot = red[r];
#pragma unroll
      for (int w = 1; w < C::WGN; ++w) tot += red[w * C::BM + r];
      const double vv = sigma2 * tot, mm = mean_const + mbuf[r];
      if (var) var[row] = vv;
      mean[row] = mm;
      if (not_finite(vv) || not_finite(mm)) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
    }
  }
}

template <int P, class C>
__global__ void __launch_bounds__(C::NT, C::MINB)
predict_kernel_fast(const double* __restrict__ Ts, int64_t Ns, BasisView b, const double* __restrict__ Pop,
                    int64_t pc, double sigma2, double mean_const, double* __restrict__ mean,
                    double* __restrict__ var, uint32_t* flags) {
  constexpr int BM = C::BM, BN = C::BN, NT = C::NT, ASP = C::ASP, BSP = C::BSP;
  constexpr int WM = C::WM, WN = C::WN, FM = C::FM, FN = C::FN, A_STAGE = C::A_STAGE, B_STAGE = C::B_STAGE;
  extern __shared__ double sm[];
  double* As = sm;                             // [2][BM][ASP]
  double* Bs = sm + 2 * A_STAGE;               // [2][BK][BSP]
  double* red = sm + 2 * (A_STAGE + B_STAGE);  // [WGN][BM]
  const int M = b.M, pM = P * M, W = table_width(P, M);
  double* tsm = red + C::WGN * BM;  // [BM][W]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = warp / C::WGN, wj = warp % C::WGN;
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
  const int gk = tid % BK, gr0 = tid / BK;  // generator: K column gk, rows gr0 + GROWS q

  auto nk_of = [&](int c) { return int(round_up(tmin<int64_t>(m, int64_t(c) * BN + BN), BK) / BK); };
  auto offsets = [&](int64_t j0, int (&off)[P]) {
#pragma unroll
    for (int d = 0; d < P; ++d) off[d] = kcol_offset(j0 + gk, m, M, pM, d, P);
  };
  auto gen_rows = [&](int stage, const int (&off)[P], int q0) {
    double* dst = As + stage * A_STAGE + gk;
#pragma unroll
    for (int qi = 0; qi < C::GPERKK; ++qi) {
      const int r = gr0 + C::GROWS * (q0 + qi);
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
    for (int kk = 0; kk < BK / 4; ++kk) gen_rows(0, off, kk * C::GPERKK);
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
    // V^T is upper triangular: a K chunk lying entirely below this warp's columns is zero
    const bool live = int64_t(n) * BK <= int64_t(c) * BN + wj * WN + WN - 1;
    const double* Ab = As + buf * A_STAGE + (wi * WM + (lane >> 2)) * ASP + (lane & 3);
    const double* Bb = Bs + buf * B_STAGE + (lane & 3) * BSP + wj * WN + (lane >> 2);
    if (live) {
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
        gen_rows(buf ^ 1, off, kk * C::GPERKK);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) gen_rows(buf ^ 1, off, kk * C::GPERKK);
    }
    cp_async_wait<0>();
    __syncthreads();
    if (n2 == 0 || !has_next) {
      fold_tile<C>(acc, vsum, mval, int64_t(c) * BN, m, wj, lane);
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
  finish_rows<C>(vsum, mval, red, As, m, wi, wj, lane, tid, row0, Ns, sigma2, mean_const, mean, var, flags);
}

// Generic K5 (p > 8 or table rows too wide to stage): runtime p, table through L1, one
// barrier-separated generation phase per step.
__global__ void __launch_bounds__(CfgLarge::NT, 1)
predict_kernel_generic(const double* __restrict__ Ts, int64_t Ns, BasisView b, const double* __restrict__ Pop,
                       int64_t pc, double sigma2, double mean_const, double* __restrict__ mean,
                       double* __restrict__ var, uint32_t* flags) {
  using C = CfgLarge;
  constexpr int BM = C::BM, BN = C::BN, NT = C::NT, ASP = C::ASP, BSP = C::BSP;
  constexpr int WM = C::WM, WN = C::WN, FM = C::FM, FN = C::FN, A_STAGE = C::A_STAGE, B_STAGE = C::B_STAGE;
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
    fold_tile<C>(acc, vsum, mval, c0, m, wj, lane);
  }
  finish_rows<C>(vsum, mval, red, As, m, wi, wj, lane, tid, row0, Ns, sigma2, mean_const, mean, var, flags);
}

}  // namespace pred
}  // namespace fagp

using namespace fagp;

namespace fagp {
namespace pred {
template <int P, class C>
int launch_fast(const double* Ts, int64_t Ns, const fagp_basis* basis, const double* op, int64_t pc, double sigma2,
                double c, double* mean, double* var, uint32_t* flags, cudaStream_t s) {
  const size_t smem = fast_smem_bytes<C>(table_width(basis->p, basis->M));
  FAGP_CUDA_TRY(cudaFuncSetAttribute(predict_kernel_fast<P, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  predict_kernel_fast<P, C><<<unsigned(ceil_div(Ns, C::BM)), C::NT, smem, s>>>(Ts, Ns, view(basis), op, pc, sigma2, c,
                                                                              mean, var, flags);
  return FAGP_OK;
}
template <class C>
int dispatch_fast(const double* Ts, int64_t Ns, const fagp_basis* basis, const double* op, int64_t pc, double sigma2,
                  double c, double* mean, double* var, uint32_t* flags, cudaStream_t s) {
  switch (basis->p) {
    case 1: return launch_fast<1, C>(Ts, Ns, basis, op, pc, sigma2, c, mean, var, flags, s);
    case 2: return launch_fast<2, C>(Ts, Ns, basis, op, pc, sigma2, c, mean, var, flags, s);
    case 3: return launch_fast<3, C>(Ts, Ns, basis, op, pc, sigma2, c, mean, var, flags, s);
    case 4: return launch_fast<4, C>(Ts, Ns, basis, op, pc, sigma2, c, mean, var, flags, s);
    case 5: return launch_fast<5, C>(Ts, Ns, basis, op, pc, sigma2, c, mean, var, flags, s);
    case 6: return launch_fast<6, C>(Ts, Ns, basis, op, pc, sigma2, c, mean, var, flags, s);
    case 7: return launch_fast<7, C>(Ts, Ns, basis, op, pc, sigma2, c, mean, var, flags, s);
    default: return launch_fast<8, C>(Ts, Ns, basis, op, pc, sigma2, c, mean, var, flags, s);
  }
}
}  // namespace pred
}  // namespace fagp

extern "C" {

int fagp_phi_matvec(const double* T, int64_t N, const fagp_basis* basis, const double* x, double mean_const,
                    double* out, uint32_t* flags, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || (N > 0 && (T == nullptr || x == nullptr || out == nullptr))) return FAGP_EINVAL;
  if (basis->p > 8) return FAGP_EUNSUPPORTED;
  return modal::matvec(T, N, basis, x, mean_const, out, flags, static_cast<cudaStream_t>(stream));
}

int fagp_predict(const double* Ts, int64_t Ns, const fagp_basis* basis, const double* predict_op, double sigma2,
                 double mean_const, double* mean, double* var, uint32_t* flags, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (Ns < 0 || predict_op == nullptr || (Ns > 0 && (Ts == nullptr || mean == nullptr))) return FAGP_EINVAL;
  if (Ns == 0) return FAGP_OK;
  if (modal::enabled(basis->p, basis->M))
    return modal::predict(Ts, Ns, basis, predict_op, sigma2, mean_const, mean, var, flags,
                          static_cast<cudaStream_t>(stream));
  const int64_t pc = round_up(basis->m + 1, pred::OP_COL_ALIGN);
  const int W = table_width(basis->p, basis->M);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const char* cfg = getenv("FAGP_PREDICT_CFG");  // tuning override: "large" | "small"
  const bool small_ok = pred::fast_smem_bytes<pred::CfgSmall>(W) * pred::CfgSmall::MINB <=
                        228 * 1024 - 1024 * pred::CfgSmall::MINB;
  const bool large_ok = pred::fast_smem_bytes<pred::CfgLarge>(W) <= pred::kMaxSmem;
  int rc = FAGP_OK;
  if (basis->p <= 8 && small_ok && !(cfg && strcmp(cfg, "large") == 0)) {
    rc = pred::dispatch_fast<pred::CfgSmall>(Ts, Ns, basis, predict_op, pc, sigma2, mean_const, mean, var, flags, s);
  } else if (basis->p <= 8 && large_ok) {
    rc = pred::dispatch_fast<pred::CfgLarge>(Ts, Ns, basis, predict_op, pc, sigma2, mean_const, mean, var, flags, s);
  } else {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(pred::predict_kernel_generic, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(pred::CfgLarge::BASE_SMEM)));
    pred::predict_kernel_generic<<<unsigned(ceil_div(Ns, pred::CfgLarge::BM)), pred::CfgLarge::NT,
                                   pred::CfgLarge::BASE_SMEM, s>>>(Ts, Ns, view(basis), predict_op, pc, sigma2,
                                                                   mean_const, mean, var, flags);
  }
  if (rc) return rc;
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // extern "C"
