// Stage (3) of the path: the m x m system.  Replaces, in order,
//   A = (s G) s + sigma2 I                       posterior.py:171-174
//   SpdFactor: dpotrf(lower) + jitter schedule   backend.py:154-189
//   u = cho_solve(A, s*t); w = s*u               posterior.py:233-235, backend.py:191-193
//   solve_inner(I) for the covariance            posterior.py:252-255  -> V = L^{-1} diag(s)
// with hand-written kernels:
//   K2  system_build_kernel   unpack the packed Gram, scale, shift, jitter
//   K3  blocked right-looking Cholesky, NB = 32:
//         chol_diag_kernel (one warp factors + inverts the diagonal block, reports the
//         1-based LAPACK pivot on breakdown), panel = A21 * inv(L11)^T and trailing
//         A22 -= L21 L21^T, both on the generic FP64-DMMA GEMM below
//   K4a trsv kernels (single CTA, forward / backward substitution)
//   K4b TRTRI by recursive doubling (diagonal-block inverses + 2 batched GEMMs per level)
// The host-side driver keeps the reference's jitter schedule: [0, b, 10b, 100b] with
// b = 1e-12 * trace(A) / m, trace in numpy's summation order.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "chol.cuh"
#include "modal.cuh"

namespace fagp {
namespace la {

// ---------------------------------------------------------------------------------------
// Generic FP64 DMMA GEMM: C = alpha * A op(B) + beta * C, row-major, optional batching
// (blockIdx.z with element strides), optional lower-triangle-only output.
constexpr int GT = 64, GK = 16, GNT = 128;
constexpr int ASP = GK + 4;  // 20 % 16 == 4
constexpr int BSP = GT + 4;  // 68 % 16 == 4

struct GemmArgs {
  int M, N, K;
  double alpha, beta;
  const double* A;
  int64_t lda, sA;
  const double* B;
  int64_t ldb, sB;
  double* C;
  int64_t ldc, sC;
  int lower_only;
  const int* info;  // skip all work when *info != 0 (after a Cholesky breakdown)
  // triangular operands: the K range of an output tile shrinks (bits; op(A) is M x K, op(B) K x N)
  //   kTriKminCol: op(B)[k][n] = 0 for k < n (lower)      -> k >= col0
  //   kTriKmaxRow: op(A)[m][k] = 0 for k > m (lower)      -> k <  row0 + GT
  //   kTriKminRow: op(A)[m][k] = 0 for k < m (upper)      -> k >= row0
  //   kTriKmaxCol: op(B)[k][n] = 0 for k > n (upper)      -> k <  col0 + GT
  int tri;
};
constexpr int kTriKminCol = 1, kTriKmaxRow = 2, kTriKminRow = 4, kTriKmaxCol = 8;

template <bool TA, bool TB>
__global__ void __launch_bounds__(GNT) dgemm_kernel(GemmArgs g) {
  if (g.info && *g.info) return;
  const int row0 = blockIdx.y * GT, col0 = blockIdx.x * GT;
  if (g.lower_only && col0 > row0 + GT - 1) return;
  const double* A = g.A + blockIdx.z * g.sA;
  const double* B = g.B + blockIdx.z * g.sB;
  double* C = g.C + blockIdx.z * g.sC;
  __shared__ double As[GT * ASP];
  __shared__ double Bs[GK * BSP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  double acc[4][4][2];
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;

  int kb = 0, ke = g.K;
  if (g.tri & kTriKminCol) kb = tmax(kb, col0);
  if (g.tri & kTriKminRow) kb = tmax(kb, row0);
  if (g.tri & kTriKmaxRow) ke = tmin(ke, row0 + GT);
  if (g.tri & kTriKmaxCol) ke = tmin(ke, col0 + GT);
  kb = kb / GK * GK;  // (the skipped range is exactly zero in the triangular operand)
  for (int k0 = kb; k0 < ke; k0 += GK) {
#pragma unroll
    for (int q = 0; q < (GT * GK) / GNT; ++q) {
      const int e = tid + q * GNT;
      if (TA) {  // A stored K x M
        const int k = e / GT, r = e % GT;
        const int gr = row0 + r, gk = k0 + k;
        As[r * ASP + k] = (gr < g.M && gk < g.K) ? A[int64_t(gk) * g.lda + gr] : 0.0;
      } else {
        const int r = e / GK, k = e % GK;
        const int gr = row0 + r, gk = k0 + k;
        As[r * ASP + k] = (gr < g.M && gk < g.K) ? A[int64_t(gr) * g.lda + gk] : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < (GT * GK) / GNT; ++q) {
      const int e = tid + q * GNT;
      if (TB) {
        const int n = e / GK, k = e % GK;
        const int gn = col0 + n, gk = k0 + k;
        Bs[k * BSP + n] = (gn < g.N && gk < g.K) ? B[int64_t(gn) * g.ldb + gk] : 0.0;
      } else {
        const int k = e / GT, n = e % GT;
        const int gn = col0 + n, gk = k0 + k;
        Bs[k * BSP + n] = (gn < g.N && gk < g.K) ? B[int64_t(gk) * g.ldb + gn] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK / 4; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) a[s] = As[(wm * 32 + s * 8 + (lane >> 2)) * ASP + kk * 4 + (lane & 3)];
#pragma unroll
      for (int t = 0; t < 4; ++t) b[t] = Bs[(kk * 4 + (lane & 3)) * BSP + wn * 32 + t * 8 + (lane >> 2)];
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int t = 0; t < 4; ++t) dmma_8x8x4(acc[s][t][0], acc[s][t][1], a[s], b[t]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int i = row0 + wm * 32 + s * 8 + (lane >> 2);
    if (i >= g.M) continue;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = col0 + wn * 32 + t * 8 + 2 * (lane & 3) + e;
        if (j >= g.N || (g.lower_only && j > i)) continue;
        double* c = C + int64_t(i) * g.ldc + j;
        const double v = g.alpha * acc[s][t][e];
        *c = (g.beta == 0.0) ? v : fma(g.beta, *c, v);
      }
    }
  }
}

// Pipelined variants for the m >= 3000 factor's GEMMs (blocked potrf panels and trailing update,
// TRTRI levels, lauum): BM x BN output tile per CTA, WM x WN warps with a (BM/WM) x (BN/WN) warp tile,
// K slabs of 16 staged by 8-byte cp.async (zero-filled past the edges, any alignment) into a
// STG-deep ring so the next slabs' loads overlap this slab's DMMAs.  Shared layouts keep every
// fragment read conflict-free: row strides = 4 (mod 16) doubles, [m][k] / [k][m] as the operand is
// stored (the transposed operand is copied as it lies, coalesced, and read transposed).  Same
// triangular K clipping, lower-only tiles, batching and info skip as above.
constexpr int BK = 16;
constexpr int BSK = BK + 4;  // [row][k] stride

__device__ __forceinline__ void cp_async_8zf(double* smem, const double* gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0));
}

template <int BM, int BN, int WM, int WN, int STG>
struct BigCfg {
  static constexpr int NT = 32 * WM * WN;
  static constexpr int FM = BM / WM / 8, FN = BN / WN / 8;
  static constexpr int AOP = BM * BSK > BK * (BM + 4) ? BM * BSK : BK * (BM + 4);
  static constexpr int BOP = BN * BSK > BK * (BN + 4) ? BN * BSK : BK * (BN + 4);
  static constexpr size_t smem = size_t(STG) * (AOP + BOP) * sizeof(double);
};

template <int BM, int BN, int WM, int WN, int STG, int MINB, bool TA, bool TB>
__global__ void __launch_bounds__(32 * WM * WN, MINB) dgemm_big_kernel(GemmArgs g) {
  using Cf = BigCfg<BM, BN, WM, WN, STG>;
  constexpr int NT = Cf::NT, FM = Cf::FM, FN = Cf::FN, AOP = Cf::AOP, BOP = Cf::BOP;
  constexpr int SRA = BM + 4, SRB = BN + 4;  // [k][row] strides
  if (g.info && *g.info) return;
  const int row0 = blockIdx.y * BM, col0 = blockIdx.x * BN;
  if (g.lower_only && col0 > row0 + BM - 1) return;
  const double* A = g.A + blockIdx.z * g.sA;
  const double* B = g.B + blockIdx.z * g.sB;
  double* C = g.C + blockIdx.z * g.sC;
  extern __shared__ double gsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  int kb = 0, ke = g.K;
  if (g.tri & kTriKminCol) kb = tmax(kb, col0);
  if (g.tri & kTriKminRow) kb = tmax(kb, row0);
  if (g.tri & kTriKmaxRow) ke = tmin(ke, row0 + BM);
  if (g.tri & kTriKmaxCol) ke = tmin(ke, col0 + BN);
  kb = kb / BK * BK;  // (tile edges are multiples of BK: the clipped range is whole slabs)
  const int nslab = ke > kb ? (ke - kb + BK - 1) / BK : 0;

  auto load = [&](int slab) {
    double* As = gsm + (slab % STG) * (AOP + BOP);
    double* Bs = As + AOP;
    const int k0 = kb + slab * BK;
#pragma unroll
    for (int q = 0; q < (BM * BK) / NT; ++q) {
      const int e = tid + q * NT;
      if (TA) {  // A stored K x M: [k][m]
        const int k = e / BM, r = e % BM, gr = row0 + r, gk = k0 + k;
        const bool ok = gr < g.M && gk < g.K;
        cp_async_8zf(As + k * SRA + r, ok ? A + int64_t(gk) * g.lda + gr : A, ok);
      } else {  // [m][k]
        const int r = e / BK, k = e % BK, gr = row0 + r, gk = k0 + k;
        const bool ok = gr < g.M && gk < g.K;
        cp_async_8zf(As + r * BSK + k, ok ? A + int64_t(gr) * g.lda + gk : A, ok);
      }
    }
#pragma unroll
    for (int q = 0; q < (BN * BK) / NT; ++q) {
      const int e = tid + q * NT;
      if (TB) {  // B stored N x K: [n][k]
        const int n = e / BK, k = e % BK, gn = col0 + n, gk = k0 + k;
        const bool ok = gn < g.N && gk < g.K;
        cp_async_8zf(Bs + n * BSK + k, ok ? B + int64_t(gn) * g.ldb + gk : B, ok);
      } else {  // [k][n]
        const int k = e / BN, n = e % BN, gn = col0 + n, gk = k0 + k;
        const bool ok = gn < g.N && gk < g.K;
        cp_async_8zf(Bs + k * SRB + n, ok ? B + int64_t(gk) * g.ldb + gn : B, ok);
      }
    }
  };

  double acc[FM][FN][2];
#pragma unroll
  for (int f = 0; f < FM; ++f)
#pragma unroll
    for (int t = 0; t < FN; ++t) acc[f][t][0] = acc[f][t][1] = 0.0;
#pragma unroll
  for (int st = 0; st < STG - 1; ++st) {
    if (st < nslab) load(st);
    cp_async_commit();
  }
  const int ar = wm * (BM / WM) + (lane >> 2), bc = wn * (BN / WN) + (lane >> 2), kl = lane & 3;
  for (int slab = 0; slab < nslab; ++slab) {
    cp_async_wait<STG - 2>();
    __syncthreads();  // slab visible to all; the ring slot the next load overwrites is free
    if (slab + STG - 1 < nslab) load(slab + STG - 1);
    cp_async_commit();
    const double* As = gsm + (slab % STG) * (AOP + BOP);
    const double* Bs = As + AOP;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int k = kk * 4 + kl;
      double a[FM], b[FN];
#pragma unroll
      for (int f = 0; f < FM; ++f) a[f] = TA ? As[k * SRA + ar + 8 * f] : As[(ar + 8 * f) * BSK + k];
#pragma unroll
      for (int t = 0; t < FN; ++t) b[t] = TB ? Bs[(bc + 8 * t) * BSK + k] : Bs[k * SRB + bc + 8 * t];
#pragma unroll
      for (int f = 0; f < FM; ++f)
#pragma unroll
        for (int t = 0; t < FN; ++t) dmma_8x8x4(acc[f][t][0], acc[f][t][1], a[f], b[t]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int f = 0; f < FM; ++f) {
    const int i = row0 + wm * (BM / WM) + f * 8 + (lane >> 2);
    if (i >= g.M) continue;
#pragma unroll
    for (int t = 0; t < FN; ++t) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = col0 + wn * (BN / WN) + t * 8 + 2 * (lane & 3) + e;
        if (j >= g.N || (g.lower_only && j > i)) continue;
        double* c = C + int64_t(i) * g.ldc + j;
        const double v = g.alpha * acc[f][t][e];
        *c = (g.beta == 0.0) ? v : fma(g.beta, *c, v);
      }
    }
  }
}

template <int BM, int BN, int WM, int WN, int STG, int MINB, bool TA, bool TB>
static int launch_big1(const GemmArgs& g, int batch, cudaStream_t s) {
  using Cf = BigCfg<BM, BN, WM, WN, STG>;
  auto kern = dgemm_big_kernel<BM, BN, WM, WN, STG, MINB, TA, TB>;
  static bool attr_set[kMaxDevices];  // the smem opt-in is per device context
  int dev = 0;
  FAGP_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= kMaxDevices || !attr_set[dev]) {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cf::smem)));
    if (dev < kMaxDevices) attr_set[dev] = true;
  }
  dim3 grid(unsigned(ceil_div(g.N, BN)), unsigned(ceil_div(g.M, BM)), unsigned(batch));
  kern<<<grid, Cf::NT, Cf::smem, s>>>(g);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

template <int BM, int BN, int WM, int WN, int STG, int MINB>
static int launch_big(const GemmArgs& g, int batch, cudaStream_t s, bool transA, bool transB) {
  if (transA)
    return transB ? launch_big1<BM, BN, WM, WN, STG, MINB, true, true>(g, batch, s)
                  : launch_big1<BM, BN, WM, WN, STG, MINB, true, false>(g, batch, s);
  return transB ? launch_big1<BM, BN, WM, WN, STG, MINB, false, true>(g, batch, s)
                : launch_big1<BM, BN, WM, WN, STG, MINB, false, false>(g, batch, s);
}

inline int gemm(bool transB, const GemmArgs& g, int batch, cudaStream_t s, bool transA = false) {
  if (g.M <= 0 || g.N <= 0 || batch <= 0) return FAGP_OK;
  static const int big_mode = [] {  // FAGP_GEMM_BIG: 0 = the unpipelined kernel everywhere; 2, 3 tile configs
    const char* e = getenv("FAGP_GEMM_BIG");
    return e ? atoi(e) : 3;
  }();
  // a large tile where it fills the GPU: both output sides >= 256 and K >= 64
  if (big_mode && g.M >= 256 && g.N >= 256 && g.K >= 64) {
    // measured (profiles/dgemm_cfg_probe_r05.txt, 4096^3 and the factor's shapes): 64 x 64 tiles
    // with the cp.async ring, 4 CTAs / SM, 31-33 TF/s against 25-30 for the unpipelined kernel;
    // 128 x 64 (2 CTAs / SM) 30-32; 128 x 128 tiles with 8 or 16 warps 27-32, and slower inside
    // the factor (coarser lower-only / triangular tiles)
    switch (big_mode) {
      case 2: return launch_big<128, 64, 4, 2, 3, 2>(g, batch, s, transA, transB);  // 32 x 32 warp tiles, 2 CTAs / SM
      case 3: return launch_big<64, 64, 2, 2, 3, 4>(g, batch, s, transA, transB);   // 32 x 32 warp tiles, 4 CTAs / SM
      default: break;
    }
  }
  dim3 grid(unsigned(ceil_div(g.N, GT)), unsigned(ceil_div(g.M, GT)), unsigned(batch));
  if (transA) {
    if (transB)
      dgemm_kernel<true, true><<<grid, GNT, 0, s>>>(g);
    else
      dgemm_kernel<true, false><<<grid, GNT, 0, s>>>(g);
  } else {
    if (transB)
      dgemm_kernel<false, true><<<grid, GNT, 0, s>>>(g);
    else
      dgemm_kernel<false, false><<<grid, GNT, 0, s>>>(g);
  }
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

// ---------------------------------------------------------------------------------------
// One warp: lower-triangular inverse of the 32x32 block in S (identity-padded beyond nb),
// lane c computes column c by forward substitution.  Result into Xs.
// Xs = S^{-1} for the lower triangular 32 x 32 S (one warp; lane c = column c, held in
// registers): column-oriented forward elimination X[j][c] = y_j / S[j][j], then
// y_r -= S[r][j] X[j][c] for r > j -- 32 dependent steps of independent FMAs (the row-oriented
// dot-product form is ~500 dependent shared-memory round trips).  Column j of S is read as
// broadcasts.
__device__ __forceinline__ void warp_trinv(const double (*S)[33], double (*Xs)[33], int lane) {
  const int c = lane;
  const double dinv = 1.0 / S[c][c];  // lane j: 1 / S[j][j]
  double y[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) y[r] = r == c ? 1.0 : 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double xj = y[j] * __shfl_sync(0xffffffffu, dinv, j);
    y[j] = xj;
#pragma unroll
    for (int r = j + 1; r < 32; ++r) y[r] = fma(-S[r][j], xj, y[r]);
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) Xs[i][c] = i >= c ? y[i] : 0.0;
}

// One step of the blocked right-looking Cholesky (NB = 32), one warp per CTA.  Every CTA
// factors the 32x32 diagonal block A[k0:k0+nb, k0:k0+nb] redundantly (lane i owns row i of
// a shared-memory copy; the loops are runtime-uniform so the SASS stays small enough for the
// instruction cache), which costs a few us and saves a launch plus a grid-wide dependency.
// CTA 0 writes L11; CTA b >= 1 solves panel row-block b-1, L21 = A21 L11^{-T}, by forward
// substitution.  A breakdown (pivot <= 0 or NaN, as LAPACK dpotrf2 tests it) records the
// 1-based global column in *info; every later kernel then exits immediately.
__global__ void __launch_bounds__(32) chol_panel_kernel(double* __restrict__ A, int64_t lda, int64_t m, int64_t k0,
                                                        int nb, int* info) {
  if (*info) return;
  __shared__ double Ls[32][33];  // L11 (for the panel solve)
  __shared__ double dinv[32];
  const int lane = threadIdx.x;
  // Lane i holds the not-yet-factored part of row i in registers, shifted so that r[0] is
  // always the current column j: every register index is a compile-time constant while the
  // j loop stays rolled (small SASS, no shared-memory aliasing in the update).
  double r[32];
#pragma unroll
  for (int c = 0; c < 32; ++c)
    r[c] = (lane < nb && c < nb) ? (c <= lane ? A[(k0 + lane) * lda + k0 + c] : 0.0) : (lane == c ? 1.0 : 0.0);
#pragma unroll 1
  for (int j = 0; j < 32; ++j) {
    const double d = __shfl_sync(0xffffffffu, r[0], j);
    if (!(d > 0.0)) {  // warp-uniform; padding pivots are exactly 1
      if (blockIdx.x == 0 && lane == 0) atomicCAS(info, 0, int(k0 + j + 1));
      return;
    }
    const double ljj = sqrt(d);
    const double inv = 1.0 / ljj;
    const double lij = lane == j ? ljj : (lane > j ? r[0] * inv : 0.0);
    Ls[lane][j] = lij;
    if (lane == j) dinv[j] = inv;
    // trailing update of this lane's row: a_{i, j+k} -= l_ij l_{j+k, j}, then shift left
#pragma unroll
    for (int k = 1; k < 32; ++k) {
      const double lkj = __shfl_sync(0xffffffffu, lij, (j + k) & 31);
      r[k - 1] = (lane >= j + k && j + k < 32) ? fma(-lij, lkj, r[k]) : r[k];
    }
    r[31] = 0.0;
  }
  __syncwarp();
  if (blockIdx.x == 0) {
    if (lane < nb)
      for (int c = 0; c <= lane; ++c) A[(k0 + lane) * lda + k0 + c] = Ls[lane][c];
    return;
  }
  // panel row: x L11^T = a, right-looking with the same shifted-register scheme
  const int64_t i0 = k0 + nb + int64_t(blockIdx.x - 1) * 32 + lane;
  const bool solve = i0 < m;
  double* row = A + (solve ? i0 : 0) * lda + k0;
#pragma unroll
  for (int c = 0; c < 32; ++c) r[c] = (solve && c < nb) ? row[c] : 0.0;
#pragma unroll 1
  for (int j = 0; j < nb; ++j) {
    const double xj = r[0] * dinv[j];
    if (solve) row[j] = xj;
#pragma unroll
    for (int k = 1; k < 32; ++k) r[k - 1] = (j + k < 32) ? fma(-xj, Ls[(j + k) & 31][j], r[k]) : r[k];
    r[31] = 0.0;
  }
}

__global__ void zero_upper_kernel(double* A, int64_t m);

int potrf_blocked(double* A, int64_t m, int64_t lda, int* info, cudaStream_t s) {
  for (int64_t k0 = 0; k0 < m; k0 += 32) {
    const int nb = int(tmin<int64_t>(32, m - k0));
    const int64_t rest = m - k0 - nb;
    chol_panel_kernel<<<unsigned(1 + ceil_div(rest, 32)), 32, 0, s>>>(A, lda, m, k0, nb, info);
    FAGP_LAUNCH_CHECK();
    if (rest <= 0) break;
    double* A21 = A + (k0 + nb) * lda + k0;
    double* A22 = A + (k0 + nb) * lda + (k0 + nb);
    GemmArgs upd{int(rest), int(rest), nb, -1.0, 1.0, A21, lda, 0, A21, lda, 0, A22, lda, 0, 1, info};
    int st = gemm(true, upd, 1, s);
    if (st) return st;
  }
  return FAGP_OK;
}

// One cooperative launch (chol.cu) unless FAGP_POTRF=blocked or the device cannot co-schedule
// the grid; scratch: chol_scratch_len(m) doubles.  Upper triangle is zeroed.
int potrf(double* A, int64_t m, int64_t lda, int* info, double* scratch, cudaStream_t s) {
  const char* e = getenv("FAGP_POTRF");
  if (!(e && strcmp(e, "blocked") == 0)) {
    const int rc = potrf_persistent(A, m, lda, info, scratch, s);
    if (rc != FAGP_EUNSUPPORTED) return rc;
  }
  const int rc = potrf_blocked(A, m, lda, info, s);
  if (rc) return rc;
  zero_upper_kernel<<<int(tmin<int64_t>(ceil_div(m * m, 256), 8 * num_sms())), 256, 0, s>>>(A, m);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

// w = V^T (V t), V = L^{-1} diag(s) taken from the TRTRI result X = L^{-1} (row stride mp):
// w = S L^{-T} L^{-1} S t = s * A^{-1}(s * t)  (posterior.py:233-235), as two parallel
// GEMVs instead of two sequential triangular solves.  Both use fixed summation orders.
// y_k = sum_{j<=k} (X[k,j] s_j) t_j: one warp per row k, lanes stride over j.
__global__ void vt_rows_kernel(const double* __restrict__ X, int64_t mp, const double* __restrict__ s,
                               const double* __restrict__ t, int64_t m, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t k = int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (k >= m) return;
  const double* Xk = X + k * mp;
  double acc = 0.0;
  for (int64_t j = lane; j <= k; j += 32) acc = fma(__dmul_rn(Xk[j], s[j]), t[j], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[k] = acc;
}

// w_j = sum_{k>=j} (X[k,j] s_j) y_k: 32 columns per CTA, 8 k-slices reduced in fixed order.
__global__ void vt_cols_kernel(const double* __restrict__ X, int64_t mp, const double* __restrict__ s,
                               const double* __restrict__ y, int64_t m, double* __restrict__ w) {
  __shared__ double part[8][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t j = int64_t(blockIdx.x) * 32 + tx;
  double acc = 0.0;
  if (j < m) {
    const double sj = s[j];
    for (int64_t k = j + ty; k < m; k += 8) acc = fma(__dmul_rn(X[k * mp + j], sj), y[k], acc);
  }
  part[ty][tx] = acc;
  __syncthreads();
  if (ty == 0 && j < m) {
    double tot = part[0][tx];
#pragma unroll
    for (int q = 1; q < 8; ++q) tot += part[q][tx];
    w[j] = tot;
  }
}

// ---------------------------------------------------------------------------------------
// Triangular solves, one CTA per right-hand side (column of X, row stride ldx).
constexpr int TS_NT = 1024;

__global__ void __launch_bounds__(TS_NT) trsv_lower_kernel(const double* L, int64_t ld, int64_t m, double* X,
                                                           int64_t ldx) {
  double* x = X + blockIdx.x;
  __shared__ double xb[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t k0 = 0; k0 < m; k0 += 32) {
    const int nb = int(tmin<int64_t>(32, m - k0));
    if (warp == 0) {
      double v = lane < nb ? x[(k0 + lane) * ldx] : 0.0;
      for (int j = 0; j < nb; ++j) {
        if (lane == j) v = v / L[(k0 + j) * ld + k0 + j];
        const double xj = __shfl_sync(0xffffffffu, v, j);
        if (lane > j && lane < nb) v -= L[(k0 + lane) * ld + k0 + j] * xj;
      }
      if (lane < nb) {
        xb[lane] = v;
        x[(k0 + lane) * ldx] = v;
      }
    }
    __syncthreads();
    for (int64_t i = k0 + nb + warp; i < m; i += TS_NT / 32) {
      double prod = lane < nb ? L[i * ld + k0 + lane] * xb[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o);
      if (lane == 0) x[i * ldx] -= prod;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(TS_NT) trsv_lower_trans_kernel(const double* L, int64_t ld, int64_t m,
                                                                 double* X, int64_t ldx) {
  double* x = X + blockIdx.x;
  __shared__ double xb[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nblk = ceil_div(m, 32);
  for (int64_t kb = nblk - 1; kb >= 0; --kb) {
    const int64_t k0 = kb * 32;
    const int nb = int(tmin<int64_t>(32, m - k0));
    if (warp == 0) {
      double v = lane < nb ? x[(k0 + lane) * ldx] : 0.0;
      for (int j = nb - 1; j >= 0; --j) {
        if (lane == j) v = v / L[(k0 + j) * ld + k0 + j];
        const double xj = __shfl_sync(0xffffffffu, v, j);
        if (lane < j) v -= L[(k0 + j) * ld + k0 + lane] * xj;
      }
      if (lane < nb) {
        xb[lane] = v;
        x[(k0 + lane) * ldx] = v;
      }
    }
    __syncthreads();
    for (int64_t j = tid; j < k0; j += TS_NT) {
      double acc = 0.0;
      for (int i = 0; i < nb; ++i) acc += L[(k0 + i) * ld + j] * xb[i];
      x[j * ldx] -= acc;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// Elementwise helpers.
__device__ __forceinline__ double packed_at(const double* P, int64_t me, int64_t i, int64_t j) {
  if (i > j) {
    int64_t t = i;
    i = j;
    j = t;
  }
  return P[i * (2 * me - i - 1) / 2 + j];
}

// A[i,j] = (s_i * G_ij) * s_j  (+ sigma2 + jitter on the diagonal); optional G and t.
__global__ void system_build_kernel(const double* __restrict__ P, const double* __restrict__ s, double sigma2,
                                    double jit, int64_t m, double* __restrict__ A, double* __restrict__ G,
                                    double* __restrict__ t) {
  const int64_t me = m + 1;
  const int64_t total = m * m;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / m, j = e - (e / m) * m;
    const double g = packed_at(P, me, i, j);
    if (G) G[e] = g;
    if (A) {
      double a = __dmul_rn(__dmul_rn(s[i], g), s[j]);
      if (i == j) {
        a = __dadd_rn(a, sigma2);
        if (jit != 0.0) a = __dadd_rn(a, jit);
      }
      A[e] = a;
    }
    if (t && j == 0) t[i] = P[i * (2 * me - i - 1) / 2 + m];
  }
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src), as np.trace uses it:
// result = 0.0 + pairwise(diag).
__device__ double np_pairwise_sum(const double* a, int64_t n) {
  // iterative emulation of the recursion with an explicit stack
  struct Frame {
    int64_t off, n;
  };
  Frame stack[64];
  double vals[64];
  int sp = 0, vp = 0;
  stack[sp++] = Frame{0, n};
  // post-order evaluation: push markers by encoding n < 0 as "combine"
  while (sp > 0) {
    Frame f = stack[--sp];
    if (f.n < 0) {
      const double r = vals[--vp];
      const double l = vals[--vp];
      vals[vp++] = l + r;
      continue;
    }
    const int64_t cnt = f.n;
    const double* p = a + f.off;
    if (cnt < 8) {
      double res = 0.0;
      for (int64_t i = 0; i < cnt; ++i) res += p[i];
      vals[vp++] = res;
    } else if (cnt <= 128) {
      double r[8];
      for (int j = 0; j < 8; ++j) r[j] = p[j];
      int64_t i;
      for (i = 8; i < cnt - (cnt % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] += p[i + j];
      double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (; i < cnt; ++i) res += p[i];
      vals[vp++] = res;
    } else {
      int64_t n2 = cnt / 2;
      n2 -= n2 % 8;
      stack[sp++] = Frame{0, -1};
      stack[sp++] = Frame{f.off + n2, cnt - n2};
      stack[sp++] = Frame{f.off, n2};
    }
  }
  return vals[0];
}

__global__ void trace_kernel(const double* A, int64_t m, double* diag_tmp, double* out) {
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) diag_tmp[i] = A[i * m + i];
  __syncthreads();
  if (threadIdx.x == 0) *out = 0.0 + np_pairwise_sum(diag_tmp, m);
}

__global__ void zero_upper_kernel(double* A, int64_t m) {
  const int64_t total = m * m;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / m, j = e - (e / m) * m;
    if (j > i) A[e] = 0.0;
  }
}

__global__ void vec_mul_kernel(const double* a, const double* b, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = __dmul_rn(a[i], b[i]);
}

// ---------------------------------------------------------------------------------------
// TRTRI by recursive doubling on an identity-padded copy of size mp2 = 32 * 2^k.
inline int64_t trtri_dim(int64_t m) {
  int64_t d = 32;
  while (d < m) d *= 2;
  return d;
}

__global__ void pad_lower_kernel(const double* L, int64_t m, int64_t ldl, int64_t mp, double* Lp) {
  const int64_t total = mp * mp;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / mp, j = e - (e / mp) * mp;
    double v;
    if (i < m && j < m)
      v = j <= i ? L[i * ldl + j] : 0.0;
    else
      v = (i == j) ? 1.0 : 0.0;
    Lp[e] = v;
  }
}

__global__ void diag_inv_kernel(const double* Lp, int64_t mp, double* X) {
  __shared__ double S[32][33];
  __shared__ double Xs[32][33];
  const int lane = threadIdx.x;
  const int64_t b0 = int64_t(blockIdx.x) * 32;
  for (int r = 0; r < 32; ++r) S[r][lane] = lane <= r ? Lp[(b0 + r) * mp + b0 + lane] : 0.0;
  __syncwarp();
  warp_trinv(S, Xs, lane);
  __syncwarp();
  for (int r = 0; r < 32; ++r) X[(b0 + r) * mp + b0 + lane] = Xs[r][lane];
}

// X = inv(Lp) (mp x mp, lower).  ws needs mp*mp (Lp) + mp*mp (X) + mp*mp/4 (Tmp) doubles.
int trtri_padded(const double* L, int64_t m, double* Lp, double* X, double* Tmp, cudaStream_t s, int64_t ldl = 0) {
  const int64_t mp = trtri_dim(m);
  const int grid = int(tmin<int64_t>(ceil_div(mp * mp, 256), 8 * num_sms()));
  pad_lower_kernel<<<grid, 256, 0, s>>>(L, m, ldl ? ldl : m, mp, Lp);
  FAGP_LAUNCH_CHECK();
  FAGP_CUDA_TRY(cudaMemsetAsync(X, 0, size_t(mp) * mp * sizeof(double), s));
  diag_inv_kernel<<<unsigned(mp / 32), 32, 0, s>>>(Lp, mp, X);
  FAGP_LAUNCH_CHECK();
  for (int64_t h = 32; h < mp; h *= 2) {
    const int count = int(mp / (2 * h));
    const int64_t dstride = 2 * h * (mp + 1);
    // Tmp_q = L21_q * X11_q
    GemmArgs g1{int(h), int(h), int(h), 1.0, 0.0, Lp + h * mp, mp, dstride, X, mp, dstride, Tmp, h, h * h, 0, nullptr,
                kTriKminCol};  // X11 lower triangular
    int st = gemm(false, g1, count, s);
    if (st) return st;
    // X21_q = -X22_q * Tmp_q
    GemmArgs g2{int(h), int(h), int(h), -1.0, 0.0, X + h * (mp + 1), mp, dstride, Tmp, h, h * h, X + h * mp, mp, dstride, 0, nullptr,
                kTriKmaxRow};  // X22 lower triangular
    st = gemm(false, g2, count, s);
    if (st) return st;
  }
  return FAGP_OK;
}

// Large systems (C4: m 4096, C5: 7776): right-looking Cholesky over kBigNB-column panels whose
// diagonal blocks run the persistent kernel (same pivot test, the breakdown column offset to the
// global one) and whose panel solve and trailing update are GEMMs on the FP64 tensor cores:
//   L_kk = chol(A_kk);  P = A_ik L_kk^{-T} (TRTRI of the block + GEMM);  A_ij -= P_i P_j^T
//   (lower-triangle tiles only);  A_ik = P
// The persistent kernel alone walks 32-column steps (latency-bound at m in the thousands: 32 ms
// at m = 7776); here it only ever sees kBigNB columns.  work: Lp / X / Tmp of trtri_dim(kBigNB)
// and a panel buffer of m x kBigNB doubles.  The upper triangle is left as is (callers zero it).
constexpr int64_t kBigNB = 512;
constexpr int64_t kBigMinM = 3000;
__global__ void zero_upper_kernel(double* A, int64_t m);

int potrf_big(double* A, int64_t m, int64_t lda, int* info, double* scratch, double* Lp, double* X, double* Tmp,
              double* P, cudaStream_t s) {
  const int64_t bp = trtri_dim(kBigNB);
  for (int64_t k0 = 0; k0 < m; k0 += kBigNB) {
    const int64_t b = tmin<int64_t>(kBigNB, m - k0);
    double* Akk = A + k0 * lda + k0;
    int rc = potrf_persistent(Akk, b, lda, info, scratch, s, int(k0));
    if (rc) return rc;
    const int64_t rest = m - k0 - b;
    if (rest <= 0) break;
    rc = trtri_padded(Akk, b, Lp, X, Tmp, s, lda);  // X = L_kk^{-1}, row stride bp
    if (rc) return rc;
    double* A21 = A + (k0 + b) * lda + k0;
    GemmArgs pan{int(rest), int(b), int(b), 1.0, 0.0, A21, lda, 0, X, bp, 0, P, b, 0, 0, info,
                 kTriKmaxCol};  // op(B) = L_kk^{-T}, upper triangular
    rc = gemm(true, pan, 1, s);  // P = A21 L_kk^{-T}
    if (rc) return rc;
    GemmArgs upd{int(rest), int(rest), int(b), -1.0, 1.0, P, b, 0, P, b, 0, A21 + b, lda, 0, 1, info};
    rc = gemm(true, upd, 1, s);  // A22 -= P P^T (lower tiles)
    if (rc) return rc;
    FAGP_CUDA_TRY(cudaMemcpy2DAsync(A21, size_t(lda) * sizeof(double), P, size_t(b) * sizeof(double),
                                    size_t(b) * sizeof(double), size_t(rest), cudaMemcpyDeviceToDevice, s));
  }
  return FAGP_OK;
}

// V[i,j] = X[i,j] * s_j for j <= i < m, else 0   (s may be null)
__global__ void scale_lower_kernel(const double* X, int64_t mp, const double* s, int64_t m, double* V) {
  const int64_t total = m * m;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / m, j = e - (e / m) * m;
    double v = 0.0;
    if (j <= i) v = s ? __dmul_rn(X[i * mp + j], s[j]) : X[i * mp + j];
    V[e] = v;
  }
}

// predict operand P (rows pr = round_up(m, 32), cols pc = round_up(m + 1, 128)):
// P[j, k] = V[k, j] = X[k, j] * s_j for j <= k < m; P[j, m] = w_j; zero elsewhere.
constexpr int OP_ROW_ALIGN = 32, OP_COL_ALIGN = 128;
inline int64_t op_rows(int64_t m) { return round_up(m, OP_ROW_ALIGN); }
inline int64_t op_cols(int64_t m) { return round_up(m + 1, OP_COL_ALIGN); }

__global__ void predict_operand_kernel(const double* X, int64_t mp, const double* s, const double* w, int64_t m,
                                       double* P, int64_t pr, int64_t pc) {
  __shared__ double tile[32][33];
  const int64_t j0 = int64_t(blockIdx.y) * 32, k0 = int64_t(blockIdx.x) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  // read X[k, j] for k in [k0, k0+32), j in [j0, j0+32): coalesced along j
  for (int r = ty; r < 32; r += 8) {
    const int64_t k = k0 + r, j = j0 + tx;
    double v = 0.0;
    if (k < m && j < m && j <= k) v = __dmul_rn(X[k * mp + j], s[j]);
    tile[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t j = j0 + r, k = k0 + tx;
    if (j < pr && k < pc) {
      double v = tile[tx][r];
      if (k == m) v = (j < m && w) ? w[j] : 0.0;
      P[j * pc + k] = v;
    }
  }
}

__global__ void set_mean_weights_kernel(double* P, const double* w, int64_t m, int64_t pc) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < m; j += int64_t(gridDim.x) * blockDim.x)
    P[j * pc + m] = w[j];
}

// w_i = s_i sum_j D_ij (s_j t_j)  (= s * A^{-1}(s * t), posterior.py:233-235) from the explicit
// inverse D: one 128-thread CTA per row, every load of a thread issued together (one round trip),
// thread-strided partial sums combined in a fixed order (shuffle tree, then the 4 warps in order).
constexpr int kGemvNT = 128;
__global__ void __launch_bounds__(kGemvNT) sym_gemv_scaled_kernel(const double* __restrict__ D, int64_t m,
                                                                  const double* __restrict__ s,
                                                                  const double* __restrict__ t,
                                                                  double* __restrict__ w) {
  __shared__ double red[kGemvNT / 32];
  const int tid = int(threadIdx.x), lane = tid & 31, warp = tid >> 5;
  const int64_t i = blockIdx.x;
  const double* Di = D + i * m;
  double acc = 0.0;
  int64_t j = tid;
  for (; j + 7 * kGemvNT < m; j += 8 * kGemvNT) {
    double d[8], u[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      d[q] = Di[j + kGemvNT * q];
      u[q] = __dmul_rn(s[j + kGemvNT * q], t[j + kGemvNT * q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = fma(d[q], u[q], acc);
  }
  {
    double d[8], u[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const bool ok = j + kGemvNT * q < m;
      d[q] = ok ? Di[j + kGemvNT * q] : 0.0;
      u[q] = ok ? __dmul_rn(s[j + kGemvNT * q], t[j + kGemvNT * q]) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (j + kGemvNT * q < m) acc = fma(d[q], u[q], acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double v = red[0];
#pragma unroll
    for (int q = 1; q < kGemvNT / 32; ++q) v += red[q];
    w[i] = __dmul_rn(s[i], v);
  }
}

// ---------------------------------------------------------------------------------------
// Workspace carving.
struct FactorWs {
  int* info;
  double* scalar;  // trace
  double* Dinv;    // 32 x 32
  double* vec;     // m
  double* Lp;      // mp2^2
  double* X;       // mp2^2
  double* Tmp;     // mp2^2 / 4
  double* D;       // m x m: X^T X for the modal predict operand
  double* chol;    // max(chol_scratch_len(m), cholinv_scratch_len(m))
  size_t bytes;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline FactorWs carve(void* base, int64_t m) {
  FactorWs w{};
  const int64_t mp = trtri_dim(m);
  size_t off = 0;
  char* b = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* p = b ? b + off : nullptr;
    off += align256(bytes);
    return p;
  };
  w.info = reinterpret_cast<int*>(take(sizeof(int)));
  w.scalar = reinterpret_cast<double*>(take(sizeof(double)));
  w.Dinv = reinterpret_cast<double*>(take(32 * 32 * sizeof(double)));
  w.vec = reinterpret_cast<double*>(take(size_t(m) * sizeof(double)));
  w.Lp = reinterpret_cast<double*>(take(size_t(mp) * mp * sizeof(double)));
  w.X = reinterpret_cast<double*>(take(size_t(mp) * mp * sizeof(double)));
  w.Tmp = reinterpret_cast<double*>(take(size_t(mp) * mp / 4 * sizeof(double) + sizeof(double)));
  w.D = reinterpret_cast<double*>(take(size_t(m) * m * sizeof(double)));
  w.chol = reinterpret_cast<double*>(take(size_t(tmax(chol_scratch_len(m), cholinv_scratch_len(m))) * sizeof(double)));
  w.bytes = off;
  return w;
}

// [info | Dinv | chol scratch | blocked-route scratch: Lp, X, Tmp of trtri_dim(kBigNB), panel m x kBigNB]
inline size_t potrf_big_bytes(int64_t m) {
  const size_t bp = size_t(trtri_dim(kBigNB));
  return 2 * align256(bp * bp * sizeof(double)) + align256(bp * bp / 4 * sizeof(double) + 8) +
         align256(size_t(m) * kBigNB * sizeof(double));
}
inline size_t potrf_ws_bytes(int64_t m) {
  return align256(sizeof(int)) + align256(32 * 32 * sizeof(double)) + align256(size_t(chol_scratch_len(m)) * sizeof(double)) +
         potrf_big_bytes(m);
}

// D = X^T X for the lower-triangular n x n X (D full symmetric; LAPACK dlauum's product), by
// recursive halving so the zero upper half of X is never multiplied:
//   X = [X11 0; X21 X22]:  D22 = X22^T X22 (recursive),  D21 = X22^T X21,
//                          D11 = X11^T X11 (recursive) + X21^T X21 (lower triangle only)
// -- about n^3 / 2 flops on the DMMA GEMM instead of the full product's 2 n^3 (C4: 4.6 -> ~1.2 ms
// at m = 4096).  Leaves (n <= 512) are one lower-only GEMM; the upper triangle is mirrored last.
__global__ void mirror_lower_kernel(double* D, int64_t n, int64_t ldd) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e - (e / n) * n;
    if (j > i) D[i * ldd + j] = D[j * ldd + i];
  }
}

static int lauum_lower_rec(const double* X, int64_t ldx, int64_t n, double* D, int64_t ldd, cudaStream_t s) {
  if (n <= 512) {
    GemmArgs g{int(n), int(n), int(n), 1.0, 0.0, X, ldx, 0, X, ldx, 0, D, ldd, 0, 1, nullptr,
               kTriKminRow | kTriKminCol};  // X^T upper, X lower
    return gemm(false, g, 1, s, true);
  }
  const int64_t h = round_up(n / 2, 64), r = n - h;
  const double* X21 = X + h * ldx;
  const double* X22 = X21 + h;
  int rc = lauum_lower_rec(X22, ldx, r, D + h * ldd + h, ldd, s);
  if (rc) return rc;
  GemmArgs g21{int(r), int(h), int(r), 1.0, 0.0, X22, ldx, 0, X21, ldx, 0, D + h * ldd, ldd, 0, 0, nullptr,
               kTriKminRow};  // op(A) = X22^T, upper triangular
  rc = gemm(false, g21, 1, s, true);
  if (rc) return rc;
  rc = lauum_lower_rec(X, ldx, h, D, ldd, s);
  if (rc) return rc;
  GemmArgs g11{int(h), int(h), int(r), 1.0, 1.0, X21, ldx, 0, X21, ldx, 0, D, ldd, 0, 1, nullptr};
  return gemm(false, g11, 1, s, true);
}

int lauum_lower(const double* X, int64_t ldx, int64_t n, double* D, int64_t ldd, cudaStream_t s) {
  int rc = lauum_lower_rec(X, ldx, n, D, ldd, s);
  if (rc) return rc;
  mirror_lower_kernel<<<int(tmin<int64_t>(ceil_div(n * n, 256), 8 * num_sms())), 256, 0, s>>>(D, n, ldd);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // namespace la
}  // namespace fagp

using namespace fagp;
using namespace fagp::la;

extern "C" {

size_t fagp_factor_workspace_size(int64_t m) {
  if (m < 1) return 0;
  return carve(nullptr, m).bytes;
}

int64_t fagp_predict_operand_len(const fagp_basis* basis) {
  if (check_basis(basis) != FAGP_OK) return -1;
  if (modal::enabled(basis->p, basis->M)) return modal::predict_op_len(basis);
  return op_rows(basis->m) * op_cols(basis->m);
}

size_t fagp_gram_unpack_workspace_size(const fagp_basis* basis) {
  if (check_basis(basis) != FAGP_OK || !modal::enabled(basis->p, basis->M)) return 0;
  return size_t(modal::scratch_len(basis)) * sizeof(double);
}

int fagp_gram_unpack(const double* gram, const fagp_basis* basis, double* G, double* t, void* workspace,
                     size_t workspace_bytes, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (gram == nullptr) return FAGP_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (modal::enabled(basis->p, basis->M)) {
    if (G) {
      if (workspace == nullptr || workspace_bytes < fagp_gram_unpack_workspace_size(basis)) return FAGP_EWORKSPACE;
      double* H = static_cast<double*>(workspace);
      st = modal::expand(gram, basis, H, H + modal::scratch_len(basis) / 2, s);
      if (st) return st;
      return modal::system(H, gram, nullptr, 0.0, 0.0, basis, nullptr, G, t, s);
    }
    return modal::system(nullptr, gram, nullptr, 0.0, 0.0, basis, nullptr, nullptr, t, s);
  }
  const int64_t m = basis->m;
  const int grid = int(tmin<int64_t>(ceil_div(m * m, 256), 8 * num_sms()));
  system_build_kernel<<<grid, 256, 0, s>>>(gram, nullptr, 0.0, 0.0, m, nullptr, G, t);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

size_t fagp_potrf_workspace_size(int64_t m) { return m < 1 ? 0 : potrf_ws_bytes(m); }

int fagp_potrf(double* A, int64_t m, int32_t* info_dev, void* workspace, size_t workspace_bytes, void* stream) {
  if (A == nullptr || m < 1 || info_dev == nullptr) return FAGP_EINVAL;
  if (workspace == nullptr || workspace_bytes < potrf_ws_bytes(m)) return FAGP_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FAGP_CUDA_TRY(cudaMemsetAsync(info_dev, 0, sizeof(int32_t), s));
  char* w = static_cast<char*>(workspace) + align256(sizeof(int)) + align256(32 * 32 * sizeof(double));
  double* diag = reinterpret_cast<double*>(w);
  const char* e = getenv("FAGP_POTRF");  // "big": the blocked large-m route at any m (tests)
  if (m >= kBigMinM || (e && strcmp(e, "big") == 0)) {
    const size_t bp = size_t(trtri_dim(kBigNB));
    char* q = w + align256(size_t(chol_scratch_len(m)) * sizeof(double));
    double* Lp = reinterpret_cast<double*>(q);
    double* X = reinterpret_cast<double*>(q + align256(bp * bp * sizeof(double)));
    double* Tmp = reinterpret_cast<double*>(q + 2 * align256(bp * bp * sizeof(double)));
    double* P = reinterpret_cast<double*>(q + 2 * align256(bp * bp * sizeof(double)) + align256(bp * bp / 4 * sizeof(double) + 8));
    int rc = potrf_big(A, m, m, reinterpret_cast<int*>(info_dev), diag, Lp, X, Tmp, P, s);
    if (rc) return rc;
    zero_upper_kernel<<<int(tmin<int64_t>(ceil_div(m * m, 256), 8 * num_sms())), 256, 0, s>>>(A, m);
    FAGP_LAUNCH_CHECK();
    return FAGP_OK;
  }
  return potrf(A, m, m, reinterpret_cast<int*>(info_dev), diag, s);
}

int fagp_potrs(const double* L, int64_t m, double* B, int64_t nrhs, void* stream) {
  if (L == nullptr || B == nullptr || m < 1 || nrhs < 0) return FAGP_EINVAL;
  if (nrhs == 0) return FAGP_OK;
  if (nrhs > 65535) return FAGP_EUNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  trsv_lower_kernel<<<unsigned(nrhs), TS_NT, 0, s>>>(L, m, m, B, nrhs);
  FAGP_LAUNCH_CHECK();
  trsv_lower_trans_kernel<<<unsigned(nrhs), TS_NT, 0, s>>>(L, m, m, B, nrhs);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

size_t fagp_trtri_workspace_size(int64_t m) {
  if (m < 1) return 0;
  const int64_t mp = trtri_dim(m);
  return align256(size_t(mp) * mp * sizeof(double)) * 2 + align256(size_t(mp) * mp / 4 * sizeof(double) + 8);
}

int fagp_trtri(const double* L, const double* s, int64_t m, double* V, void* workspace, size_t workspace_bytes,
               void* stream) {
  if (L == nullptr || V == nullptr || m < 1) return FAGP_EINVAL;
  if (workspace == nullptr || workspace_bytes < fagp_trtri_workspace_size(m)) return FAGP_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t mp = trtri_dim(m);
  double* Lp = static_cast<double*>(workspace);
  double* X = reinterpret_cast<double*>(static_cast<char*>(workspace) + align256(size_t(mp) * mp * sizeof(double)));
  double* Tmp = reinterpret_cast<double*>(reinterpret_cast<char*>(X) + align256(size_t(mp) * mp * sizeof(double)));
  int rc = trtri_padded(L, m, Lp, X, Tmp, st);
  if (rc) return rc;
  const int grid = int(tmin<int64_t>(ceil_div(m * m, 256), 8 * num_sms()));
  scale_lower_kernel<<<grid, 256, 0, st>>>(X, mp, s, m, V);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

int fagp_dgemm(int32_t trans_a, int32_t trans_b, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
               int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* stream) {
  if (M < 0 || N < 0 || K < 0 || C == nullptr || (K > 0 && (A == nullptr || B == nullptr))) return FAGP_EINVAL;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return FAGP_EUNSUPPORTED;
  if (ceil_div(M, GT) > 65535) return FAGP_EUNSUPPORTED;
  GemmArgs g{int(M), int(N), int(K), alpha, beta, A, lda, 0, B, ldb, 0, C, ldc, 0, 0, nullptr};
  return gemm(trans_b != 0, g, 1, static_cast<cudaStream_t>(stream), trans_a != 0);
}

int fagp_set_mean_weights(double* predict_op, const double* w, const fagp_basis* basis, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (predict_op == nullptr || w == nullptr) return FAGP_EINVAL;
  if (modal::enabled(basis->p, basis->M))
    return modal::set_weights(predict_op, w, basis, static_cast<cudaStream_t>(stream));
  const int64_t m = basis->m;
  set_mean_weights_kernel<<<unsigned(ceil_div(m, 256)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      predict_op, w, m, op_cols(m));
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

int fagp_factor(const double* packed, const fagp_basis* basis, const double* sqrt_lam, double sigma2,
                int32_t jitter_attempts, double* L, double* G, double* t, double* w, double* predict_op,
                double* jitter_out, int32_t* pivot_out, void* workspace, size_t workspace_bytes, void* stream) {
  {
    int st = check_basis(basis);
    if (st) return st;
  }
  const int64_t m = basis->m;
  const bool pm = modal::enabled(basis->p, basis->M);
  if (packed == nullptr || sqrt_lam == nullptr || L == nullptr || t == nullptr || w == nullptr ||
      jitter_attempts < 0)
    return FAGP_EINVAL;
  if (!(sigma2 > 0.0) || !std::isfinite(sigma2)) return FAGP_EINVAL;
  FactorWs ws = carve(workspace, m);
  if (workspace == nullptr || workspace_bytes < ws.bytes) return FAGP_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = int(tmin<int64_t>(ceil_div(m * m, 256), 8 * num_sms()));
  if (pivot_out) *pivot_out = 0;
  if (jitter_out) *jitter_out = 0.0;

  // modal form: the pair-indexed H (P^p <= m^2 <= mp^2 doubles) lives in ws.Lp until the
  // factorisation succeeds (ws.X is the expansion's temporary)
  if (pm) {
    int rc = modal::expand(packed, basis, ws.Lp, ws.X, s);
    if (rc) return rc;
  }
  // G and t once (A is rebuilt per attempt below)
  auto build = [&](double jit, double* A_, double* G_, double* t_) -> int {
    if (pm) return modal::system(ws.Lp, packed, sqrt_lam, sigma2, jit, basis, A_, G_, t_, s);
    system_build_kernel<<<grid, 256, 0, s>>>(packed, sqrt_lam, sigma2, jit, m, A_, G_, t_);
    FAGP_LAUNCH_CHECK();
    return FAGP_OK;
  };
  {
    int rc = build(0.0, nullptr, G, t);
    if (rc) return rc;
  }

  double base = 0.0;
  bool have_base = false;
  int info_h = 0;
  for (int attempt = 0; attempt <= jitter_attempts; ++attempt) {
    double jit = 0.0;
    if (attempt > 0) {
      if (!have_base) {
        // trace of the un-jittered A, in numpy's summation order (np.trace)
        int rc0 = build(0.0, L, nullptr, nullptr);
        if (rc0) return rc0;
        trace_kernel<<<1, 256, 0, s>>>(L, m, ws.vec, ws.scalar);
        FAGP_LAUNCH_CHECK();
        double tr = 0.0;
        FAGP_CUDA_TRY(cudaMemcpyAsync(&tr, ws.scalar, sizeof(double), cudaMemcpyDeviceToHost, s));
        FAGP_CUDA_TRY(cudaStreamSynchronize(s));
        base = 1e-12 * tr / double(m);
        have_base = true;
      }
      double p10 = 1.0;
      for (int k = 1; k < attempt; ++k) p10 *= 10.0;
      jit = base * p10;
    }
    {
      int rc1 = build(jit, L, nullptr, nullptr);
      if (rc1) return rc1;
    }
    FAGP_CUDA_TRY(cudaMemsetAsync(ws.info, 0, sizeof(int), s));
    // (the block TRTRI buffers and D double as the blocked factorisation's scratch: both are
    // only needed after it)
    int rc = m >= kBigMinM ? potrf_big(L, m, m, ws.info, ws.chol, ws.Lp, ws.X, ws.Tmp, ws.D, s)
                           : potrf(L, m, m, ws.info, ws.chol, s);
    if (rc) return rc;
    FAGP_CUDA_TRY(cudaMemcpyAsync(&info_h, ws.info, sizeof(int), cudaMemcpyDeviceToHost, s));
    FAGP_CUDA_TRY(cudaStreamSynchronize(s));
    if (jitter_out) *jitter_out = jit;
    if (info_h == 0) break;
  }
  if (info_h != 0) {
    if (pivot_out) *pivot_out = info_h;
    return FAGP_ENOTPD;
  }
  zero_upper_kernel<<<grid, 256, 0, s>>>(L, m);
  FAGP_LAUNCH_CHECK();
  // V = L^{-1} diag(s) by TRTRI, then w = V^T (V t) = s * A^{-1}(s * t) and the predict operand
  {
    int rc = trtri_padded(L, m, ws.Lp, ws.X, ws.Tmp, s);
    if (rc) return rc;
  }
  const int64_t mp = trtri_dim(m);
  vt_rows_kernel<<<unsigned(ceil_div(m, 8)), 256, 0, s>>>(ws.X, mp, sqrt_lam, t, m, ws.vec);
  FAGP_LAUNCH_CHECK();
  vt_cols_kernel<<<unsigned(ceil_div(m, 32)), dim3(32, 8), 0, s>>>(ws.X, mp, sqrt_lam, ws.vec, m, w);
  FAGP_LAUNCH_CHECK();
  if (predict_op) {
    if (pm) {
      // D = X^T X (X = L^{-1}, lower), then the pair-folded Ct = fold(S D S) and w
      int rc = lauum_lower(ws.X, mp, m, ws.D, m, s);
      if (rc) return rc;
      rc = modal::build_predict_op(ws.D, sqrt_lam, w, basis, predict_op, ws.Lp, ws.X, s);
      if (rc) return rc;
    } else {
      const int64_t pr = op_rows(m), pc = op_cols(m);
      dim3 g2(unsigned(ceil_div(pc, 32)), unsigned(ceil_div(pr, 32)));
      predict_operand_kernel<<<g2, dim3(32, 8), 0, s>>>(ws.X, mp, sqrt_lam, w, m, predict_op, pr, pc);
      FAGP_LAUNCH_CHECK();
    }
  }
  return FAGP_OK;
}


constexpr int64_t kFactorInvMaxM = 2048;

// The hot-path variant of fagp_factor for the modal shapes: the same A, jitter schedule,
// breakdown index, w and predict operand, but A^{-1} comes from one persistent kernel (potrf,
// trtri and X^T X fused, chol.cu) instead of 2 m/32 + 12 launches, and L is not returned.
int fagp_factor_inv(const double* packed, const fagp_basis* basis, const double* sqrt_lam, double sigma2,
                    int32_t jitter_attempts, double* Ainv, double* G, double* t, double* w, double* predict_op,
                    double* jitter_out, int32_t* pivot_out, void* workspace, size_t workspace_bytes, void* stream) {
  {
    int st = check_basis(basis);
    if (st) return st;
  }
  const int64_t m = basis->m;
  // latency-bound systems only: above a few thousand features the blocked route's large
  // GEMM tiles (fagp_factor) win
  if (!modal::enabled(basis->p, basis->M) || m > kFactorInvMaxM) return FAGP_EUNSUPPORTED;
  if (packed == nullptr || sqrt_lam == nullptr || t == nullptr || w == nullptr || Ainv == nullptr ||
      jitter_attempts < 0)
    return FAGP_EINVAL;
  if (!(sigma2 > 0.0) || !std::isfinite(sigma2)) return FAGP_EINVAL;
  FactorWs ws = carve(workspace, m);
  if (workspace == nullptr || workspace_bytes < ws.bytes) return FAGP_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (pivot_out) *pivot_out = 0;
  if (jitter_out) *jitter_out = 0.0;
  double* D = Ainv;
  double* A = ws.X;  // m x m (the expansion's temporary until the system is built)
  int rc = modal::expand(packed, basis, ws.Lp, ws.X, s);
  if (rc) return rc;
  rc = modal::system(ws.Lp, packed, sqrt_lam, sigma2, 0.0, basis, nullptr, G, t, s);
  if (rc) return rc;
  double base = 0.0;
  bool have_base = false;
  int info_h = 0;
  for (int attempt = 0; attempt <= jitter_attempts; ++attempt) {
    double jit = 0.0;
    if (attempt > 0) {
      if (!have_base) {
        rc = modal::system(ws.Lp, packed, sqrt_lam, sigma2, 0.0, basis, A, nullptr, nullptr, s);
        if (rc) return rc;
        trace_kernel<<<1, 256, 0, s>>>(A, m, ws.vec, ws.scalar);
        FAGP_LAUNCH_CHECK();
        double tr = 0.0;
        FAGP_CUDA_TRY(cudaMemcpyAsync(&tr, ws.scalar, sizeof(double), cudaMemcpyDeviceToHost, s));
        FAGP_CUDA_TRY(cudaStreamSynchronize(s));
        base = 1e-12 * tr / double(m);
        have_base = true;
      }
      double p10 = 1.0;
      for (int k = 1; k < attempt; ++k) p10 *= 10.0;
      jit = base * p10;
    }
    rc = modal::system(ws.Lp, packed, sqrt_lam, sigma2, jit, basis, A, nullptr, nullptr, s);
    if (rc) return rc;
    FAGP_CUDA_TRY(cudaMemsetAsync(ws.info, 0, sizeof(int), s));
    rc = chol_inverse_persistent(A, m, m, ws.info, ws.chol, ws.D, D, m, s);
    if (rc) return rc;
    FAGP_CUDA_TRY(cudaMemcpyAsync(&info_h, ws.info, sizeof(int), cudaMemcpyDeviceToHost, s));
    FAGP_CUDA_TRY(cudaStreamSynchronize(s));
    if (jitter_out) *jitter_out = jit;
    if (info_h == 0) break;
  }
  if (info_h != 0) {
    if (pivot_out) *pivot_out = info_h;
    return FAGP_ENOTPD;
  }
  sym_gemv_scaled_kernel<<<unsigned(m), kGemvNT, 0, s>>>(D, m, sqrt_lam, t, w);
  FAGP_LAUNCH_CHECK();
  if (predict_op) {
    rc = modal::build_predict_op(D, sqrt_lam, w, basis, predict_op, ws.Lp, ws.X, s);
    if (rc) return rc;
  }
  return FAGP_OK;
}


// Attempt 0 of fagp_factor_inv (no jitter) enqueued without any host synchronisation: the
// system, the fused inverse, w and the predict operand are issued unconditionally and the
// breakdown index is copied asynchronously to *info_host (pinned host memory; read it after the
// stream has synchronised).  A caller can enqueue the predict right behind it, so the GPU runs
// factor -> predict back to back; only when *info_host != 0 (a breakdown: the jitter schedule
// is needed) must it call fagp_factor_inv and redo what followed.
int fagp_factor_inv_async(const double* packed, const fagp_basis* basis, const double* sqrt_lam, double sigma2,
                          double* Ainv, double* G, double* t, double* w, double* predict_op, int32_t* info_host,
                          void* workspace, size_t workspace_bytes, void* stream) {
  {
    int st = check_basis(basis);
    if (st) return st;
  }
  const int64_t m = basis->m;
  if (!modal::enabled(basis->p, basis->M) || m > kFactorInvMaxM) return FAGP_EUNSUPPORTED;
  if (packed == nullptr || sqrt_lam == nullptr || t == nullptr || w == nullptr || Ainv == nullptr ||
      info_host == nullptr)
    return FAGP_EINVAL;
  if (!(sigma2 > 0.0) || !std::isfinite(sigma2)) return FAGP_EINVAL;
  FactorWs ws = carve(workspace, m);
  if (workspace == nullptr || workspace_bytes < ws.bytes) return FAGP_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* A = ws.X;
  int rc = modal::expand(packed, basis, ws.Lp, ws.X, s);
  if (rc) return rc;
  rc = modal::system(ws.Lp, packed, sqrt_lam, sigma2, 0.0, basis, A, G, t, s);
  if (rc) return rc;
  FAGP_CUDA_TRY(cudaMemsetAsync(ws.info, 0, sizeof(int), s));
  rc = chol_inverse_persistent(A, m, m, ws.info, ws.chol, ws.D, Ainv, m, s);
  if (rc) return rc;
  FAGP_CUDA_TRY(cudaMemcpyAsync(info_host, ws.info, sizeof(int), cudaMemcpyDeviceToHost, s));
  sym_gemv_scaled_kernel<<<unsigned(m), kGemvNT, 0, s>>>(Ainv, m, sqrt_lam, t, w);
  FAGP_LAUNCH_CHECK();
  if (predict_op) {
    rc = modal::build_predict_op(Ainv, sqrt_lam, w, basis, predict_op, ws.Lp, ws.X, s);
    if (rc) return rc;
  }
  return FAGP_OK;
}

size_t fagp_spd_inverse_workspace_size(int64_t m) {
  if (m < 1) return 0;
  return align256(sizeof(int)) + align256(size_t(cholinv_scratch_len(m)) * sizeof(double)) +
         align256(size_t(m) * m * sizeof(double));
}

int fagp_spd_inverse(double* A, int64_t m, double* Ainv, int32_t* info_dev, void* workspace, size_t workspace_bytes,
                     void* stream) {
  if (A == nullptr || Ainv == nullptr || info_dev == nullptr || m < 1 || A == Ainv) return FAGP_EINVAL;
  if (workspace == nullptr || workspace_bytes < fagp_spd_inverse_workspace_size(m)) return FAGP_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* scratch = reinterpret_cast<double*>(static_cast<char*>(workspace) + align256(sizeof(int)));
  double* X = reinterpret_cast<double*>(reinterpret_cast<char*>(scratch) +
                                        align256(size_t(cholinv_scratch_len(m)) * sizeof(double)));
  FAGP_CUDA_TRY(cudaMemsetAsync(info_dev, 0, sizeof(int32_t), s));
  return chol_inverse_persistent(A, m, m, info_dev, scratch, X, Ainv, m, s);
}

}  // extern "C"
