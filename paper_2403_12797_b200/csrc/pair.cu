// Pair-structured Gram and variance: the tensor-product symmetry of the Mercer features.
//
// Every feature is a product of per-dimension eigenfunctions, Phi[r,(a_0..a_{p-1})] =
// prod_d phi_d,a_d(x_rd) (mercer.py:284-292), so
//
//   G[(a),(a')] = sum_r prod_d phi_d,a_d phi_d,a'_d = H[pi(a_0,a'_0), ..., pi(a_{p-1},a'_{p-1})]
//
// depends only on the UNORDERED pair {a_d, a'_d} in every dimension.  With P = M(M+1)/2
// pairs per dimension G has only P^p distinct entries (55^3 = 166,375 at p=3, M=10, against
// m(m+1)/2 = 500,500), and they are a plain rectangular GEMM over the data rows:
//
//   H = U_L^T U_R,  U_L[r, lambda] = prod_{d<pL} q_d[r, pi_d],  U_R[r, rho] = prod_{d>=pL} q_d[r, pi_d],
//   q_d[r, {a,a'}] = phi_d,a(x_rd) phi_d,a'(x_rd).
//
// Likewise the posterior variance var_i = sigma2 * phi_i^T C phi_i with C = V^T V = S A^{-1} S
// (posterior.py:249-263, diag) folds onto pairs:
//
//   var_i = sigma2 * sum_{pi} Ct[pi] prod_d q_d[i, pi_d],
//   Ct[pi] = sum over the orderings (a_d, a'_d) of every pi_d of C[(a), (a')],
//
// computed as Y = Q_K Ct (K = the pair combos of the last dims, tensor cores) followed by a
// fused epilogue sum_nu Y[i, nu] prod_{d < pN} q_d[i, nu_d].  This is ~3x (p=3) to ~7x (p=5)
// less tensor-core work than the SYRK / triangular forms.  Used for p >= 2; for p = 1 the pair
// form is the SYRK itself and the direct kernels (gram.cu, predict.cu) are used.
//
// Kernels in this file (all FP64; tensor work on mma.m8n8k4.f64 = SASS DMMA):
//   KP1  pair_gram_kernel<FA, FB>   generated-operand GEMM over row chunks, split-K partials
//   KP1b pair_gram_reduce_kernel     fixed-order split-K sum -> H, non-finite flag
//        (t = Phi^T r comes out of the same GEMM as 'singleton' tiles)
//   KP2  pair_system_kernel          A = (s_i G_ij) s_j + sigma2 I (+ jitter) gathered from H
//   KP4  ctilde_kernel               Ct from D = X^T X (X = L^{-1}) and s
//   KP5  pair_var_kernel<FK, FE>     Y = Q_K Ct tiles with the q-product epilogue -> var
//   KP5m mean_kernel                 mean = c + Phi* w by nested per-dimension sums
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "pair.cuh"

namespace fagp {
namespace pairk {

// ---------------------------------------------------------------------------------------
// Offsets of the factors of one generated column.  A column is a product of up to
// 2 * (number of dims) table entries; unused factor slots point at the table's 1.0 entry,
// padding columns at its 0.0 entry (first slot).

// pair index -> (a, a'), a <= a'
__device__ __forceinline__ void pair_decode(int pi, int M, int& a, int& b) {
  int base = 0, x = 0;
  while (pi >= base + (M - x)) {
    base += M - x;
    ++x;
  }
  a = x;
  b = x + (pi - base);
}

// Factors of pair-combo column `col` over the F/2 dims starting at d0 (mixed radix P, first
// slowest): 2 per dim; invalid columns -> (zero, one, one, ...).  Fully unrolled so the
// offsets live in registers.
template <int F>
__device__ __forceinline__ void combo_offsets(int64_t col, int64_t ncols, int d0, int M, int P, int pM,
                                              int (&off)[F]) {
  static_assert(F % 2 == 0, "two factors per dimension");
  unsigned q = col < ncols ? unsigned(col) : 0u;  // pair-combo counts stay below 2^31 (enabled())
#pragma unroll
  for (int e = F / 2 - 1; e >= 0; --e) {
    const int pi = int(q % unsigned(P));
    q /= unsigned(P);
    int a, b;
    pair_decode(pi, M, a, b);
    off[2 * e] = (d0 + e) * M + a;
    off[2 * e + 1] = (d0 + e) * M + b;
  }
  if (col >= ncols) {
    off[0] = table_col_zero(pM);
#pragma unroll
    for (int f = 1; f < F; ++f) off[f] = table_col_one(pM);
  }
}

// Singleton columns for t = Phi^T r: column `col` over the F/2 dims starting at d0 (mixed
// radix M): factors (phi_d,a, 1) per dim; with_r puts the residual entry in slot 1.
template <int F>
__device__ __forceinline__ void single_offsets(int64_t col, int64_t ncols, int d0, int M, int pM, bool with_r,
                                               int (&off)[F]) {
  int64_t q = col < ncols ? col : 0;
#pragma unroll
  for (int e = F / 2 - 1; e >= 0; --e) {
    off[2 * e] = (d0 + e) * M + int(q % M);
    off[2 * e + 1] = table_col_one(pM);
    q /= M;
  }
  if (with_r) off[1] = table_col_r(pM);
  if (col >= ncols) {
    off[0] = table_col_zero(pM);
#pragma unroll
    for (int f = 1; f < F; ++f) off[f] = table_col_one(pM);
  }
}

// ---------------------------------------------------------------------------------------
// KP1: H tile = sum over a row chunk of U_L^T U_R, both operands generated per row.  The
// last stA x stB tiles of the grid are "singleton" tiles that produce t = Phi^T r the same
// way: A columns prod_{d<pL} phi_d,a_d, B columns r * prod_{d>=pL} phi_d,a_d.
constexpr int GBM = 128, GBN = 56, GBK = 16, GNT = 128;  // 4 warps, warp tile 32 x 56
constexpr int GSPA = GBM + 4, GSPB = GBN + 12;          // % 16 == 4
constexpr int GFM = 4, GFN = 7;
constexpr int GA_STAGE = GBK * GSPA, GB_STAGE = GBK * GSPB;

inline size_t gram_smem(int W) {
  return (size_t(2) * (GA_STAGE + GB_STAGE) + size_t(2) * GBK * W) * sizeof(double);
}

template <int FA, int FB>
__global__ void __launch_bounds__(GNT, 3)
pair_gram_kernel(const double* __restrict__ T, int64_t N, BasisView b, PairPlan pl, double* __restrict__ ws) {
  extern __shared__ double sm[];
  double* As = sm;                         // [2][GBK][GSPA]
  double* Bs = sm + 2 * GA_STAGE;          // [2][GBK][GSPB]
  double* tbuf = Bs + 2 * GB_STAGE;        // [2][GBK][W]
  const int M = b.M, pM = b.p * M, W = table_width(b.p, M);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npair = pl.gtA * pl.gtB;
  const int tile = pl.tile0 + int(blockIdx.x % pl.nrun), chunk = int(blockIdx.x / pl.nrun);
  const int64_t r0 = int64_t(chunk) * pl.chunk_rows;
  const int64_t r1 = tmin<int64_t>(N, r0 + pl.chunk_rows);

  // generator role: A column tid (4 rows per k-step); B column tid % GBN for the first
  // 2 GBN threads, which split each k-step's 4 rows in halves (balances the warps)
  int offA[FA], offB[FB];
  const bool genB = tid < 2 * GBN;
  const int bcol = tid % GBN, bhalf = tid / GBN;
  if (tile < npair) {
    const int ta = tile / pl.gtB, tb = tile % pl.gtB;
    combo_offsets<FA>(int64_t(ta) * GBM + tid, pl.GA, 0, M, pl.P, pM, offA);
    combo_offsets<FB>(int64_t(tb) * GBN + bcol, pl.GB, pl.pL, M, pl.P, pM, offB);
  } else {
    const int ta = (tile - npair) / pl.stB, tb = (tile - npair) % pl.stB;
    single_offsets<FA>(int64_t(ta) * GBM + tid, pl.SA, 0, M, pM, false, offA);
    single_offsets<FB>(int64_t(tb) * GBN + bcol, pl.SB, pl.pL, M, pM, true, offB);
  }

  auto load_tab = [&](int slot, int64_t base) {
    double* dst = tbuf + slot * (GBK * W);
    const int nrows = int(tmax<int64_t>(0, tmin<int64_t>(GBK, r1 - base)));
    const int nd = nrows * W;
    const double* src = T + base * W;
    for (int i = tid; i < nd / 2; i += GNT) cp_async_16(dst + 2 * i, src + 2 * i);
    for (int i = nd + tid; i < GBK * W; i += GNT) dst[i] = 0.0;
    cp_async_commit();
  };
  auto gen_rows = [&](int stage, int kk) {
    const double* tb_ = tbuf + stage * (GBK * W);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = kk * 4 + i;
      const double* Tr = tb_ + k * W;
      double v = Tr[offA[0]];
#pragma unroll
      for (int f = 1; f < FA; ++f) v = __dmul_rn(v, Tr[offA[f]]);
      As[stage * GA_STAGE + k * GSPA + tid] = v;
    }
    if (genB) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int k = kk * 4 + bhalf * 2 + i;
        const double* Tr = tb_ + k * W;
        double u = Tr[offB[0]];
#pragma unroll
        for (int f = 1; f < FB; ++f) u = __dmul_rn(u, Tr[offB[f]]);
        Bs[stage * GB_STAGE + k * GSPB + bcol] = u;
      }
    }
  };

  double acc[GFM][GFN][2];
#pragma unroll
  for (int s = 0; s < GFM; ++s)
#pragma unroll
    for (int t = 0; t < GFN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;

  const int nchunks = int(ceil_div(tmax<int64_t>(r1 - r0, 0), GBK));
  load_tab(0, r0);
  cp_async_wait<0>();
  __syncthreads();
  load_tab(1, r0 + GBK);
#pragma unroll
  for (int kk = 0; kk < GBK / 4; ++kk) gen_rows(0, kk);
  cp_async_wait<0>();
  __syncthreads();
  for (int n = 0; n < nchunks; ++n) {
    const int cur = n & 1, nxt = cur ^ 1;
    if (n + 2 < nchunks) load_tab(cur, r0 + int64_t(n + 2) * GBK);
    const double* Ab = As + cur * GA_STAGE + (lane & 3) * GSPA + warp * 32 + (lane >> 2);
    const double* Bb = Bs + cur * GB_STAGE + (lane & 3) * GSPB + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < GBK / 4; ++kk) {
      double a[GFM], bb[GFN];
#pragma unroll
      for (int s = 0; s < GFM; ++s) a[s] = Ab[kk * 4 * GSPA + s * 8];
#pragma unroll
      for (int t = 0; t < GFN; ++t) bb[t] = Bb[kk * 4 * GSPB + t * 8];
#pragma unroll
      for (int s = 0; s < GFM; ++s)
#pragma unroll
        for (int t = 0; t < GFN; ++t) dmma_8x8x4(acc[s][t][0], acc[s][t][1], a[s], bb[t]);
#ifndef FAGP_DIAG_NOGEN
      gen_rows(nxt, kk);  // chunk n+1 (garbage past the last chunk, never read)
#endif
    }
    cp_async_wait<0>();
    __syncthreads();
  }
  double* out = ws + (size_t(chunk) * pl.nrun + (tile - pl.tile0)) * size_t(GBM * GBN);
#pragma unroll
  for (int s = 0; s < GFM; ++s) {
    const int i = warp * 32 + s * 8 + (lane >> 2);
#pragma unroll
    for (int t = 0; t < GFN; ++t) {
      const int j = t * 8 + 2 * (lane & 3);
      *reinterpret_cast<double2*>(out + i * GBN + j) = make_double2(acc[s][t][0], acc[s][t][1]);
    }
  }
}

// KP1 (warp-specialised): 4 consumer warps issue only fragment loads and DMMAs; 2 producer
// warps stage table rows (cp.async), generate the U_L / U_R tiles of each 16-row chunk into
// a 3-stage shared-memory ring and hand them over with named barriers (FULL[s] / EMPTY[s]),
// so generation never interrupts the tensor-core instruction stream.
constexpr int WS_STAGES = 3, WS_CONS = 4, WS_PROD = 2;
constexpr int WS_NT = 32 * (WS_CONS + WS_PROD);
constexpr int WS_PT = 32 * WS_PROD;  // producer threads

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

inline size_t gram_ws_smem(int W) {
  return size_t(WS_STAGES) * (GA_STAGE + GB_STAGE + size_t(GBK) * W) * sizeof(double);
}

template <int FA, int FB>
__global__ void __launch_bounds__(WS_NT, 2)
pair_gram_ws_kernel(const double* __restrict__ T, int64_t N, BasisView b, PairPlan pl, double* __restrict__ ws) {
  extern __shared__ double sm[];
  const int M = b.M, pM = b.p * M, W = table_width(b.p, M);
  double* As = sm;                                   // [STAGES][GBK][GSPA]
  double* Bs = As + WS_STAGES * GA_STAGE;            // [STAGES][GBK][GSPB]
  double* Tb = Bs + WS_STAGES * GB_STAGE;            // [STAGES][GBK][W]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npair = pl.gtA * pl.gtB;
  const int tile = pl.tile0 + int(blockIdx.x % pl.nrun), chunk = int(blockIdx.x / pl.nrun);
  const int64_t r0 = int64_t(chunk) * pl.chunk_rows;
  const int64_t r1 = tmin<int64_t>(N, r0 + pl.chunk_rows);
  const int nchunks = int(ceil_div(tmax<int64_t>(r1 - r0, 0), GBK));
  constexpr int FULL0 = 1, EMPTY0 = 1 + WS_STAGES, PROD = 1 + 2 * WS_STAGES;

  if (warp >= WS_CONS) {
    // ---------------- producers ----------------
    const int pt = tid - 32 * WS_CONS;  // 0..63
    int offA0[FA], offA1[FA], offB[FB];
    const bool genB = pt < GBN;
    if (tile < npair) {
      const int ta = tile / pl.gtB, tb = tile % pl.gtB;
      combo_offsets<FA>(int64_t(ta) * GBM + pt, pl.GA, 0, M, pl.P, pM, offA0);
      combo_offsets<FA>(int64_t(ta) * GBM + pt + WS_PT, pl.GA, 0, M, pl.P, pM, offA1);
      combo_offsets<FB>(int64_t(tb) * GBN + pt, pl.GB, pl.pL, M, pl.P, pM, offB);
    } else {
      const int ta = (tile - npair) / pl.stB, tb = (tile - npair) % pl.stB;
      single_offsets<FA>(int64_t(ta) * GBM + pt, pl.SA, 0, M, pM, false, offA0);
      single_offsets<FA>(int64_t(ta) * GBM + pt + WS_PT, pl.SA, 0, M, pM, false, offA1);
      single_offsets<FB>(int64_t(tb) * GBN + pt, pl.SB, pl.pL, M, pM, true, offB);
    }
    auto load_tab = [&](int slot, int64_t base) {
      double* dst = Tb + slot * (GBK * W);
      const int nrows = int(tmax<int64_t>(0, tmin<int64_t>(GBK, r1 - base)));
      const int nd = nrows * W;
      const double* src = T + base * W;
      for (int i = pt; i < nd / 2; i += WS_PT) cp_async_16(dst + 2 * i, src + 2 * i);
      for (int i = nd + pt; i < GBK * W; i += WS_PT) dst[i] = 0.0;
      cp_async_commit();
    };
    if (nchunks > 0) load_tab(0, r0);
    for (int n = 0; n < nchunks; ++n) {
      const int slot = n % WS_STAGES;
      // table rows of chunk n are in Tb[slot]; prefetch chunk n+1's into the next slot (its
      // previous content, chunk n+1-STAGES, was consumed by this warp group long ago)
      if (n + 1 < nchunks) load_tab((n + 1) % WS_STAGES, r0 + int64_t(n + 1) * GBK);
      if (n + 1 < nchunks) cp_async_wait<1>(); else cp_async_wait<0>();
      named_sync(PROD, WS_PT);  // chunk n's table visible to all producers
      if (n >= WS_STAGES) named_sync(EMPTY0 + slot, WS_NT);  // consumers released this slot
      const double* tb = Tb + slot * (GBK * W);
      double* Ad = As + slot * GA_STAGE;
      double* Bd = Bs + slot * GB_STAGE;
#pragma unroll 4
      for (int k = 0; k < GBK; ++k) {
        const double* Tr = tb + k * W;
        double v0 = Tr[offA0[0]], v1 = Tr[offA1[0]];
#pragma unroll
        for (int f = 1; f < FA; ++f) {
          v0 = __dmul_rn(v0, Tr[offA0[f]]);
          v1 = __dmul_rn(v1, Tr[offA1[f]]);
        }
        Ad[k * GSPA + pt] = v0;
        Ad[k * GSPA + pt + WS_PT] = v1;
        if (genB) {
          double u = Tr[offB[0]];
#pragma unroll
          for (int f = 1; f < FB; ++f) u = __dmul_rn(u, Tr[offB[f]]);
          Bd[k * GSPB + pt] = u;
        }
      }
      named_arrive(FULL0 + slot, WS_NT);
    }
    return;
  }

  // ---------------- consumers ----------------
  double acc[GFM][GFN][2];
#pragma unroll
  for (int s = 0; s < GFM; ++s)
#pragma unroll
    for (int t = 0; t < GFN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;
  for (int n = 0; n < nchunks; ++n) {
    const int slot = n % WS_STAGES;
    named_sync(FULL0 + slot, WS_NT);
    const double* Ab = As + slot * GA_STAGE + (lane & 3) * GSPA + warp * 32 + (lane >> 2);
    const double* Bb = Bs + slot * GB_STAGE + (lane & 3) * GSPB + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < GBK / 4; ++kk) {
      double a[GFM], bb[GFN];
#pragma unroll
      for (int s = 0; s < GFM; ++s) a[s] = Ab[kk * 4 * GSPA + s * 8];
#pragma unroll
      for (int t = 0; t < GFN; ++t) bb[t] = Bb[kk * 4 * GSPB + t * 8];
#pragma unroll
      for (int s = 0; s < GFM; ++s)
#pragma unroll
        for (int t = 0; t < GFN; ++t) dmma_8x8x4(acc[s][t][0], acc[s][t][1], a[s], bb[t]);
    }
    // release the slot unless the producers will never refill it
    if (n + WS_STAGES < nchunks) named_arrive(EMPTY0 + slot, WS_NT);
  }
  double* out = ws + (size_t(chunk) * pl.nrun + (tile - pl.tile0)) * size_t(GBM * GBN);
#pragma unroll
  for (int s = 0; s < GFM; ++s) {
    const int i = warp * 32 + s * 8 + (lane >> 2);
#pragma unroll
    for (int t = 0; t < GFN; ++t) {
      const int j = t * 8 + 2 * (lane & 3);
      *reinterpret_cast<double2*>(out + i * GBN + j) = make_double2(acc[s][t][0], acc[s][t][1]);
    }
  }
}

// KP1b: H[lambda * GB + rho] and t[lambda' * SB + rho'] = sum_s partial[s][tile][..] in
// chunk order (deterministic); any non-finite entry flags a non-finite feature.
__global__ void pair_gram_reduce_kernel(const double* __restrict__ ws, PairPlan pl, double* __restrict__ out,
                                        uint32_t* flags) {
  const int64_t nH = pl.GA * pl.GB, nt = pl.SA * pl.SB;
  const int npair = pl.gtA * pl.gtB;
  const size_t stride = size_t(pl.nrun) * GBM * GBN;
  const int64_t e0 = pl.tile0 > 0 ? nH : 0;  // t-only runs produce just t
  bool bad = false;
  for (int64_t e = e0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nH + nt;
       e += int64_t(gridDim.x) * blockDim.x) {
    int tile;
    int64_t lam, rho;
    if (e < nH) {
      lam = e / pl.GB;
      rho = e - lam * pl.GB;
      tile = int(lam / GBM) * pl.gtB + int(rho / GBN);
    } else {
      const int64_t q = e - nH;
      lam = q / pl.SB;
      rho = q - lam * pl.SB;
      tile = npair + int(lam / GBM) * pl.stB + int(rho / GBN);
    }
    const double* src = ws + size_t(tile - pl.tile0) * GBM * GBN + size_t(lam % GBM) * GBN + size_t(rho % GBN);
    double sum = 0.0;
    for (int s = 0; s < pl.S; ++s) sum += src[s * stride];
    out[e - e0] = sum;
    bad |= not_finite(sum);
  }
  if (bad) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
}

// ---------------------------------------------------------------------------------------
// KP2: A[i,j] = (s_i G_ij) s_j (+ sigma2 + jitter on the diagonal), G_ij gathered from H;
// optional full G and t copy.  (posterior.py:171-174)
__device__ __forceinline__ int64_t h_index(int64_t i, int64_t j, int p, int M, int P) {
  int64_t key = 0, pw = 1;
  for (int d = p - 1; d >= 0; --d) {
    const int a = int(i % M), c = int(j % M);
    i /= M;
    j /= M;
    const int lo = a < c ? a : c, hi = a < c ? c : a;
    key += pw * (int64_t(lo) * M - int64_t(lo) * (lo - 1) / 2 + (hi - lo));
    pw *= P;
  }
  return key;
}

__global__ void pair_system_kernel(const double* __restrict__ H, const double* __restrict__ s, double sigma2,
                                   double jit, BasisView b, int P, double* __restrict__ A, double* __restrict__ G) {
  const int64_t m = b.m, total = m * m;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / m, j = e - (e / m) * m;
    const double g = H[h_index(i, j, b.p, b.M, P)];
    if (G) G[e] = g;
    if (A) {
      double a = __dmul_rn(__dmul_rn(s[i], g), s[j]);
      if (i == j) {
        a = __dadd_rn(a, sigma2);
        if (jit != 0.0) a = __dadd_rn(a, jit);
      }
      A[e] = a;
    }
  }
}

// ---------------------------------------------------------------------------------------
// KP4: Ct[kappa][nu] over the predict layout (nu = pair combo of dims < pN, kappa = combo of
// dims >= pN), Ct[pi] = sum over orderings of (s_j D_jj') s_j', D = X^T X, X = L^{-1}.
__global__ void ctilde_kernel(const double* __restrict__ D, int64_t ldd, const double* __restrict__ s, BasisView b,
                              PairPlan pl, double* __restrict__ Ct) {
  const int M = b.M, p = b.p, P = pl.P;
  const int64_t total = pl.KP * pl.NP;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t kap = e / pl.NP, nu = e - (e / pl.NP) * pl.NP;
    double v = 0.0;
    if (kap < pl.KR && nu < pl.NR) {
      int lo[FAGP_MAX_P], hi[FAGP_MAX_P];
      int64_t q = kap;
      for (int d = p - 1; d >= pl.pN; --d) {
        pair_decode(int(q % P), M, lo[d], hi[d]);
        q /= P;
      }
      q = nu;
      for (int d = pl.pN - 1; d >= 0; --d) {
        pair_decode(int(q % P), M, lo[d], hi[d]);
        q /= P;
      }
      int nflip = 0;
      int fd[FAGP_MAX_P];
      for (int d = 0; d < p; ++d)
        if (lo[d] != hi[d]) fd[nflip++] = d;
      for (int o = 0; o < (1 << nflip); ++o) {
        int64_t j = 0, jj = 0;
        for (int d = 0; d < p; ++d) {
          int x = lo[d], y = hi[d];
          for (int f = 0; f < nflip; ++f)
            if (fd[f] == d && ((o >> f) & 1)) {
              x = hi[d];
              y = lo[d];
            }
          j = j * M + x;
          jj = jj * M + y;
        }
        v += s ? __dmul_rn(__dmul_rn(s[j], D[j * ldd + jj]), s[jj]) : D[j * ldd + jj];
      }
    }
    Ct[e] = v;
  }
}

// ---------------------------------------------------------------------------------------
// KP5: var for BM test rows: Y = Q_K Ct over K chunks (Q_K generated from the staged table
// rows: product of the pair values of dims >= pN), then var_i = sigma2 sum_nu Y[i,nu] E[i,nu]
// with E = product of the pair values of dims < pN.  Ct streams from L2 by cp.async.
constexpr int VBM = 128, VBN = 56, VBK = 16;
constexpr int VASP = VBK + 4, VBSP = VBN + 12;           // 20, 68 (% 16 == 4)
constexpr int VFN = 7;
constexpr int VA_STAGE = VBM * VASP, VB_STAGE = VBK * VBSP;

inline size_t var_smem(int W) {
  return (size_t(2) * (VA_STAGE + VB_STAGE) + size_t(VBM) * W + VBM) * sizeof(double);
}

template <int FK, int FE, int NW>
__global__ void __launch_bounds__(32 * NW, 2)
pair_var_kernel(const double* __restrict__ Ts, int64_t Ns, BasisView b, PairPlan pl, const double* __restrict__ Ct,
                double sigma2, double* __restrict__ var, uint32_t* flags) {
  constexpr int VNT = 32 * NW;             // NW warps stacked along the rows
  constexpr int VWM = VBM / NW, VFM = VWM / 8;
  constexpr int GGRP = VNT / VBK;          // generator row groups
  constexpr int GPERKK = VBM / GGRP / (VBK / 4);  // generated rows per thread per k-step
  extern __shared__ double sm[];
  double* As = sm;                     // [2][VBM][VASP]
  double* Bs = sm + 2 * VA_STAGE;      // [2][VBK][VBSP]
  double* tsm = Bs + 2 * VB_STAGE;     // [VBM][W]
  double* red = tsm + 0;               // reused after the main loop
  const int M = b.M, pM = b.p * M, W = table_width(b.p, M);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t row0 = int64_t(blockIdx.x) * VBM;
  {
    const int nd = int(tmin<int64_t>(VBM, Ns - row0)) * W;
    const double* src = Ts + row0 * W;
    for (int i = tid; i < nd / 2; i += VNT) cp_async_16(tsm + 2 * i, src + 2 * i);
    for (int i = nd + tid; i < VBM * W; i += VNT) tsm[i] = 0.0;
    cp_async_commit();
  }
  const int gk = tid % VBK, gr0 = tid / VBK;  // generator: K column gk, rows gr0 + GGRP q
  const int nkc = int(pl.KP / VBK);
  const int ntn = int(pl.NP / VBN);

  auto load_b = [&](int stage, int64_t k0, int64_t n0) {
    double* dst = Bs + stage * VB_STAGE;
    for (int e = tid; e < VBK * VBN / 2; e += VNT) {
      const int k = e / (VBN / 2), n2 = e % (VBN / 2);
      cp_async_16(dst + k * VBSP + 2 * n2, Ct + (k0 + k) * pl.NP + n0 + 2 * n2);
    }
    cp_async_commit();
  };
  auto gen_rows = [&](int stage, const int (&off)[FK], int q0) {
    double* dst = As + stage * VA_STAGE + gk;
#pragma unroll
    for (int qi = 0; qi < GPERKK; ++qi) {
      const int r = gr0 + GGRP * (q0 + qi);
      const double* Tr = tsm + r * W;
      double v = Tr[off[0]];
#pragma unroll
      for (int f = 1; f < FK; ++f) v = __dmul_rn(v, Tr[off[f]]);
      dst[r * VASP] = v;
    }
  };

  double vsum[VFM];
#pragma unroll
  for (int s = 0; s < VFM; ++s) vsum[s] = 0.0;
  double acc[VFM][VFN][2];
#pragma unroll
  for (int s = 0; s < VFM; ++s)
#pragma unroll
    for (int t = 0; t < VFN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;

  cp_async_wait<0>();
  __syncthreads();
  load_b(0, 0, 0);
  {
    int off[FK];
    combo_offsets<FK>(gk, pl.KR, pl.pN, M, pl.P, pM, off);
#pragma unroll
    for (int kk = 0; kk < VBK / 4; ++kk) gen_rows(0, off, kk * GPERKK);
  }
  cp_async_wait<0>();
  __syncthreads();

  int tn = 0, kc = 0, buf = 0;
  while (true) {
    int tn2 = tn, kc2 = kc + 1;
    if (kc2 == nkc) {
      tn2 = tn + 1;
      kc2 = 0;
    }
    const bool has_next = tn2 < ntn;
    if (has_next) load_b(buf ^ 1, int64_t(kc2) * VBK, int64_t(tn2) * VBN);
    int off[FK];
    combo_offsets<FK>(int64_t(kc2) * VBK + gk, pl.KR, pl.pN, M, pl.P, pM, off);
    const double* Ab = As + buf * VA_STAGE + (warp * VWM + (lane >> 2)) * VASP + (lane & 3);
    const double* Bb = Bs + buf * VB_STAGE + (lane & 3) * VBSP + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < VBK / 4; ++kk) {
      double a[VFM], bb[VFN];
#pragma unroll
      for (int s = 0; s < VFM; ++s) a[s] = Ab[s * 8 * VASP + kk * 4];
#pragma unroll
      for (int t = 0; t < VFN; ++t) bb[t] = Bb[kk * 4 * VBSP + t * 8];
#pragma unroll
      for (int s = 0; s < VFM; ++s)
#pragma unroll
        for (int t = 0; t < VFN; ++t) dmma_8x8x4(acc[s][t][0], acc[s][t][1], a[s], bb[t]);
#ifndef FAGP_DIAG_NOGEN
      gen_rows(buf ^ 1, off, kk * GPERKK);
#endif
    }
    cp_async_wait<0>();
    __syncthreads();
    if (kc2 == 0 || !has_next) {
      // epilogue of column tile tn: vsum_i += Y[i, nu] * E[i, nu]
#pragma unroll
      for (int t = 0; t < VFN; ++t) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t nu = int64_t(tn) * VBN + t * 8 + 2 * (lane & 3) + e;
          int offe[FE];
          combo_offsets<FE>(nu, pl.NR, 0, M, pl.P, pM, offe);
#pragma unroll
          for (int s = 0; s < VFM; ++s) {
            const double* Tr = tsm + (warp * VWM + s * 8 + (lane >> 2)) * W;
            double ev = Tr[offe[0]];
#pragma unroll
            for (int f = 1; f < FE; ++f) ev = __dmul_rn(ev, Tr[offe[f]]);
            vsum[s] = fma(acc[s][t][e], ev, vsum[s]);
          }
        }
      }
#pragma unroll
      for (int s = 0; s < VFM; ++s)
#pragma unroll
        for (int t = 0; t < VFN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;
    }
    if (!has_next) break;
    tn = tn2;
    kc = kc2;
    buf ^= 1;
  }
  // lanes sharing a row (same lane >> 2) hold disjoint columns: fixed-order xor reduction
#pragma unroll
  for (int s = 0; s < VFM; ++s) {
    double v = vsum[s];
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    vsum[s] = v;
  }
  if ((lane & 3) == 0) {
#pragma unroll
    for (int s = 0; s < VFM; ++s) {
      const int64_t row = row0 + warp * VWM + s * 8 + (lane >> 2);
      if (row < Ns) {
        const double vv = sigma2 * vsum[s];
        var[row] = vv;
        if (not_finite(vv)) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
      }
    }
  }
  (void)red;
}

// ---------------------------------------------------------------------------------------
// KP5m: mean_i = c + sum_j w_j Phi[i, j], one thread per test row, w broadcast from shared
// memory: mean - c = sum_u prefix_u(i) * sum_c phi_{p-1,c}(i) w[u M + c], with the innermost
// dimension's values in registers (M <= MREG) and the prefix product over dims < p-1 kept up
// to date by an odometer on its digits.
constexpr int MNT = 128, MREG = 16;
template <int P>
__global__ void __launch_bounds__(MNT) mean_kernel(const double* __restrict__ Ts, int64_t Ns, BasisView b,
                                                   const double* __restrict__ w, double mean_const,
                                                   double* __restrict__ mean, uint32_t* flags) {
  extern __shared__ double sm[];
  const int M = b.M, W = table_width(P, M);
  const int WS = W | 1;  // odd row stride: conflict-free per-thread rows
  const int64_t m = b.m;
  double* ws_ = sm;      // [m]
  double* tsm = sm + m;  // [MNT][WS]
  const int tid = threadIdx.x;
  for (int64_t j = tid; j < m; j += MNT) ws_[j] = w[j];
  const int64_t row0 = int64_t(blockIdx.x) * MNT;
  const int nr = int(tmin<int64_t>(MNT, Ns - row0));
  for (int e = tid; e < MNT * W; e += MNT) {
    const int rl = e / W, c = e - (e / W) * W;
    tsm[rl * WS + c] = rl < nr ? Ts[(row0 + rl) * W + c] : 0.0;
  }
  __syncthreads();
  if (tid >= nr) return;
  const double* Tr = tsm + tid * WS;
  double f[MREG];
#pragma unroll
  for (int c = 0; c < MREG; ++c) f[c] = c < M ? Tr[(P - 1) * M + c] : 0.0;
  int dig[P > 1 ? P - 1 : 1];
#pragma unroll
  for (int d = 0; d < P - 1; ++d) dig[d] = 0;
  const int64_t U = m / M;
  double total = 0.0;
  for (int64_t u = 0; u < U; ++u) {
    const double* wu = ws_ + u * M;
    double acc = 0.0;
    if (M <= MREG) {
#pragma unroll
      for (int c = 0; c < MREG; ++c)
        if (c < M) acc = fma(f[c], wu[c], acc);
    } else {
      for (int c = 0; c < M; ++c) acc = fma(Tr[(P - 1) * M + c], wu[c], acc);
    }
    double pre = 1.0;
#pragma unroll
    for (int d = 0; d < P - 1; ++d) pre = __dmul_rn(pre, Tr[d * M + dig[d]]);
    total = fma(pre, acc, total);
#pragma unroll
    for (int d = P - 2; d >= 0; --d) {  // odometer, last prefix digit fastest
      if (++dig[d] < M) break;
      dig[d] = 0;
    }
  }
  const double mm = mean_const + total;
  mean[row0 + tid] = mm;
  if (not_finite(mm)) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
}

}  // namespace pairk
}  // namespace fagp

// =======================================================================================
// Host side
namespace fagp {
namespace pairk {

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

bool enabled(int p, int M) {
  if (p < 2 || p > 8 || M < 1) return false;
  const int64_t P = int64_t(M) * (M + 1) / 2;
  // every split keeps factor counts within the instantiated templates (<= 8 factors) and
  // pair-combo indices in 31 bits
  return ipow(P, p) < (int64_t(1) << 31);
}

PairPlan make_plan(int64_t N, int p, int M, bool t_only) {
  PairPlan pl{};
  pl.P = M * (M + 1) / 2;
  pl.Hlen = ipow(pl.P, p);
  // Gram split: padding efficiency of the 128 x 56 tiles, discounted by the generation
  // DMULs per DMMA ((FA-1) per A element, (FB-1) per B element)
  double best = -1.0;
  for (int pL = 1; pL <= p - 1; ++pL) {
    if (pL > 4 || p - pL > 4) continue;
    const int64_t GA = ipow(pl.P, pL), GB = ipow(pl.P, p - pL);
    const double eff = double(GA) / double(round_up(GA, 128)) * double(GB) / double(round_up(GB, 56));
    const double dmul = (128.0 * (2 * pL - 1) + 56.0 * (2 * (p - pL) - 1)) / 28.0 / 32.0 * 2.0 / 16.0;
    const double score = eff / (1.0 + dmul);
    if (score > best + 1e-12) {
      best = score;
      pl.pL = pL;
    }
  }
  pl.GA = ipow(pl.P, pl.pL);
  pl.GB = ipow(pl.P, p - pl.pL);
  pl.gtA = int(ceil_div(pl.GA, 128));
  pl.gtB = int(ceil_div(pl.GB, 56));
  pl.SA = ipow(M, pl.pL);
  pl.SB = ipow(M, p - pl.pL);
  pl.stA = int(ceil_div(pl.SA, 128));
  pl.stB = int(ceil_div(pl.SB, 56));
  // variance split
  best = -1.0;
  for (int pN = 1; pN <= p - 1; ++pN) {
    if (pN > 4 || p - pN > 4) continue;
    const int64_t NR = ipow(pl.P, pN), KR = ipow(pl.P, p - pN);
    const double eff = double(NR) / double(round_up(NR, 56)) * double(KR) / double(round_up(KR, 16));
    const double dmul = (2 * (p - pN) - 1) * (128.0 * 16.0) / (128.0 * 56.0 * 16.0 / 256.0) / 32.0 * 2.0 / 16.0;
    const double score = eff / (1.0 + dmul);
    if (score > best + 1e-12) {
      best = score;
      pl.pN = pN;
    }
  }
  pl.NR = ipow(pl.P, pl.pN);
  pl.KR = ipow(pl.P, p - pl.pN);
  pl.NP = round_up(pl.NR, 56);
  pl.KP = round_up(pl.KR, 16);
  // tiles launched, then split-K over rows: 3 CTAs per SM
  pl.tile0 = t_only ? pl.gtA * pl.gtB : 0;
  pl.nrun = (t_only ? 0 : pl.gtA * pl.gtB) + pl.stA * pl.stB;
  const int64_t tiles = pl.nrun;
  const int64_t max_chunks = tmax<int64_t>(1, ceil_div(N, 16));
  const int64_t slots = int64_t(num_sms()) * 3;
  int64_t bestS = 1;
  double beste = -1.0;
  for (int64_t S = 1; S <= tmin<int64_t>(max_chunks, 4096); ++S) {
    const int64_t ctas = S * tiles;
    const double eff = double(ctas) / double(ceil_div(ctas, slots) * slots);
    if ((ctas >= 2 * slots || S == max_chunks) && eff >= 0.96) {
      bestS = S;
      break;
    }
    if (eff > beste + 1e-9) {
      beste = eff;
      bestS = S;
    }
  }
  pl.chunk_rows = round_up(tmax<int64_t>(1, ceil_div(tmax<int64_t>(N, 1), bestS)), 16);
  pl.S = int(tmax<int64_t>(1, ceil_div(N, pl.chunk_rows)));
  return pl;
}

int64_t gram_len(const fagp_basis* b) { return make_plan(0, b->p, b->M).Hlen + b->m; }

size_t gram_workspace(int64_t N, const fagp_basis* b) {
  const PairPlan pl = make_plan(N, b->p, b->M);
  return size_t(pl.S) * pl.nrun * GBM * GBN * sizeof(double);
}

size_t tmatvec_workspace(int64_t N, const fagp_basis* b) {
  const PairPlan pl = make_plan(N, b->p, b->M, true);
  return size_t(pl.S) * pl.nrun * GBM * GBN * sizeof(double);
}

static bool gram_ws_enabled() {
  // Experimental: the warp-specialised kernel measured 17.6 ms vs 13.8 ms for the
  // interleaved one at C3 (producer DMULs lose the FP64 pipe to the DMMA stream); opt in
  // with FAGP_GRAM_WS=1.
  const char* e = getenv("FAGP_GRAM_WS");
  return e && e[0] == '1';
}

template <int FA>
static int launch_gram_fb(int FB, const double* T, int64_t N, const fagp_basis* b, const PairPlan& pl, double* ws,
                          size_t smem, unsigned grid, cudaStream_t s) {
  const int W = table_width(b->p, b->M);
  const bool wsk = gram_ws_enabled() && gram_ws_smem(W) * 2 <= 227 * 1024;
  auto go = [&](auto kern, int nt, size_t sm) -> int {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    kern<<<grid, nt, sm, s>>>(T, N, view(b), pl, ws);
    return FAGP_OK;
  };
  if (wsk) {
    const size_t sm = gram_ws_smem(W);
    switch (FB) {
      case 2: return go(pair_gram_ws_kernel<FA, 2>, WS_NT, sm);
      case 4: return go(pair_gram_ws_kernel<FA, 4>, WS_NT, sm);
      case 6: return go(pair_gram_ws_kernel<FA, 6>, WS_NT, sm);
      case 8: return go(pair_gram_ws_kernel<FA, 8>, WS_NT, sm);
      default: return FAGP_EUNSUPPORTED;
    }
  }
  switch (FB) {
    case 2: return go(pair_gram_kernel<FA, 2>, GNT, smem);
    case 4: return go(pair_gram_kernel<FA, 4>, GNT, smem);
    case 6: return go(pair_gram_kernel<FA, 6>, GNT, smem);
    case 8: return go(pair_gram_kernel<FA, 8>, GNT, smem);
    default: return FAGP_EUNSUPPORTED;
  }
}

static int run_gram(const PairPlan& pl, const double* T, int64_t N, const fagp_basis* b, double* out, double* ws,
                    uint32_t* flags, cudaStream_t s) {
  const int W = table_width(b->p, b->M);
  const size_t smem = gram_smem(W);
  if (smem > 227 * 1024) return FAGP_EUNSUPPORTED;
  const unsigned grid = unsigned(size_t(pl.S) * pl.nrun);
  const int FA = 2 * pl.pL, FB = 2 * (b->p - pl.pL);
  int rc;
  switch (FA) {
    case 2: rc = launch_gram_fb<2>(FB, T, N, b, pl, ws, smem, grid, s); break;
    case 4: rc = launch_gram_fb<4>(FB, T, N, b, pl, ws, smem, grid, s); break;
    case 6: rc = launch_gram_fb<6>(FB, T, N, b, pl, ws, smem, grid, s); break;
    case 8: rc = launch_gram_fb<8>(FB, T, N, b, pl, ws, smem, grid, s); break;
    default: rc = FAGP_EUNSUPPORTED;
  }
  if (rc) return rc;
  FAGP_LAUNCH_CHECK();
  pair_gram_reduce_kernel<<<unsigned(tmin<int64_t>(ceil_div(pl.Hlen + b->m, 256), 16 * num_sms())), 256, 0, s>>>(
      ws, pl, out, flags);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

int gram(const double* T, int64_t N, const fagp_basis* b, double* out, void* ws, size_t ws_bytes, uint32_t* flags,
         cudaStream_t s) {
  if (ws == nullptr || ws_bytes < gram_workspace(N, b)) return FAGP_EWORKSPACE;
  return run_gram(make_plan(N, b->p, b->M), T, N, b, out, static_cast<double*>(ws), flags, s);
}

int tmatvec(const double* T, int64_t N, const fagp_basis* b, double* t, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (ws == nullptr || ws_bytes < tmatvec_workspace(N, b)) return FAGP_EWORKSPACE;
  return run_gram(make_plan(N, b->p, b->M, true), T, N, b, t, static_cast<double*>(ws), nullptr, s);
}

__global__ void copy_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

int system(const double* g, const double* sqrt_lam, double sigma2, double jit, const fagp_basis* b, double* A,
           double* G, double* t, cudaStream_t s) {
  const PairPlan pl = make_plan(0, b->p, b->M);
  const int64_t m = b->m;
  if (A || G) {
    const int grid = int(tmin<int64_t>(ceil_div(m * m, 256), 8 * num_sms()));
    pair_system_kernel<<<grid, 256, 0, s>>>(g, sqrt_lam, sigma2, jit, view(b), pl.P, A, G);
    FAGP_LAUNCH_CHECK();
  }
  if (t) {
    copy_kernel<<<unsigned(ceil_div(m, 256)), 256, 0, s>>>(g + pl.Hlen, t, m);
    FAGP_LAUNCH_CHECK();
  }
  return FAGP_OK;
}

int64_t predict_op_len(const fagp_basis* b) {
  const PairPlan pl = make_plan(0, b->p, b->M);
  return pl.KP * pl.NP + b->m;
}

int build_predict_op(const double* D, const double* sqrt_lam, const double* w, const fagp_basis* b, double* op,
                     cudaStream_t s) {
  const PairPlan pl = make_plan(0, b->p, b->M);
  const int grid = int(tmin<int64_t>(ceil_div(pl.KP * pl.NP, 256), 16 * num_sms()));
  ctilde_kernel<<<grid, 256, 0, s>>>(D, b->m, sqrt_lam, view(b), pl, op);
  FAGP_LAUNCH_CHECK();
  return set_weights(op, w, b, s);
}

int set_weights(double* op, const double* w, const fagp_basis* b, cudaStream_t s) {
  const PairPlan pl = make_plan(0, b->p, b->M);
  copy_kernel<<<unsigned(ceil_div(b->m, 256)), 256, 0, s>>>(w, op + pl.KP * pl.NP, b->m);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

static int var_warps() {
  const char* e = getenv("FAGP_VAR_WARPS");  // tuning override: 4 | 8
  return (e && atoi(e) == 8) ? 8 : 4;
}

template <int FK, int NW>
static int launch_var_nw(int FE, const double* Ts, int64_t Ns, const fagp_basis* b, const PairPlan& pl,
                         const double* Ct, double sigma2, double* var, uint32_t* flags, size_t smem, cudaStream_t s) {
  auto go = [&](auto kern) -> int {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<unsigned(ceil_div(Ns, VBM)), 32 * NW, smem, s>>>(Ts, Ns, view(b), pl, Ct, sigma2, var, flags);
    return FAGP_OK;
  };
  switch (FE) {
    case 2: return go(pair_var_kernel<FK, 2, NW>);
    case 4: return go(pair_var_kernel<FK, 4, NW>);
    case 6: return go(pair_var_kernel<FK, 6, NW>);
    case 8: return go(pair_var_kernel<FK, 8, NW>);
    default: return FAGP_EUNSUPPORTED;
  }
}

int matvec(const double* T, int64_t N, const fagp_basis* b, const double* x, double c, double* y, uint32_t* flags,
           cudaStream_t s) {
  if (N == 0) return FAGP_OK;
  const int W = table_width(b->p, b->M);
  const size_t msmem = (size_t(b->m) + size_t(MNT) * (W | 1)) * sizeof(double);
  if (msmem > 227 * 1024) return FAGP_EUNSUPPORTED;
  auto go = [&](auto kern) -> int {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(msmem)));
    kern<<<unsigned(ceil_div(N, MNT)), MNT, msmem, s>>>(T, N, view(b), x, c, y, flags);
    return FAGP_OK;
  };
  int rc;
  switch (b->p) {
    case 1: rc = go(mean_kernel<1>); break;
    case 2: rc = go(mean_kernel<2>); break;
    case 3: rc = go(mean_kernel<3>); break;
    case 4: rc = go(mean_kernel<4>); break;
    case 5: rc = go(mean_kernel<5>); break;
    case 6: rc = go(mean_kernel<6>); break;
    case 7: rc = go(mean_kernel<7>); break;
    case 8: rc = go(mean_kernel<8>); break;
    default: rc = FAGP_EUNSUPPORTED;
  }
  if (rc) return rc;
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

template <int FK>
static int launch_var_fe(int FE, const double* Ts, int64_t Ns, const fagp_basis* b, const PairPlan& pl,
                         const double* Ct, double sigma2, double* var, uint32_t* flags, size_t smem, cudaStream_t s) {
  if (var_warps() == 4) return launch_var_nw<FK, 4>(FE, Ts, Ns, b, pl, Ct, sigma2, var, flags, smem, s);
  return launch_var_nw<FK, 8>(FE, Ts, Ns, b, pl, Ct, sigma2, var, flags, smem, s);
}

int predict(const double* Ts, int64_t Ns, const fagp_basis* b, const double* op, double sigma2, double mean_const,
            double* mean, double* var, uint32_t* flags, cudaStream_t s) {
  const PairPlan pl = make_plan(0, b->p, b->M);
  const int W = table_width(b->p, b->M);
  if (var) {
    const size_t smem = var_smem(W);
    if (smem > 227 * 1024) return FAGP_EUNSUPPORTED;
    const int FK = 2 * (b->p - pl.pN), FE = 2 * pl.pN;
    int rc;
    switch (FK) {
      case 2: rc = launch_var_fe<2>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      case 4: rc = launch_var_fe<4>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      case 6: rc = launch_var_fe<6>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      case 8: rc = launch_var_fe<8>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      default: rc = FAGP_EUNSUPPORTED;
    }
    if (rc) return rc;
    FAGP_LAUNCH_CHECK();
  }
  const size_t msmem = (size_t(b->m) + size_t(MNT) * (W | 1)) * sizeof(double);
  if (msmem > 227 * 1024) return FAGP_EUNSUPPORTED;
  auto go = [&](auto kern) -> int {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(msmem)));
    kern<<<unsigned(ceil_div(Ns, MNT)), MNT, msmem, s>>>(Ts, Ns, view(b), op + pl.KP * pl.NP, mean_const, mean, flags);
    return FAGP_OK;
  };
  int rc;
  switch (b->p) {
    case 2: rc = go(mean_kernel<2>); break;
    case 3: rc = go(mean_kernel<3>); break;
    case 4: rc = go(mean_kernel<4>); break;
    case 5: rc = go(mean_kernel<5>); break;
    case 6: rc = go(mean_kernel<6>); break;
    case 7: rc = go(mean_kernel<7>); break;
    default: rc = go(mean_kernel<8>); break;
  }
  if (rc) return rc;
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // namespace pairk
}  // namespace fagp
