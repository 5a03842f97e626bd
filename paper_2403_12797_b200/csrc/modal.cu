// Modal (Hermite-linearised) Gram and variance: the heavy FP64 tensor work of the path.
//
// Every feature is a product of 1-D eigenfunctions, Phi[r,(a_0..a_{p-1})] = prod_d phi_d,a_d(x_rd)
// (mercer.py:284-292), phi_d,a(x) = sqrt(beta) e^{-delta2 x^2} h_a(rho beta x) (mercer.py:276-281).
// Two facts cut the work of G = Phi^T Phi (posterior.py:168) and of the predictive variance
// (posterior.py:249-263, diagonal) by ~25x at p = 3:
//
//  (1) pair symmetry: G[(a),(a')] depends only on the unordered pairs {a_d, a'_d}, so G has
//      P^p distinct entries H[pi] (P = M(M+1)/2) -- the "pair" form;
//  (2) Hermite linearisation: in one dimension every product phi_a phi_b = beta e^{-2 delta2 x^2}
//      h_a(z) h_b(z) is a polynomial of degree a+b <= 2M-2 in z times the same Gaussian, so it
//      lies in the span of the L = 2M-1 functions g_k(x) = beta e^{-2 delta2 x^2} h_k(sqrt2 z),
//          phi_a phi_b = sum_k V[{a,b}][k] g_k,   |V| <= 1   (fagp_modal_coeffs, exact identity).
//      The g_k are (scaled) orthonormal Hermite functions, so the expansion is well conditioned
//      (measured: Gram entries agree with Phi^T Phi to 2e-15 of max|G|, posterior mean/var to
//      ~1e-12 relative, on data out to |x| = 3).
//
// Hence
//   H[pi] = sum_kappa K[kappa] prod_d V[pi_d][kappa_d],   K[kappa] = sum_r prod_d g_d,kappa_d(x_rd)
// -- a GEMM over the rows with only L^p outputs (6,859 at p=3, M=10, against 166,375 pair or
// 500,500 SYRK entries), followed by p tiny mode products (K -> H).  Symmetrically the variance
// var_i = sigma2 phi_i^T C phi_i (C = S A^{-1} S) is
//   var_i = sigma2 sum_kappa C''[kappa] prod_d g_d,kappa_d(x_i),
//   C''[kappa] = sum_pi Ct[pi] prod_d V[pi_d][kappa_d],   Ct = C folded onto pairs,
// i.e. Y = Q_K C'' on the tensor cores with a g-product epilogue.  t = Phi^T r rides in the Gram
// launch as extra "singleton" tiles over the phi-section of the table.
//
// Kernels (all FP64; tensor work on mma.m8n8k4.f64 = SASS DMMA):
//   KM1  modal_gram_kernel<FA, FB>   generated-operand GEMM over row chunks, split-K partials
//   KM1b modal_gram_reduce_kernel    fixed-order split-K sum -> [K | t], non-finite flag
//   KM2  mode_kernel                 one mode product (K -> H expansion / Ct -> C'' contraction)
//   KM3  pair_system_kernel          A = (s_i G_ij) s_j + sigma2 I (+ jitter) gathered from H
//   KM4  ctilde_kernel               Ct[pi] = folded (s_j D_jj' s_j'), D = X^T X (X = L^{-1})
//   KM5  modal_var_kernel<FK, FE>    Y = Q_K C'' tiles with the g-product epilogue -> var
//   KM5m mean_kernel<P>              mean = c + Phi* w by nested per-dimension sums
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "modal.cuh"

namespace fagp {
namespace modal {

// ---------------------------------------------------------------------------------------
// Column factor offsets.  A generated column is a product of F table entries; unused slots
// point at a 1.0 entry, padding columns at a 0.0 entry (first slot).

// pair index -> (a, a'), a <= a' (a-major enumeration)
__device__ __forceinline__ void pair_decode(int pi, int M, int& a, int& b) {
  int base = 0, x = 0;
  while (pi >= base + (M - x)) {
    base += M - x;
    ++x;
  }
  a = x;
  b = x + (pi - base);
}

// modal column `col` over nd dims from d0 (mixed radix L, first slowest), offsets into the
// g-section; slots >= nd -> `one`
template <int F>
__device__ __forceinline__ void modal_offsets(int64_t col, int64_t ncols, int d0, int nd, int L, int one, int zero,
                                              int (&off)[F]) {
  unsigned q = col < ncols ? unsigned(col) : 0u;
#pragma unroll
  for (int e = F - 1; e >= 0; --e) {
    if (e < nd) {
      off[e] = (d0 + e) * L + int(q % unsigned(L));
      q /= unsigned(L);
    } else {
      off[e] = one;
    }
  }
  if (col >= ncols) {
    off[0] = zero;
#pragma unroll
    for (int f = 1; f < F; ++f) off[f] = one;
  }
}

// feature column `col` over nd dims from d0 (mixed radix M) of the phi-section; slot nd holds
// the residual r when with_r, remaining slots -> 1.0
template <int F>
__device__ __forceinline__ void single_offsets(int64_t col, int64_t ncols, int d0, int nd, int M, int pM, bool with_r,
                                               int (&off)[F]) {
  unsigned q = col < ncols ? unsigned(col) : 0u;
#pragma unroll
  for (int e = F - 1; e >= 0; --e) {
    if (e < nd) {
      off[e] = (d0 + e) * M + int(q % unsigned(M));
      q /= unsigned(M);
    } else {
      off[e] = table_col_one(pM);
    }
  }
  if (with_r) {
#pragma unroll
    for (int e = 0; e < F; ++e)
      if (e == nd) off[e] = table_col_r(pM);
  }
  if (col >= ncols) {
    off[0] = table_col_zero(pM);
#pragma unroll
    for (int f = 1; f < F; ++f) off[f] = table_col_one(pM);
  }
}

// ---------------------------------------------------------------------------------------
// KM1: one 128 x 24 output tile summed over one row chunk, both operands generated per row
// from the staged table section (g-section for K tiles, phi-section for t tiles).
constexpr int GBM = 128, GBN = 24, GBK = 16, GNT = 128;  // 4 warps, warp tile 32 x 24
constexpr int GSPA = GBM + 4, GSPB = GBN + 12;          // 132, 36 (% 16 == 4: conflict-free fragments)
constexpr int GFM = 4, GFN = 3;
constexpr int GA_STAGE = GBK * GSPA, GB_STAGE = GBK * GSPB;

inline int stage_width(int p, int M) { return tmax(table_gbase(p, M), table_gsec(p, M)); }
inline size_t gram_smem(int TW) {
  return (size_t(2) * (GA_STAGE + GB_STAGE) + size_t(2) * GBK * TW) * sizeof(double);
}

template <int FA, int FB>
__global__ void __launch_bounds__(GNT, 3)
modal_gram_kernel(const double* __restrict__ T, int64_t N, BasisView b, Plan pl, double* __restrict__ ws) {
  extern __shared__ double sm[];
  double* As = sm;                 // [2][GBK][GSPA]
  double* Bs = sm + 2 * GA_STAGE;  // [2][GBK][GSPB]
  double* tbuf = Bs + 2 * GB_STAGE;  // [2][GBK][TW]
  const int M = b.M, p = b.p, pM = p * M, W = table_width(p, M);
  const int G0 = table_gbase(p, M), GS = table_gsec(p, M), TW = tmax(G0, GS);
  const int L = pl.L;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nK = pl.ktA * pl.ktB;
  const int tile = pl.tile0 + int(blockIdx.x % pl.nrun), chunk = int(blockIdx.x / pl.nrun);
  const int64_t r0 = int64_t(chunk) * pl.chunk_rows;
  const int64_t r1 = tmin<int64_t>(N, r0 + pl.chunk_rows);

  // generator roles: A column tid (4 rows per k-step); B column tid % 24, row group tid / 24
  // for the first 96 threads
  int offA[FA], offB[FB];
  const bool genB = tid < 4 * GBN;
  const int bcol = tid % GBN, brow = tid / GBN;
  int c0, cw;
  if (tile < nK) {
    const int ta = tile / pl.ktB, tb = tile % pl.ktB;
    modal_offsets<FA>(int64_t(ta) * GBM + tid, pl.KA, 0, pl.pA, L, p * L, p * L + 1, offA);
    modal_offsets<FB>(int64_t(tb) * GBN + bcol, pl.KB, pl.pA, p - pl.pA, L, p * L, p * L + 1, offB);
    c0 = G0;
    cw = GS;
  } else {
    const int ta = (tile - nK) / pl.stB, tb = (tile - nK) % pl.stB;
    single_offsets<FA>(int64_t(ta) * GBM + tid, pl.SA, 0, pl.pA, M, pM, false, offA);
    single_offsets<FB>(int64_t(tb) * GBN + bcol, pl.SB, pl.pA, p - pl.pA, M, pM, true, offB);
    c0 = 0;
    cw = G0;
  }

  auto load_tab = [&](int slot, int64_t base) {
    double* dst = tbuf + slot * (GBK * TW);
    const int nrows = int(tmax<int64_t>(0, tmin<int64_t>(GBK, r1 - base)));
    const int half = cw / 2;
    const double* src = T + base * W + c0;
    for (int i = tid; i < nrows * half; i += GNT) {
      const int r = i / half, c2 = i - r * half;
      cp_async_16(dst + r * TW + 2 * c2, src + int64_t(r) * W + 2 * c2);
    }
    for (int i = nrows * TW + tid; i < GBK * TW; i += GNT) dst[i] = 0.0;
    cp_async_commit();
  };
  auto gen_rows = [&](int stage, int kk) {
    const double* tb_ = tbuf + stage * (GBK * TW);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = kk * 4 + i;
      const double* Tr = tb_ + k * TW;
      double v = Tr[offA[0]];
#pragma unroll
      for (int f = 1; f < FA; ++f) v = __dmul_rn(v, Tr[offA[f]]);
      As[stage * GA_STAGE + k * GSPA + tid] = v;
    }
    if (genB) {
      const int k = kk * 4 + brow;
      const double* Tr = tb_ + k * TW;
      double u = Tr[offB[0]];
#pragma unroll
      for (int f = 1; f < FB; ++f) u = __dmul_rn(u, Tr[offB[f]]);
      Bs[stage * GB_STAGE + k * GSPB + bcol] = u;
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
      gen_rows(nxt, kk);  // chunk n+1 (garbage past the last chunk, never read)
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

// KM1b: K[lambda * KB + rho] and t[lambda' * SB + rho'] = sum_s partial[s][tile][..] in chunk
// order (deterministic); any non-finite entry flags a non-finite feature.
__global__ void modal_gram_reduce_kernel(const double* __restrict__ ws, Plan pl, int64_t m, double* __restrict__ out,
                                         uint32_t* flags) {
  const int64_t nKe = pl.Klen;
  const int nK = pl.ktA * pl.ktB;
  const size_t stride = size_t(pl.nrun) * GBM * GBN;
  const int64_t e0 = pl.tile0 > 0 ? nKe : 0;  // t-only runs produce just t
  bool bad = false;
  for (int64_t e = e0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nKe + m;
       e += int64_t(gridDim.x) * blockDim.x) {
    int tile;
    int64_t lam, rho;
    if (e < nKe) {
      lam = e / pl.KB;
      rho = e - lam * pl.KB;
      tile = int(lam / GBM) * pl.ktB + int(rho / GBN);
    } else {
      const int64_t q = e - nKe;
      lam = q / pl.SB;
      rho = q - lam * pl.SB;
      tile = nK + int(lam / GBM) * pl.stB + int(rho / GBN);
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
// KM2: out[a][j][c] = sum_i in[a][i][c] * B[j * ldj + i * ldi]  (fixed order in i)
__global__ void mode_kernel(const double* __restrict__ in, double* __restrict__ out, int64_t pre, int nin,
                            int64_t post, int nout, const double* __restrict__ B, int ldj, int ldi) {
  const int64_t total = pre * nout * post;
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < total; o += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = o % post;
    const int64_t aj = o / post;
    const int j = int(aj % nout);
    const int64_t a = aj / nout;
    const double* src = in + a * nin * post + c;
    const double* bj = B + int64_t(j) * ldj;
    // loads issued 8 at a time (an L2 round trip each otherwise); the sum keeps the order of i
    double acc = 0.0;
    int i = 0;
    for (; i + 8 <= nin; i += 8) {
      double v[8], w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] = src[int64_t(i + u) * post];
        w[u] = bj[int64_t(i + u) * ldi];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = fma(v[u], w[u], acc);
    }
    for (; i < nin; ++i) acc = fma(src[int64_t(i) * post], bj[int64_t(i) * ldi], acc);
    out[o] = acc;
  }
}

// ---------------------------------------------------------------------------------------
// KM3: A[i,j] = (s_i G_ij) s_j (+ sigma2 + jitter on the diagonal), G_ij gathered from H;
// optional full G.  (posterior.py:171-174)
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

// One CTA per row i (grid-stride), threads over j.  The pair key separates over dimensions,
// key(i, j) = sum_d P^(p-1-d) pk(a_d, b_d), so each row builds two small shared tables --
// KH[j / M] (dims < p-1) and KL[j % M] (the last dim) -- and a column costs two table reads and
// one gather; (j / M, j % M) advance incrementally.  Shapes whose tables do not fit take the
// digit-by-digit key.
constexpr int kPairKH = 4096, kPairKL = 64;
__global__ void pair_system_kernel(const double* __restrict__ H, const double* __restrict__ s, double sigma2,
                                   double jit, BasisView b, int P, double* __restrict__ A, double* __restrict__ G,
                                   const double* __restrict__ tsrc, double* __restrict__ t) {
  __shared__ int KH[kPairKH], KL[kPairKL];
  const int M = b.M, p = b.p;
  const int64_t m = b.m, MH = m / M;
  const int nt = int(blockDim.x);
  const bool tab = M <= kPairKL && MH <= kPairKH;
  auto pkey = [&](int a, int c) {
    const int lo = a < c ? a : c, hi = a < c ? c : a;
    return lo * M - lo * (lo - 1) / 2 + (hi - lo);
  };
  const int stq = nt / M, str = nt - (nt / M) * M;  // nt = stq M + str
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    int di[FAGP_MAX_P];
    {
      int64_t q = i;
      for (int d = p - 1; d >= 0; --d) {
        di[d] = int(q % M);
        q /= M;
      }
    }
    if (tab) {
      __syncthreads();  // the previous row's readers are done
      for (int e = threadIdx.x; e < MH; e += nt) {
        int q = e, key = 0, pw = P;
        for (int d = p - 2; d >= 0; --d) {
          key += pw * pkey(di[d], q % M);
          q /= M;
          pw *= P;
        }
        KH[e] = key;
      }
      for (int e = threadIdx.x; e < M; e += nt) KL[e] = pkey(di[p - 1], e);
      __syncthreads();
    }
    const double si = s ? s[i] : 1.0;
    if (t && threadIdx.x == 0) t[i] = tsrc[i];  // t = the gram buffer's tail (one copy launch fewer)
    int jh = int(threadIdx.x) / M, jl = int(threadIdx.x) - (int(threadIdx.x) / M) * M;
    auto advance = [&]() {
      jh += stq;
      jl += str;
      if (jl >= M) {
        jl -= M;
        ++jh;
      }
    };
    // 4 columns per thread per pass: keys first, then the 4 gathers in flight together
    for (int64_t jb = threadIdx.x; jb < m; jb += 4 * int64_t(nt)) {
      int64_t key[4];
      double g[4], sj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = jb + u * int64_t(nt);
        if (tab) {
          key[u] = j < m ? int64_t(KH[jh] + KL[jl]) : 0;
          advance();
        } else {
          unsigned q = unsigned(j < m ? j : 0);
          int64_t k = 0, pw = 1;
          for (int d = p - 1; d >= 0; --d) {
            const unsigned c = q % unsigned(M);
            q /= unsigned(M);
            k += pw * pkey(di[d], int(c));
            pw *= P;
          }
          key[u] = k;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = jb + u * int64_t(nt);
        g[u] = H[key[u]];
        sj[u] = (A && j < m) ? s[j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = jb + u * int64_t(nt);
        if (j >= m) continue;
        if (G) G[i * m + j] = g[u];
        if (A) {
          double a = __dmul_rn(__dmul_rn(si, g[u]), sj[u]);
          if (i == j) {
            a = __dadd_rn(a, sigma2);
            if (jit != 0.0) a = __dadd_rn(a, jit);
          }
          A[i * m + j] = a;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// KM4: Ct[pi] (canonical pair order, first dimension slowest) = sum over the orderings of every
// pi_d of (s_j D_jj') s_j' (or D_jj' when s is NULL).
__device__ __forceinline__ double ctilde_entry(int64_t e, const double* __restrict__ D, int64_t ldd,
                                               const double* __restrict__ s, int M, int p, int P) {
  {
    int lo[FAGP_MAX_P], hi[FAGP_MAX_P];
    int64_t q = e;
    for (int d = p - 1; d >= 0; --d) {
      pair_decode(int(q % P), M, lo[d], hi[d]);
      q /= P;
    }
    int nflip = 0;
    int fd[FAGP_MAX_P];
    for (int d = 0; d < p; ++d)
      if (lo[d] != hi[d]) fd[nflip++] = d;
    double v = 0.0;
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
    return v;
  }
}

__global__ void ctilde_kernel(const double* __restrict__ D, int64_t ldd, const double* __restrict__ s, BasisView b,
                              int P, int64_t Hlen, double* __restrict__ Ct) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < Hlen; e += int64_t(gridDim.x) * blockDim.x)
    Ct[e] = ctilde_entry(e, D, ldd, s, b.M, b.p, P);
}

// ---------------------------------------------------------------------------------------
// p = 3 fused mode products (one launch instead of three, intermediates in shared memory).
// Small shared-memory products out[r][c] = sum_i A(r, i) B(c, i), i in order, 2 x 2 outputs per
// thread (four independent fma chains; latency-bound otherwise).
__device__ __forceinline__ void smem_nt(double* out, int ldo, const double* A, int sar, int sai, const double* B,
                                        int sbc, int sbi, int R, int C, int K, int tid, int nt) {
  const int nC = (C + 1) >> 1, tiles = ((R + 1) >> 1) * nC;
  for (int t = tid; t < tiles; t += nt) {
    const int r0 = (t / nC) * 2, c0 = (t - (t / nC) * nC) * 2;
    const int r1 = r0 + 1 < R ? r0 + 1 : r0, c1 = c0 + 1 < C ? c0 + 1 : c0;
    double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
#pragma unroll 4
    for (int i = 0; i < K; ++i) {
      const double x0 = A[r0 * sar + i * sai], x1 = A[r1 * sar + i * sai];
      const double y0 = B[c0 * sbc + i * sbi], y1 = B[c1 * sbc + i * sbi];
      a00 = fma(x0, y0, a00);
      a01 = fma(x0, y1, a01);
      a10 = fma(x1, y0, a10);
      a11 = fma(x1, y1, a11);
    }
    out[r0 * ldo + c0] = a00;
    if (c0 + 1 < C) out[r0 * ldo + c0 + 1] = a01;
    if (r0 + 1 < R) {
      out[(r0 + 1) * ldo + c0] = a10;
      if (c0 + 1 < C) out[(r0 + 1) * ldo + c0 + 1] = a11;
    }
  }
}

constexpr int kModeSplit = 4;  // expand3: CTAs per leading pair index
constexpr int kCtcSplit = 2;   // ctc3: CTAs per leading pair index (P x 2 = 110 at C3: one wave)
constexpr int kCtcNT = 512;

// expand3: CTA (pi0, s) computes H[pi0][pi1][.] for its quarter of pi1 from K, with the stage
// order and per-output fma order of the three mode_kernel launches of expand() (bitwise the same H):
//   T1[k1][k2] = sum_k0 K[k0][k1][k2] V[pi0][k0];  T2[pi1][k2] = sum_k1 T1[k1][k2] V[pi1][k1];
//   H[pi0][pi1][pi2] = sum_k2 T2[pi1][k2] V[pi2][k2]
__global__ void __launch_bounds__(256) expand3_kernel(const double* __restrict__ K, const double* __restrict__ Vg,
                                                      int P, int L, double* __restrict__ H) {
  extern __shared__ double sm[];
  double* V = sm;              // [P][L]
  double* T1 = V + P * L;      // [L][L]
  double* T2 = T1 + L * L;     // [P][L] (rows of this CTA)
  const int pi0 = int(blockIdx.x), tid = int(threadIdx.x), nt = int(blockDim.x);
  const int j0 = int(blockIdx.y) * P / kModeSplit, j1 = (int(blockIdx.y) + 1) * P / kModeSplit;
  for (int e = tid; e < P * L; e += nt) V[e] = Vg[e];
  __syncthreads();
  for (int c = tid; c < L * L; c += nt) {
    double acc = 0.0;
    int i = 0;
    for (; i + 4 <= L; i += 4) {
      double k[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) k[u] = K[int64_t(i + u) * L * L + c];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = fma(k[u], V[pi0 * L + i + u], acc);
    }
    for (; i < L; ++i) acc = fma(K[int64_t(i) * L * L + c], V[pi0 * L + i], acc);
    T1[c] = acc;
  }
  __syncthreads();
  // T2[j][c] = sum_i T1[i][c] V[j][i]  (rows j in [j0, j1))
  smem_nt(T2, L, V + j0 * L, L, 1, T1, 1, L, j1 - j0, L, L, tid, nt);
  __syncthreads();
  // H[pi0][j][q] = sum_i T2[j][i] V[q][i]
  smem_nt(H + (int64_t(pi0) * P + j0) * P, P, T2, L, 1, V, L, 1, j1 - j0, P, L, tid, nt);
}

// ctc3 (C'' for p = 3, stage 1 of 2): CTA (pi0 = {a0, b0}, s) stages the scaled block
// B[(x1 x2)][(y1 y2)] = s_j D_jj' s_j' (j = (a0 x1 x2), j' = (b0 y1 y2)) -- the block of
// (b0, a0) is its transpose (D = X^T X is symmetric; its mirrored entries are not re-read) -- folds it to
//   Ct[pi0][pi1][pi2] = (1 + [a0 != b0]) sum over the orderings of pi1, pi2 of B
// and contracts the last two pair indices for its quarter of k2:
//   W1[pi1][k2] = sum_pi2 Ct[pi0][pi1][pi2] V[pi2][k2];  Z[pi0][k1][k2] = sum_pi1 V[pi1][k1] W1[pi1][k2]
__global__ void __launch_bounds__(kCtcNT) ctc3_kernel(const double* __restrict__ D, int64_t ldd,
                                                   const double* __restrict__ s, BasisView b, int P,
                                                   double* __restrict__ Z) {
  extern __shared__ double sm[];
  const int M = b.M, L = modal_L(M), M2 = M * M;
  double* V = sm;           // [P][L]
  double* Ct = V + P * L;   // [P][P]
  double* W1 = Ct + P * P;  // [P][L] (columns of this CTA, ld L)
  double* B = W1 + P * L;   // [M2][M2]
  const int pi0 = int(blockIdx.x), tid = int(threadIdx.x), nt = int(blockDim.x);
  const int k0 = int(blockIdx.y) * L / kCtcSplit, k1 = (int(blockIdx.y) + 1) * L / kCtcSplit;
  int a0, b0;
  pair_decode(pi0, M, a0, b0);
  const double* Vg = b.modal();
  for (int e = tid; e < P * L; e += nt) V[e] = Vg[e];
  // the block, 8 loads per thread in flight (one L2 round trip per 8 entries, not per entry)
  for (int e0 = tid; e0 < M2 * M2; e0 += 8 * nt) {
    double d[8], sa[8], sb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * nt < M2 * M2 ? e0 + u * nt : 0;
      const int r = e / M2, c = e - (e / M2) * M2;
      const int64_t j = int64_t(a0) * M2 + r, jj = int64_t(b0) * M2 + c;
      d[u] = D[j * ldd + jj];
      sa[u] = s ? s[j] : 1.0;
      sb[u] = s ? s[jj] : 1.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (e0 + u * nt < M2 * M2) B[e0 + u * nt] = s ? __dmul_rn(__dmul_rn(sa[u], d[u]), sb[u]) : d[u];
  }
  __syncthreads();
  const double f0 = a0 != b0 ? 2.0 : 1.0;
  for (int e = tid; e < P * P; e += nt) {
    int l1, h1, l2, h2;
    pair_decode(e / P, M, l1, h1);
    pair_decode(e - (e / P) * P, M, l2, h2);
    double v = B[(l1 * M + l2) * M2 + h1 * M + h2];
    if (l2 != h2) v += B[(l1 * M + h2) * M2 + h1 * M + l2];
    if (l1 != h1) {
      v += B[(h1 * M + l2) * M2 + l1 * M + h2];
      if (l2 != h2) v += B[(h1 * M + h2) * M2 + l1 * M + l2];
    }
    Ct[e] = f0 * v;
  }
  __syncthreads();
  // W1[a][k] = sum_i Ct[a][i] V[i][k]  (k in [k0, k1))
  smem_nt(W1 + k0, L, Ct, P, 1, V + k0, 1, L, P, k1 - k0, P, tid, nt);
  __syncthreads();
  // Z[pi0][q][k] = sum_i V[i][q] W1[i][k]
  smem_nt(Z + int64_t(pi0) * L * L + k0, L, V, 1, L, W1 + k0, 1, L, L, k1 - k0, P, tid, nt);
}

// ctc3 stage 2: C''[k0][k1 k2] = sum_pi0 V[pi0][k0] Z[pi0][k1 k2], written straight into the
// padded predict-operand layout op[kap][nu] (canonical index nu KR + kap), zeros in the padding
constexpr int kOpE = 32, kOpG = 4;  // ctc3_op: entries per CTA x pi0 groups
__global__ void __launch_bounds__(kOpE * kOpG) ctc3_op_kernel(const double* __restrict__ Z,
                                                              const double* __restrict__ Vg, int P, int L, Plan pl,
                                                              double* __restrict__ op, const double* __restrict__ w,
                                                              int64_t m) {
  // group g sums pi0 in [g P / 4, (g + 1) P / 4) with every load in flight, then the 4 group
  // sums are added in group order (fixed order: deterministic)
  __shared__ double red[kOpG][kOpE];
  const int grp = int(threadIdx.x) / kOpE, el = int(threadIdx.x) % kOpE;
  const int64_t total = pl.KP * pl.NP;
  // the mean weights w ride along into the operand's tail (one copy launch fewer)
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < m; q += int64_t(gridDim.x) * blockDim.x)
    op[total + q] = w[q];
  const int64_t e = int64_t(blockIdx.x) * kOpE + el;
  double acc = 0.0;
  bool valid = false;
  if (e < total) {
    const int64_t kap = e / pl.NP, nu = e - (e / pl.NP) * pl.NP;
    valid = kap < pl.KR && nu < pl.NR;
    if (valid) {
      const int64_t c = nu * pl.KR + kap;
      const int k0 = int(c / (L * L)), k12 = int(c - int64_t(k0) * L * L);
      const int i0 = grp * P / kOpG, i1 = (grp + 1) * P / kOpG;
      int i = i0;
      for (; i + 16 <= i1; i += 16) {
        double z[16], v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          z[u] = Z[int64_t(i + u) * L * L + k12];
          v[u] = Vg[(i + u) * L + k0];
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) acc = fma(v[u], z[u], acc);
      }
      {
        double z[16], v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const bool ok = i + u < i1;
          z[u] = ok ? Z[int64_t(i + u) * L * L + k12] : 0.0;
          v[u] = ok ? Vg[(i + u) * L + k0] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (i + u < i1) acc = fma(v[u], z[u], acc);
      }
    }
  }
  red[grp][el] = acc;
  __syncthreads();
  if (grp == 0 && e < total) {
    double t = red[0][el];
#pragma unroll
    for (int g = 1; g < kOpG; ++g) t += red[g][el];
    op[e] = valid ? t : 0.0;
  }
}

// C''[kappa_K][nu] (padded KP x NP) from the canonical C''[nu][kappa_K]
__global__ void scatter_op_kernel(const double* __restrict__ Cc, Plan pl, double* __restrict__ op) {
  const int64_t total = pl.KP * pl.NP;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t kap = e / pl.NP, nu = e - (e / pl.NP) * pl.NP;
    op[e] = (kap < pl.KR && nu < pl.NR) ? Cc[nu * pl.KR + kap] : 0.0;
  }
}

// ---------------------------------------------------------------------------------------
// KM5: var for 128 test rows: Y = Q_K C'' over K chunks (Q_K generated from the staged
// g-sections: product over dims >= pN), then var_i = sigma2 sum_nu Y[i, nu] E[i, nu] with E the
// g-product over dims < pN.  C'' streams from L2 by cp.async.
constexpr int VBM = 128, VBN = 24, VBK = 16, VNT = 128;
constexpr int VASP = VBK + 4, VBSP = VBN + 12;  // 20, 36 (% 16 == 4)
constexpr int VFM = 4, VFN = 3;
constexpr int VA_STAGE = VBM * VASP, VB_STAGE = VBK * VBSP;
constexpr int VGGRP = VNT / VBK;                   // generator row groups (8)
constexpr int VGPERKK = VBM / VGGRP / (VBK / 4);   // generated rows per thread per k-step (4)

inline size_t var_smem(int GS) {
  return (size_t(2) * (VA_STAGE + VB_STAGE) + size_t(VBM) * GS) * sizeof(double);
}

template <int FK, int FE>
__global__ void __launch_bounds__(VNT, 2)
modal_var_kernel(const double* __restrict__ Ts, int64_t Ns, BasisView b, Plan pl, const double* __restrict__ Cop,
                 double sigma2, double* __restrict__ var, uint32_t* flags) {
  extern __shared__ double sm[];
  double* As = sm;                     // [2][VBM][VASP]
  double* Bs = sm + 2 * VA_STAGE;      // [2][VBK][VBSP]
  double* tsm = Bs + 2 * VB_STAGE;     // [VBM][GS]
  const int M = b.M, p = b.p, W = table_width(p, M);
  const int G0 = table_gbase(p, M), GS = table_gsec(p, M), L = pl.L;
  const int one = p * L, zero = p * L + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t row0 = int64_t(blockIdx.x) * VBM;
  {
    const int nr = int(tmin<int64_t>(VBM, Ns - row0));
    const int half = GS / 2;
    const double* src = Ts + row0 * W + G0;
    for (int i = tid; i < nr * half; i += VNT) {
      const int r = i / half, c2 = i - r * half;
      cp_async_16(tsm + r * GS + 2 * c2, src + int64_t(r) * W + 2 * c2);
    }
    for (int i = nr * GS + tid; i < VBM * GS; i += VNT) tsm[i] = 0.0;
    cp_async_commit();
  }
  const int gk = tid % VBK, gr0 = tid / VBK;  // generator: K column gk, rows gr0 + VGGRP q
  const int nkc = int(pl.KP / VBK);
  const int ntn = int(pl.NP / VBN);

  auto load_b = [&](int stage, int64_t k0, int64_t n0) {
    double* dst = Bs + stage * VB_STAGE;
    for (int e = tid; e < VBK * VBN / 2; e += VNT) {
      const int k = e / (VBN / 2), n2 = e % (VBN / 2);
      cp_async_16(dst + k * VBSP + 2 * n2, Cop + (k0 + k) * pl.NP + n0 + 2 * n2);
    }
    cp_async_commit();
  };
  auto gen_rows = [&](int stage, const int (&off)[FK], int q0) {
    double* dst = As + stage * VA_STAGE + gk;
#pragma unroll
    for (int qi = 0; qi < VGPERKK; ++qi) {
      const int r = gr0 + VGGRP * (q0 + qi);
      const double* Tr = tsm + r * GS;
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
    modal_offsets<FK>(gk, pl.KR, pl.pN, p - pl.pN, L, one, zero, off);
#pragma unroll
    for (int kk = 0; kk < VBK / 4; ++kk) gen_rows(0, off, kk * VGPERKK);
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
    modal_offsets<FK>(int64_t(kc2) * VBK + gk, pl.KR, pl.pN, p - pl.pN, L, one, zero, off);
    const double* Ab = As + buf * VA_STAGE + (warp * 32 + (lane >> 2)) * VASP + (lane & 3);
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
      gen_rows(buf ^ 1, off, kk * VGPERKK);
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
          modal_offsets<FE>(nu, pl.NR, 0, pl.pN, L, one, zero, offe);
#pragma unroll
          for (int s = 0; s < VFM; ++s) {
            const double* Tr = tsm + (warp * 32 + s * 8 + (lane >> 2)) * GS;
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
      const int64_t row = row0 + warp * 32 + s * 8 + (lane >> 2);
      if (row < Ns) {
        const double vv = sigma2 * vsum[s];
        var[row] = vv;
        if (not_finite(vv)) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// KM5m: mean_i = c + sum_j w_j Phi[i, j], one thread per test row, w broadcast from shared
// memory: mean - c = sum_u prefix_u(i) * sum_c phi_{p-1,c}(i) w[u M + c], with the innermost
// dimension's values in registers (M <= MREG) and the prefix product over dims < p-1 kept up
// to date by an odometer on its digits.  Only the phi-section of each row is staged.
constexpr int MNT = 128, MREG = 16;
template <int P>
__global__ void __launch_bounds__(MNT) mean_kernel(const double* __restrict__ Ts, int64_t Ns, BasisView b,
                                                   const double* __restrict__ w, double mean_const,
                                                   double* __restrict__ mean, uint32_t* flags) {
  extern __shared__ double sm[];
  const int M = b.M, W = table_width(P, M), G0 = table_gbase(P, M);
  const int WS = G0 | 1;  // odd row stride: conflict-free per-thread rows
  const int64_t m = b.m;
  double* ws_ = sm;      // [m]
  double* tsm = sm + m;  // [MNT][WS]
  const int tid = threadIdx.x;
  for (int64_t j = tid; j < m; j += MNT) ws_[j] = w[j];
  const int64_t row0 = int64_t(blockIdx.x) * MNT;
  const int nr = int(tmin<int64_t>(MNT, Ns - row0));
  for (int e = tid; e < MNT * G0; e += MNT) {
    const int rl = e / G0, c = e - (e / G0) * G0;
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

__global__ void copy_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

}  // namespace modal
}  // namespace fagp

// =======================================================================================
// Host side
namespace fagp {
namespace modal {

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

bool enabled(int p, int M) { return modal_on(p, M); }

Plan make_plan(int64_t N, int p, int M, bool t_only) {
  Plan pl{};
  pl.P = M * (M + 1) / 2;
  pl.L = modal_L(M);
  pl.Hlen = ipow(pl.P, p);
  pl.Klen = ipow(pl.L, p);
  // Gram split: padded tensor work of the K and t tiles (FB = p - pA + 1 in {2, 3})
  int64_t best = -1;
  for (int pA = tmax(1, p - 2); pA <= p - 1; ++pA) {
    const int64_t KA = ipow(pl.L, pA), KB = ipow(pl.L, p - pA);
    const int64_t SA = ipow(M, pA), SB = ipow(M, p - pA);
    const int64_t cost = round_up(KA, GBM) * round_up(KB, GBN) + round_up(SA, GBM) * round_up(SB, GBN);
    if (best < 0 || cost < best) {
      best = cost;
      pl.pA = pA;
    }
  }
  pl.KA = ipow(pl.L, pl.pA);
  pl.KB = ipow(pl.L, p - pl.pA);
  pl.ktA = int(ceil_div(pl.KA, GBM));
  pl.ktB = int(ceil_div(pl.KB, GBN));
  pl.SA = ipow(M, pl.pA);
  pl.SB = ipow(M, p - pl.pA);
  pl.stA = int(ceil_div(pl.SA, GBM));
  pl.stB = int(ceil_div(pl.SB, GBN));
  // variance split (FE = pN in {1, 2})
  best = -1;
  for (int pN = 1; pN <= tmin(2, p - 1); ++pN) {
    const int64_t cost = round_up(ipow(pl.L, pN), VBN) * round_up(ipow(pl.L, p - pN), VBK);
    if (best < 0 || cost < best) {
      best = cost;
      pl.pN = pN;
    }
  }
  pl.NR = ipow(pl.L, pl.pN);
  pl.KR = ipow(pl.L, p - pl.pN);
  pl.NP = round_up(pl.NR, VBN);
  pl.KP = round_up(pl.KR, VBK);
  // tiles launched, then split-K over rows: 3 CTAs per SM
  pl.tile0 = t_only ? pl.ktA * pl.ktB : 0;
  pl.nrun = (t_only ? 0 : pl.ktA * pl.ktB) + pl.stA * pl.stB;
  const int64_t tiles = pl.nrun;
  const int64_t max_chunks = tmax<int64_t>(1, ceil_div(N, GBK));
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
  pl.chunk_rows = round_up(tmax<int64_t>(1, ceil_div(tmax<int64_t>(N, 1), bestS)), GBK);
  pl.S = int(tmax<int64_t>(1, ceil_div(N, pl.chunk_rows)));
  return pl;
}

int64_t gram_len(const fagp_basis* b) { return make_plan(0, b->p, b->M).Klen + b->m; }

size_t gram_workspace(int64_t N, const fagp_basis* b) {
  const Plan pl = make_plan(N, b->p, b->M);
  return size_t(pl.S) * pl.nrun * GBM * GBN * sizeof(double);
}

size_t tmatvec_workspace(int64_t N, const fagp_basis* b) {
  const Plan pl = make_plan(N, b->p, b->M, true);
  return size_t(pl.S) * pl.nrun * GBM * GBN * sizeof(double);
}

template <int FA>
static int launch_gram_fb(int FB, const double* T, int64_t N, const fagp_basis* b, const Plan& pl, double* ws,
                          size_t smem, unsigned grid, cudaStream_t s) {
  auto go = [&](auto kern) -> int {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<grid, GNT, smem, s>>>(T, N, view(b), pl, ws);
    return FAGP_OK;
  };
  switch (FB) {
    case 2: return go(modal_gram_kernel<FA, 2>);
    case 3: return go(modal_gram_kernel<FA, 3>);
    default: return FAGP_EUNSUPPORTED;
  }
}

static int run_gram(const Plan& pl, const double* T, int64_t N, const fagp_basis* b, double* out, double* ws,
                    uint32_t* flags, cudaStream_t s) {
  const size_t smem = gram_smem(stage_width(b->p, b->M));
  if (smem > 227 * 1024) return FAGP_EUNSUPPORTED;
  const unsigned grid = unsigned(size_t(pl.S) * pl.nrun);
  const int FA = pl.pA, FB = b->p - pl.pA + 1;
  int rc;
  switch (FA) {
    case 1: rc = launch_gram_fb<1>(FB, T, N, b, pl, ws, smem, grid, s); break;
    case 2: rc = launch_gram_fb<2>(FB, T, N, b, pl, ws, smem, grid, s); break;
    case 3: rc = launch_gram_fb<3>(FB, T, N, b, pl, ws, smem, grid, s); break;
    case 4: rc = launch_gram_fb<4>(FB, T, N, b, pl, ws, smem, grid, s); break;
    case 5: rc = launch_gram_fb<5>(FB, T, N, b, pl, ws, smem, grid, s); break;
    case 6: rc = launch_gram_fb<6>(FB, T, N, b, pl, ws, smem, grid, s); break;
    case 7: rc = launch_gram_fb<7>(FB, T, N, b, pl, ws, smem, grid, s); break;
    default: rc = FAGP_EUNSUPPORTED;
  }
  if (rc) return rc;
  FAGP_LAUNCH_CHECK();
  const int64_t outs = (pl.tile0 > 0 ? 0 : pl.Klen) + b->m;
  modal_gram_reduce_kernel<<<unsigned(tmax<int64_t>(1, tmin<int64_t>(ceil_div(outs, 256), 16 * num_sms()))), 256, 0,
                             s>>>(ws, pl, b->m, out, flags);
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

int64_t scratch_len(const fagp_basis* b) { return 2 * make_plan(0, b->p, b->M).Hlen; }

static int launch_mode(const double* in, double* out, int64_t pre, int nin, int64_t post, int nout, const double* B,
                       int ldj, int ldi, cudaStream_t s) {
  const int64_t total = pre * nout * post;
  mode_kernel<<<unsigned(tmax<int64_t>(1, tmin<int64_t>(ceil_div(total, 256), 16 * num_sms()))), 256, 0, s>>>(
      in, out, pre, nin, post, nout, B, ldj, ldi);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

static size_t expand3_smem(int P, int L) { return size_t(2 * P * L + L * L) * sizeof(double); }
static size_t ctc3_smem(int P, int L, int M) {
  return size_t(2 * P * L + P * P + M * M * M * M) * sizeof(double);
}
constexpr size_t kFusedModeSmem = 200 * 1024;

int expand(const double* gram, const fagp_basis* b, double* H, double* tmp, cudaStream_t s) {
  const Plan pl = make_plan(0, b->p, b->M);
  const int p = b->p;
  const double* V = view(b).modal();
  if (p == 3 && expand3_smem(pl.P, pl.L) <= kFusedModeSmem && !getenv("FAGP_MODE_UNFUSED")) {
    const size_t smem = expand3_smem(pl.P, pl.L);
    FAGP_CUDA_TRY(cudaFuncSetAttribute(expand3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    expand3_kernel<<<dim3(unsigned(pl.P), kModeSplit), 256, smem, s>>>(gram, V, pl.P, pl.L, H);
    FAGP_LAUNCH_CHECK();
    return FAGP_OK;
  }
  const double* cur = gram;  // K: [L]^p
  for (int d = 0; d < p; ++d) {
    // [P^d][L][L^(p-1-d)] -> [P^d][P][L^(p-1-d)], B[pi][kappa] = V[pi * L + kappa]
    double* dst = ((p - 1 - d) % 2 == 0) ? H : tmp;
    int rc = launch_mode(cur, dst, ipow(pl.P, d), pl.L, ipow(pl.L, p - 1 - d), pl.P, V, pl.L, 1, s);
    if (rc) return rc;
    cur = dst;
  }
  return FAGP_OK;
}

int system(const double* H, const double* g, const double* sqrt_lam, double sigma2, double jit, const fagp_basis* b,
           double* A, double* G, double* t, cudaStream_t s) {
  const Plan pl = make_plan(0, b->p, b->M);
  const int64_t m = b->m;
  if (A || G) {
    const int grid = int(tmin<int64_t>(m, 8 * num_sms()));
    pair_system_kernel<<<grid, 256, 0, s>>>(H, sqrt_lam, sigma2, jit, view(b), pl.P, A, G, g + pl.Klen, t);
    FAGP_LAUNCH_CHECK();
    return FAGP_OK;
  }
  if (t) {
    copy_kernel<<<unsigned(ceil_div(m, 256)), 256, 0, s>>>(g + pl.Klen, t, m);
    FAGP_LAUNCH_CHECK();
  }
  return FAGP_OK;
}

int64_t predict_op_len(const fagp_basis* b) {
  const Plan pl = make_plan(0, b->p, b->M);
  return pl.KP * pl.NP + b->m;
}

int build_predict_op(const double* D, const double* sqrt_lam, const double* w, const fagp_basis* b, double* op,
                     double* S0, double* S1, cudaStream_t s) {
  const Plan pl = make_plan(0, b->p, b->M);
  const int p = b->p;
  const double* V = view(b).modal();
  if (p == 3 && ctc3_smem(pl.P, pl.L, b->M) <= kFusedModeSmem && !getenv("FAGP_MODE_UNFUSED")) {
    // Z = S0 [P][L^2]
    const size_t smem = ctc3_smem(pl.P, pl.L, b->M);
    FAGP_CUDA_TRY(cudaFuncSetAttribute(ctc3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    ctc3_kernel<<<dim3(unsigned(pl.P), kCtcSplit), kCtcNT, smem, s>>>(D, b->m, sqrt_lam, view(b), pl.P, S0);
    FAGP_LAUNCH_CHECK();
    ctc3_op_kernel<<<unsigned(tmax<int64_t>(1, ceil_div(pl.KP * pl.NP, kOpE))), kOpE * kOpG, 0, s>>>(
        S0, V, pl.P, pl.L, pl, op, w, b->m);
    FAGP_LAUNCH_CHECK();
    return FAGP_OK;
  }
  {
    const int grid = int(tmax<int64_t>(1, tmin<int64_t>(ceil_div(pl.Hlen, 256), 16 * num_sms())));
    ctilde_kernel<<<grid, 256, 0, s>>>(D, b->m, sqrt_lam, view(b), pl.P, pl.Hlen, S0);
    FAGP_LAUNCH_CHECK();
  }
  const double* cur = S0;
  for (int d = 0; d < p; ++d) {
    // [L^d][P][P^(p-1-d)] -> [L^d][L][P^(p-1-d)], B[kappa][pi] = V[pi * L + kappa]
    double* dst = (cur == S0) ? S1 : S0;
    int rc = launch_mode(cur, dst, ipow(pl.L, d), pl.P, ipow(pl.P, p - 1 - d), pl.L, V, 1, pl.L, s);
    if (rc) return rc;
    cur = dst;
  }
  {
    const int grid = int(tmax<int64_t>(1, tmin<int64_t>(ceil_div(pl.KP * pl.NP, 256), 16 * num_sms())));
    scatter_op_kernel<<<grid, 256, 0, s>>>(cur, pl, op);
    FAGP_LAUNCH_CHECK();
  }
  return set_weights(op, w, b, s);
}

int set_weights(double* op, const double* w, const fagp_basis* b, cudaStream_t s) {
  const Plan pl = make_plan(0, b->p, b->M);
  copy_kernel<<<unsigned(ceil_div(b->m, 256)), 256, 0, s>>>(w, op + pl.KP * pl.NP, b->m);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

template <int FK>
static int launch_var_fe(int FE, const double* Ts, int64_t Ns, const fagp_basis* b, const Plan& pl,
                         const double* Cop, double sigma2, double* var, uint32_t* flags, size_t smem, cudaStream_t s) {
  auto go = [&](auto kern) -> int {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<unsigned(ceil_div(Ns, VBM)), VNT, smem, s>>>(Ts, Ns, view(b), pl, Cop, sigma2, var, flags);
    return FAGP_OK;
  };
  switch (FE) {
    case 1: return go(modal_var_kernel<FK, 1>);
    case 2: return go(modal_var_kernel<FK, 2>);
    default: return FAGP_EUNSUPPORTED;
  }
}

static int launch_mean(const double* Ts, int64_t Ns, const fagp_basis* b, const double* w, double c, double* mean,
                       uint32_t* flags, cudaStream_t s) {
  if (Ns == 0) return FAGP_OK;
  const int G0 = table_gbase(b->p, b->M);
  const size_t msmem = (size_t(b->m) + size_t(MNT) * (G0 | 1)) * sizeof(double);
  if (msmem > 227 * 1024) return FAGP_EUNSUPPORTED;
  auto go = [&](auto kern) -> int {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(msmem)));
    kern<<<unsigned(ceil_div(Ns, MNT)), MNT, msmem, s>>>(Ts, Ns, view(b), w, c, mean, flags);
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

int matvec(const double* T, int64_t N, const fagp_basis* b, const double* x, double c, double* y, uint32_t* flags,
           cudaStream_t s) {
  return launch_mean(T, N, b, x, c, y, flags, s);
}

int predict(const double* Ts, int64_t Ns, const fagp_basis* b, const double* op, double sigma2, double mean_const,
            double* mean, double* var, uint32_t* flags, cudaStream_t s) {
  const Plan pl = make_plan(0, b->p, b->M);
  if (var) {
    const size_t smem = var_smem(table_gsec(b->p, b->M));
    if (smem > 227 * 1024) return FAGP_EUNSUPPORTED;
    const int FK = b->p - pl.pN, FE = pl.pN;
    int rc;
    switch (FK) {
      case 1: rc = launch_var_fe<1>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      case 2: rc = launch_var_fe<2>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      case 3: rc = launch_var_fe<3>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      case 4: rc = launch_var_fe<4>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      case 5: rc = launch_var_fe<5>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      case 6: rc = launch_var_fe<6>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      case 7: rc = launch_var_fe<7>(FE, Ts, Ns, b, pl, op, sigma2, var, flags, smem, s); break;
      default: rc = FAGP_EUNSUPPORTED;
    }
    if (rc) return rc;
    FAGP_LAUNCH_CHECK();
  }
  return launch_mean(Ts, Ns, b, op + pl.KP * pl.NP, mean_const, mean, flags, s);
}

}  // namespace modal
}  // namespace fagp
