// Stage (2) of the path: tensor-product features generated on chip and contracted into
// the Gram matrix on the FP64 tensor pipe (DMMA), plus t = Phi^T (y - c) as an extra
// column.  Replaces posterior.py:168 (`backend.gemm(es.phi, es.phi, transpose_a=True)`,
// which numpy routes to DSYRK) and posterior.py:229,233 (`gemm(phi, r, transpose_a=True)`).
//
// Data layout
//   T      (N, W) table rows from fagp_basis_eval: [phi_{d,i}(x_rd) (p*M) | r | 1 | 0 | pad]
//   ext    Phi_ext = [Phi | r | 0-pad] of width Tt*BT, Tt = ceil((m+1)/BT); never in HBM
//   ws     split-K partial tiles [S][npairs][BT][BT]  (upper-triangle tile pairs only)
//   packed (m+1)(m+2)/2 upper triangle of Phi_ext^T Phi_ext, row-major
//
// Every column of Phi_ext is a product of p table entries of the same row: feature
// column j multiplies phi_{d, i_d(j)} in the reference's broadcast order
// (mercer.py:287-291); the residual column multiplies (r, 1, 1, ...) and padding columns
// (0, 1, 1, ...).  So generation is one branch-free gather-multiply per element.
//
// K1 (gram_kernel_fast<P>): one CTA per (upper tile pair, row chunk), 8 warps on 64x32
// DMMA warp tiles.  The table rows of chunk n+2 arrive by cp.async while the Phi tiles of
// chunk n+1 are generated into shared memory interleaved with the DMMA k-loop of chunk n,
// so generation fills issue slots between DMMAs instead of running as a separate phase.
// K1b (gram_reduce_kernel): sums the split-K partials in chunk order (deterministic, no
// atomics) and flags a non-finite diagonal (G_jj is non-finite iff a feature of column j
// is), which keeps the per-element path check-free.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "modal.cuh"

namespace fagp {
namespace gram {

constexpr int BK = 32;         // rows per pipeline stage (large / generic kernels)
constexpr size_t kMaxSmem = 227 * 1024;

// Tile configuration of the fast kernel: output tile BT x BT, warp grid WGM x WGN, NT = 2 BT
// threads (one generated Phi column per thread), MINB CTAs per SM.
template <int BT_, int WGM_, int WGN_, int MINB_, int BK_>
struct Cfg {
  static constexpr int BT = BT_, WGM = WGM_, WGN = WGN_, MINB = MINB_, BKC = BK_;
  static constexpr int NT = 32 * WGM * WGN;
  static constexpr int SP = BT + 4;  // SP % 16 == 4 -> conflict-free DMMA fragment loads
  static constexpr int WM = BT / WGM, WN = BT / WGN, FM = WM / 8, FN = WN / 8;
  static constexpr int STAGE = BKC * SP;  // doubles per operand per stage
  static_assert(NT == 2 * BT, "one generated column per thread");
  static_assert(SP % 16 == 4, "fragment bank mapping");
};
using CfgSmall = Cfg<64, 2, 2, 4, 16>;    // 64x64 tiles, 4 warps of 32x32, 16-row stages, 4 CTAs/SM
using CfgLarge = Cfg<128, 2, 4, 1, 32>;   // 128x128 tiles, 8 warps of 64x32, 32-row stages, 1 CTA/SM

struct Plan {
  int BT;             // tile edge
  int bk;             // rows per pipeline stage
  int Tt;             // tiles per side of the extended matrix
  int npairs;         // Tt (Tt + 1) / 2
  int S;              // row chunks (split-K)
  int64_t chunk_rows; // rows per chunk (multiple of BK)
};

inline Plan make_plan(int64_t N, int64_t m, int BT, int ctas_per_sm, int bk) {
  Plan pl;
  pl.BT = BT;
  pl.bk = bk;
  pl.Tt = int(ceil_div(m + 1, BT));
  pl.npairs = pl.Tt * (pl.Tt + 1) / 2;
  const int64_t max_chunks = tmax<int64_t>(1, ceil_div(N, bk));
  const int64_t slots = int64_t(num_sms()) * ctas_per_sm;
  int64_t best_S = 1;
  double best_eff = -1.0;
  for (int64_t S = 1; S <= tmin<int64_t>(max_chunks, 4096); ++S) {
    const int64_t ctas = S * pl.npairs;
    const double eff = double(ctas) / double(ceil_div(ctas, slots) * slots);
    const bool enough = ctas >= 2 * slots || S == max_chunks;
    if (enough && eff >= 0.96) {
      best_S = S;
      break;
    }
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best_S = S;
    }
  }
  pl.chunk_rows = round_up(tmax<int64_t>(1, ceil_div(tmax<int64_t>(N, 1), best_S)), bk);
  pl.S = int(tmax<int64_t>(1, ceil_div(N, pl.chunk_rows)));
  return pl;
}

__device__ __forceinline__ void pair_coords(int pair, int Tt, int& ti, int& tj) {
  int t = 0, rem = pair;
  while (rem >= Tt - t) {
    rem -= Tt - t;
    ++t;
  }
  ti = t;
  tj = t + rem;
}

// Table offset of factor d of extended column `col`: feature digit, residual (r, 1, ...)
// or zero padding (0, 1, ...).
__device__ __forceinline__ int col_offset(int64_t col, int64_t m, int M, int pM, int d, int p) {
  if (col < m) {
    int64_t q = col;
    for (int e = p - 1; e > d; --e) q /= M;
    return d * M + int(q % M);
  }
  if (d == 0) return col == m ? table_col_r(pM) : table_col_zero(pM);
  return table_col_one(pM);
}

template <class C>
inline size_t fast_smem_bytes(int W) {
  return size_t(4) * C::STAGE * sizeof(double) + size_t(2) * C::BKC * W * sizeof(double);
}

template <int P, class C>
__global__ void __launch_bounds__(C::NT, C::MINB)
gram_kernel_fast(const double* __restrict__ T, int64_t N, BasisView b, Plan pl, double* __restrict__ ws) {
  constexpr int BT = C::BT, NT = C::NT, SP = C::SP, STAGE = C::STAGE;
  constexpr int WM = C::WM, WN = C::WN, FM = C::FM, FN = C::FN, BK = C::BKC;
  extern __shared__ double sm[];
  const int M = b.M, pM = P * M, W = table_width(P, M);
  double* tbuf = sm + 4 * STAGE;  // [2][BK][W] staged table rows
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pair = blockIdx.x % pl.npairs;
  const int chunk = blockIdx.x / pl.npairs;
  int ti, tj;
  pair_coords(pair, pl.Tt, ti, tj);
  const bool diag = ti == tj;
  const int64_t r0 = int64_t(chunk) * pl.chunk_rows;
  const int64_t r1 = tmin<int64_t>(N, r0 + pl.chunk_rows);
  const int64_t m = b.m;

  // generator role: thread owns one column of one operand tile (gh = 0: tile ti -> buffer
  // 0, gh = 1: tile tj -> buffer 1; a diagonal pair simply generates its tile twice) and
  // generates rows 4kk..4kk+3 of the next chunk during DMMA k-step kk
  const int gc = tid % BT, gh = tid / BT;
  const int64_t gcol = int64_t(gh ? tj : ti) * BT + gc;
  int off[P];
#pragma unroll
  for (int d = 0; d < P; ++d) off[d] = col_offset(gcol, m, M, pM, d, P);

  auto load_tab = [&](int slot, int64_t base) {
    double* dst = tbuf + slot * (BK * W);
    const int nrows = int(tmax<int64_t>(0, tmin<int64_t>(BK, r1 - base)));
    const int nd = nrows * W;  // W is even: 16-byte copies, 16-byte aligned rows
    const double* src = T + base * W;
    for (int i = tid; i < nd / 2; i += NT) cp_async_16(dst + 2 * i, src + 2 * i);
    for (int i = nd + tid; i < BK * W; i += NT) dst[i] = 0.0;  // rows past the chunk end
    cp_async_commit();
  };
  auto gen_rows = [&](int stage, int kk) {
    double* dst = sm + (stage * 2 + gh) * STAGE + gc;
    const double* tb = tbuf + stage * (BK * W);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = kk * 4 + i;
      const double* Tr = tb + k * W;
      double v = Tr[off[0]];
#pragma unroll
      for (int d = 1; d < P; ++d) v = __dmul_rn(v, Tr[off[d]]);
      dst[k * SP] = v;
    }
  };

  const int wi = warp / C::WGN, wj = warp % C::WGN;
  const bool active = !diag || (wj * WN + WN - 1 >= wi * WM);  // blocks strictly below the diagonal idle
  double acc[FM][FN][2];
#pragma unroll
  for (int s = 0; s < FM; ++s)
#pragma unroll
    for (int t = 0; t < FN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;

  const int nchunks = int(ceil_div(tmax<int64_t>(r1 - r0, 0), BK));
  load_tab(0, r0);
  cp_async_wait<0>();
  __syncthreads();
  load_tab(1, r0 + BK);
#pragma unroll
  for (int kk = 0; kk < BK / 4; ++kk) gen_rows(0, kk);
  cp_async_wait<0>();
  __syncthreads();
  for (int n = 0; n < nchunks; ++n) {
    const int cur = n & 1, nxt = cur ^ 1;
    // table slot cur (chunk n) was consumed by the generation of chunk n one iteration ago
    if (n + 2 < nchunks) load_tab(cur, r0 + int64_t(n + 2) * BK);
    const double* As = sm + (cur * 2) * STAGE + (lane & 3) * SP + wi * WM + (lane >> 2);
    const double* Bs = sm + (cur * 2 + 1) * STAGE + (lane & 3) * SP + wj * WN + (lane >> 2);
    if (active) {
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        double a[FM], bb[FN];
#pragma unroll
        for (int s = 0; s < FM; ++s) a[s] = As[kk * 4 * SP + s * 8];
#pragma unroll
        for (int t = 0; t < FN; ++t) bb[t] = Bs[kk * 4 * SP + t * 8];
#pragma unroll
        for (int s = 0; s < FM; ++s)
#pragma unroll
          for (int t = 0; t < FN; ++t) dmma_8x8x4(acc[s][t][0], acc[s][t][1], a[s], bb[t]);
        gen_rows(nxt, kk);  // chunk n+1 (garbage past the last chunk, never read)
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) gen_rows(nxt, kk);
    }
    cp_async_wait<0>();
    __syncthreads();
  }

  if (active) {
    double* tile = ws + (size_t(chunk) * pl.npairs + pair) * size_t(BT * BT);
#pragma unroll
    for (int s = 0; s < FM; ++s) {
      const int i = wi * WM + s * 8 + (lane >> 2);
#pragma unroll
      for (int t = 0; t < FN; ++t) {
        const int j = wj * WN + t * 8 + 2 * (lane & 3);
        *reinterpret_cast<double2*>(tile + i * BT + j) = make_double2(acc[s][t][0], acc[s][t][1]);
      }
    }
  }
}

// Generic K1 for shapes outside the fast path (p > 8 or table rows too wide to stage):
// runtime p, table entries read through L1, one barrier-separated phase per chunk.
__global__ void __launch_bounds__(CfgLarge::NT, 1)
gram_kernel_generic(const double* __restrict__ T, int64_t N, BasisView b, Plan pl, double* __restrict__ ws) {
  using C = CfgLarge;
  constexpr int BT = C::BT, NT = C::NT, SP = C::SP, STAGE = C::STAGE;
  constexpr int WM = C::WM, WN = C::WN, FM = C::FM, FN = C::FN;
  extern __shared__ double sm[];
  int* col_off = reinterpret_cast<int*>(sm + 4 * STAGE);  // [p][NT], private per thread
  const int M = b.M, p = b.p, pM = p * M, W = table_width(p, M);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pair = blockIdx.x % pl.npairs;
  const int chunk = blockIdx.x / pl.npairs;
  int ti, tj;
  pair_coords(pair, pl.Tt, ti, tj);
  const bool diag = ti == tj;
  const int64_t r0 = int64_t(chunk) * pl.chunk_rows;
  const int64_t r1 = tmin<int64_t>(N, r0 + pl.chunk_rows);
  const int gc = tid % BT, gh = tid / BT;
  const int64_t gcol = int64_t(gh ? tj : ti) * BT + gc;
  for (int d = 0; d < p; ++d) col_off[d * NT + tid] = col_offset(gcol, b.m, M, pM, d, p);

  auto generate = [&](int64_t base) {
    double* dst = sm + gh * STAGE + gc;
    for (int k = 0; k < BK; ++k) {
      const int64_t row = base + k;
      double v = 0.0;
      if (row < r1) {
        const double* Tr = T + row * W;
        v = __ldg(Tr + col_off[tid]);
        for (int d = 1; d < p; ++d) v = __dmul_rn(v, __ldg(Tr + col_off[d * NT + tid]));
      }
      dst[k * SP] = v;
    }
  };
  const int wi = warp / 4, wj = warp % 4;
  const bool active = !diag || (wj * WN + WN - 1 >= wi * WM);
  double acc[FM][FN][2];
#pragma unroll
  for (int s = 0; s < FM; ++s)
#pragma unroll
    for (int t = 0; t < FN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;
  const int nchunks = int(ceil_div(tmax<int64_t>(r1 - r0, 0), BK));
  for (int n = 0; n < nchunks; ++n) {
    generate(r0 + int64_t(n) * BK);
    __syncthreads();
    if (active) {
      const double* As = sm + (lane & 3) * SP + wi * WM + (lane >> 2);
      const double* Bs = sm + STAGE + (lane & 3) * SP + wj * WN + (lane >> 2);
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        double a[FM], bb[FN];
#pragma unroll
        for (int s = 0; s < FM; ++s) a[s] = As[kk * 4 * SP + s * 8];
#pragma unroll
        for (int t = 0; t < FN; ++t) bb[t] = Bs[kk * 4 * SP + t * 8];
#pragma unroll
        for (int s = 0; s < FM; ++s)
#pragma unroll
          for (int t = 0; t < FN; ++t) dmma_8x8x4(acc[s][t][0], acc[s][t][1], a[s], bb[t]);
      }
    }
    __syncthreads();
  }
  if (active) {
    double* tile = ws + (size_t(chunk) * pl.npairs + pair) * size_t(BT * BT);
#pragma unroll
    for (int s = 0; s < FM; ++s) {
      const int i = wi * WM + s * 8 + (lane >> 2);
#pragma unroll
      for (int t = 0; t < FN; ++t) {
        const int j = wj * WN + t * 8 + 2 * (lane & 3);
        *reinterpret_cast<double2*>(tile + i * BT + j) = make_double2(acc[s][t][0], acc[s][t][1]);
      }
    }
  }
}

// K1b: packed[i, j] = sum_s ws[s][pair(i, j)][i % BT][j % BT] in chunk order.
__global__ void gram_reduce_kernel(const double* __restrict__ ws, int64_t m, Plan pl, double* __restrict__ packed,
                                   uint32_t* flags) {
  const int64_t me = m + 1;
  const int BT = pl.BT;
  for (int64_t i = blockIdx.y; i < me; i += gridDim.y) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < i || j >= me) continue;
    const int ti = int(i / BT), tj = int(j / BT);
    const int pair = ti * pl.Tt - ti * (ti - 1) / 2 + (tj - ti);
    const size_t off = size_t(i % BT) * BT + size_t(j % BT);
    const size_t stride = size_t(pl.npairs) * BT * BT;
    const double* src = ws + size_t(pair) * BT * BT + off;
    // loads issued 8 at a time (an L2 round trip each otherwise); the sum keeps chunk order
    double sum = 0.0;
    int s = 0;
    for (; s + 8 <= pl.S; s += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = src[(s + u) * stride];
#pragma unroll
      for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; s < pl.S; ++s) sum += src[s * stride];
    packed[i * (2 * me - i - 1) / 2 + j] = sum;
    if (i == j && i < m && not_finite(sum)) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
  }
}

}  // namespace gram
}  // namespace fagp

using namespace fagp;

namespace fagp {
namespace gram {
// Which kernel runs for a basis; the workspace size depends on it.
struct Choice {
  bool fast;
  bool small;  // CfgSmall (else CfgLarge)
  Plan plan;
};
inline Choice choose(int64_t N, const fagp_basis* b) {
  const int W = table_width(b->p, b->M);
  Choice c{};
  c.fast = b->p <= 8 && fast_smem_bytes<CfgLarge>(W) <= kMaxSmem;
  const char* cfg = getenv("FAGP_GRAM_CFG");  // tuning override: "large" | "small"
  c.small = c.fast && fast_smem_bytes<CfgSmall>(W) * CfgSmall::MINB <= 228 * 1024 - CfgSmall::MINB * 1024 &&
            !(cfg && strcmp(cfg, "large") == 0);
  c.plan = c.small ? make_plan(N, b->m, CfgSmall::BT, CfgSmall::MINB, CfgSmall::BKC)
                    : make_plan(N, b->m, CfgLarge::BT, 1, CfgLarge::BKC);
  return c;
}
template <int P, class C>
int launch_fast(const double* T, int64_t N, const fagp_basis* basis, const Plan& pl, double* ws, cudaStream_t s) {
  const size_t smem = fast_smem_bytes<C>(table_width(basis->p, basis->M));
  FAGP_CUDA_TRY(cudaFuncSetAttribute(gram_kernel_fast<P, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  gram_kernel_fast<P, C><<<unsigned(size_t(pl.S) * pl.npairs), C::NT, smem, s>>>(T, N, view(basis), pl, ws);
  return FAGP_OK;
}
template <class C>
int dispatch_fast(const double* T, int64_t N, const fagp_basis* basis, const Plan& pl, double* ws, cudaStream_t s) {
  switch (basis->p) {
    case 1: return launch_fast<1, C>(T, N, basis, pl, ws, s);
    case 2: return launch_fast<2, C>(T, N, basis, pl, ws, s);
    case 3: return launch_fast<3, C>(T, N, basis, pl, ws, s);
    case 4: return launch_fast<4, C>(T, N, basis, pl, ws, s);
    case 5: return launch_fast<5, C>(T, N, basis, pl, ws, s);
    case 6: return launch_fast<6, C>(T, N, basis, pl, ws, s);
    case 7: return launch_fast<7, C>(T, N, basis, pl, ws, s);
    default: return launch_fast<8, C>(T, N, basis, pl, ws, s);
  }
}
}  // namespace gram
}  // namespace fagp

extern "C" {

int64_t fagp_gram_len(const fagp_basis* basis) {
  if (check_basis(basis) != FAGP_OK) return -1;
  if (modal::enabled(basis->p, basis->M)) return modal::gram_len(basis);
  return (basis->m + 1) * (basis->m + 2) / 2;
}

size_t fagp_gram_workspace_size(int64_t N, const fagp_basis* basis) {
  if (check_basis(basis) != FAGP_OK || N < 0) return 0;
  if (modal::enabled(basis->p, basis->M)) return modal::gram_workspace(N, basis);
  const gram::Plan pl = gram::choose(N, basis).plan;
  return size_t(pl.S) * pl.npairs * pl.BT * pl.BT * sizeof(double);
}

int fagp_gram(const double* T, int64_t N, const fagp_basis* basis, double* gram_ext_packed, void* workspace,
              size_t workspace_bytes, uint32_t* flags, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || gram_ext_packed == nullptr || (N > 0 && T == nullptr)) return FAGP_EINVAL;
  if (modal::enabled(basis->p, basis->M))
    return modal::gram(T, N, basis, gram_ext_packed, workspace, workspace_bytes, flags, static_cast<cudaStream_t>(stream));
  const gram::Choice ch = gram::choose(N, basis);
  const gram::Plan pl = ch.plan;
  const size_t need = size_t(pl.S) * pl.npairs * pl.BT * pl.BT * sizeof(double);
  if (workspace == nullptr || workspace_bytes < need) return FAGP_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* ws = static_cast<double*>(workspace);
  int rc = FAGP_OK;
  if (ch.fast) {
    rc = ch.small ? gram::dispatch_fast<gram::CfgSmall>(T, N, basis, pl, ws, s)
                  : gram::dispatch_fast<gram::CfgLarge>(T, N, basis, pl, ws, s);
  } else {
    const size_t gsmem = size_t(4) * gram::CfgLarge::STAGE * sizeof(double) + size_t(basis->p) * gram::CfgLarge::NT * sizeof(int);
    FAGP_CUDA_TRY(cudaFuncSetAttribute(gram::gram_kernel_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gsmem)));
    gram::gram_kernel_generic<<<unsigned(size_t(pl.S) * pl.npairs), gram::CfgLarge::NT, gsmem, s>>>(T, N, view(basis), pl, ws);
  }
  if (rc) return rc;
  FAGP_LAUNCH_CHECK();
  const int64_t me = basis->m + 1;
  dim3 grid(unsigned(ceil_div(me, 256)), unsigned(tmin<int64_t>(me, 65535)));
  gram::gram_reduce_kernel<<<grid, 256, 0, s>>>(ws, basis->m, pl, gram_ext_packed, flags);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

size_t fagp_phi_tmatvec_workspace_size(int64_t N, const fagp_basis* basis) {
  if (check_basis(basis) != FAGP_OK || N < 0) return 0;
  if (modal::enabled(basis->p, basis->M)) return modal::tmatvec_workspace(N, basis);
  // direct form: the packed [G | t] Gram and its workspace (p = 1: the SYRK is the cheap part)
  return fagp_gram_workspace_size(N, basis) + size_t(round_up(fagp_gram_len(basis), 2)) * sizeof(double);
}

int fagp_phi_tmatvec(double* T, int64_t N, const fagp_basis* basis, const double* v, double* out, void* workspace,
                     size_t workspace_bytes, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || out == nullptr || (N > 0 && (T == nullptr || v == nullptr))) return FAGP_EINVAL;
  if (workspace == nullptr || workspace_bytes < fagp_phi_tmatvec_workspace_size(N, basis)) return FAGP_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (N == 0) {
    FAGP_CUDA_TRY(cudaMemsetAsync(out, 0, size_t(basis->m) * sizeof(double), s));
    return FAGP_OK;
  }
  st = fagp_set_residual(T, N, basis, v, 0.0, stream);
  if (st) return st;
  if (modal::enabled(basis->p, basis->M)) return modal::tmatvec(T, N, basis, out, workspace, workspace_bytes, s);
  const size_t gws = fagp_gram_workspace_size(N, basis);
  double* packed = reinterpret_cast<double*>(static_cast<char*>(workspace) + gws);
  st = fagp_gram(T, N, basis, packed, workspace, gws, nullptr, stream);
  if (st) return st;
  return fagp_gram_unpack(packed, basis, nullptr, out, nullptr, 0, stream);
}

}  // extern "C"
