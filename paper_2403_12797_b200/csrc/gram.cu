// Stage (2) of the path: tensor-product features generated on chip and contracted into
// the Gram matrix on the FP64 tensor pipe (DMMA), plus t = Phi^T (y - c) as an extra
// column.  Replaces posterior.py:168 (`backend.gemm(es.phi, es.phi, transpose_a=True)`,
// which numpy routes to DSYRK) and posterior.py:229,233 (`gemm(phi, r, transpose_a=True)`).
//
// Data layout
//   T      (N, p*M)   per-row 1-D eigenfunction table from fagp_basis_eval (HBM, read via L1)
//   ext    Phi_ext = [Phi | r | 0-pad] of width Tt*BT, Tt = ceil((m+1)/BT); never in HBM
//   ws     split-K partial tiles [S][npairs][BT][BT]  (upper-triangle tile pairs only)
//   packed (m+1)(m+2)/2 upper triangle of Phi_ext^T Phi_ext, row-major
//
// K1 (gram_kernel): one CTA per (tile pair, row chunk).  Each pipeline stage generates
// BK rows of the two Phi column tiles into shared memory -- Phi[r, j] is the product of p
// table entries in the reference's broadcast order (mercer.py:287-291) -- and 8 warps
// contract them with mma.m8n8k4.f64 (64x32 warp tiles, accumulators in registers).
// Deterministic: each CTA sums its rows in a fixed order and K1b adds the chunk
// partials in chunk order; no floating-point atomics.
#include "common.cuh"

namespace fagp {
namespace gram {

constexpr int BT = 128;        // output tile edge
constexpr int BK = 32;         // rows per pipeline stage
constexpr int NT = 256;        // threads per CTA (8 warps)
constexpr int SP = BT + 4;     // smem row stride in doubles; SP % 16 == 4 -> conflict-free fragments
constexpr int WM = 64, WN = 32;
constexpr int FM = WM / 8, FN = WN / 8;
constexpr int STAGE = BK * SP;  // doubles per operand per stage

struct Plan {
  int Tt;             // tiles per side of the extended matrix
  int npairs;         // Tt (Tt + 1) / 2
  int S;              // row chunks (split-K)
  int64_t chunk_rows; // rows per chunk (multiple of BK)
};

inline Plan make_plan(int64_t N, int64_t m) {
  Plan pl;
  pl.Tt = int(ceil_div(m + 1, BT));
  pl.npairs = pl.Tt * (pl.Tt + 1) / 2;
  const int64_t max_chunks = tmax<int64_t>(1, ceil_div(N, BK));
  const int sms = num_sms();
  int64_t best_S = 1;
  double best_eff = -1.0;
  for (int64_t S = 1; S <= tmin<int64_t>(max_chunks, 4096); ++S) {
    const int64_t ctas = S * pl.npairs;
    const double eff = double(ctas) / double(ceil_div(ctas, sms) * sms);
    const bool enough = ctas >= 2 * sms || S == max_chunks;
    if (enough && eff >= 0.96) {
      best_S = S;
      best_eff = 2.0;
      break;
    }
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best_S = S;
    }
  }
  pl.chunk_rows = round_up(tmax<int64_t>(1, ceil_div(tmax<int64_t>(N, 1), best_S)), BK);
  pl.S = int(tmax<int64_t>(1, ceil_div(N, pl.chunk_rows)));
  return pl;
}

inline size_t smem_bytes(int p) { return size_t(4) * STAGE * sizeof(double) + size_t(p) * NT * sizeof(int); }

__device__ __forceinline__ void pair_coords(int pair, int Tt, int& ti, int& tj) {
  int t = 0, rem = pair;
  while (rem >= Tt - t) {
    rem -= Tt - t;
    ++t;
  }
  ti = t;
  tj = t + rem;
}

__global__ void __launch_bounds__(NT, 1)
gram_kernel(const double* __restrict__ T, const double* __restrict__ y, double mean_const, int64_t N,
            BasisView b, Plan pl, double* __restrict__ ws, uint32_t* flags) {
  extern __shared__ double sm[];
  int* col_off = reinterpret_cast<int*>(sm + 4 * STAGE);  // [p][NT], private per thread
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pair = blockIdx.x % pl.npairs;
  const int chunk = blockIdx.x / pl.npairs;
  int ti, tj;
  pair_coords(pair, pl.Tt, ti, tj);
  const bool diag = ti == tj;
  const int64_t r0 = int64_t(chunk) * pl.chunk_rows;
  const int64_t r1 = tmin<int64_t>(N, r0 + pl.chunk_rows);
  const int64_t m = b.m;
  const int M = b.M, p = b.p, pM = p * M;

  // ---- generator role: one Phi column per thread (two tiles for off-diagonal pairs) ----
  const int gc = tid % BT, gh = tid / BT;
  const int gtile = diag ? ti : (gh ? tj : ti);
  const int64_t gcol = int64_t(gtile) * BT + gc;
  const int gop = diag ? 0 : gh;
  const int krow0 = diag ? gh : 0, kstep = diag ? 2 : 1;
  const int kind = gcol < m ? 0 : (gcol == m ? 1 : 2);  // feature | residual | zero pad
  if (kind == 0) {
    int64_t q = gcol;
    for (int d = p - 1; d >= 0; --d) {
      col_off[d * NT + tid] = d * M + int(q % M);
      q /= M;
    }
  }
  bool bad = false;

  auto generate = [&](int stage, int64_t base) {
    double* dst = sm + (stage * 2 + gop) * STAGE + gc;
#pragma unroll 4
    for (int k = krow0; k < BK; k += kstep) {
      const int64_t row = base + k;
      double v = 0.0;
      if (row < r1) {
        if (kind == 0) {
          const double* Tr = T + row * pM;
          v = __ldg(Tr + col_off[tid]);
          for (int d = 1; d < p; ++d) v = __dmul_rn(v, __ldg(Tr + col_off[d * NT + tid]));
          bad |= not_finite(v);
        } else if (kind == 1) {
          v = __dsub_rn(__ldg(y + row), mean_const);
        }
      }
      dst[k * SP] = v;
    }
  };

  // ---- consumer role: 2 x 4 warp grid of 64 x 32 tiles ----
  const int wi = warp / 4, wj = warp % 4;
  const bool active = !diag || (wj * WN + WN - 1 >= wi * WM);  // skip blocks strictly below diag
  double acc[FM][FN][2];
#pragma unroll
  for (int s = 0; s < FM; ++s)
#pragma unroll
    for (int t = 0; t < FN; ++t) acc[s][t][0] = acc[s][t][1] = 0.0;

  const int nchunks = int(ceil_div(tmax<int64_t>(r1 - r0, 0), BK));
  if (nchunks > 0) generate(0, r0);
  __syncthreads();
  for (int n = 0; n < nchunks; ++n) {
    if (n + 1 < nchunks) generate((n + 1) & 1, r0 + int64_t(n + 1) * BK);
    if (active) {
      const double* As = sm + ((n & 1) * 2) * STAGE + (lane & 3) * SP + wi * WM + (lane >> 2);
      const double* Bs = sm + ((n & 1) * 2 + (diag ? 0 : 1)) * STAGE + (lane & 3) * SP + wj * WN + (lane >> 2);
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
  if (bad) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
}

// K1b: packed[i, j] = sum_s ws[s][pair(i, j)][i % BT][j % BT] in chunk order.
__global__ void gram_reduce_kernel(const double* __restrict__ ws, int64_t m, Plan pl,
                                   double* __restrict__ packed) {
  const int64_t me = m + 1;
  const int64_t i = blockIdx.y;
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < i || j >= me) return;
  const int ti = int(i / BT), tj = int(j / BT);
  const int pair = ti * pl.Tt - ti * (ti - 1) / 2 + (tj - ti);
  const size_t off = size_t(i % BT) * BT + size_t(j % BT);
  const size_t stride = size_t(pl.npairs) * BT * BT;
  const double* src = ws + size_t(pair) * BT * BT + off;
  double sum = 0.0;
  for (int s = 0; s < pl.S; ++s) sum += src[s * stride];
  packed[i * (2 * me - i - 1) / 2 + j] = sum;
}

}  // namespace gram
}  // namespace fagp

using namespace fagp;

extern "C" {

int64_t fagp_gram_packed_len(int64_t m) {
  if (m < 1) return -1;
  return (m + 1) * (m + 2) / 2;
}

size_t fagp_gram_workspace_size(int64_t N, const fagp_basis* basis) {
  if (check_basis(basis) != FAGP_OK || N < 0) return 0;
  gram::Plan pl = gram::make_plan(N, basis->m);
  return size_t(pl.S) * pl.npairs * gram::BT * gram::BT * sizeof(double);
}

int fagp_gram(const double* T, const double* y, double mean_const, int64_t N, const fagp_basis* basis,
              double* gram_ext_packed, void* workspace, size_t workspace_bytes, uint32_t* flags,
              void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || gram_ext_packed == nullptr || (N > 0 && (T == nullptr || y == nullptr))) return FAGP_EINVAL;
  gram::Plan pl = gram::make_plan(N, basis->m);
  const size_t need = size_t(pl.S) * pl.npairs * gram::BT * gram::BT * sizeof(double);
  if (workspace == nullptr || workspace_bytes < need) return FAGP_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t smem = gram::smem_bytes(basis->p);
  FAGP_CUDA_TRY(cudaFuncSetAttribute(gram::gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  double* ws = static_cast<double*>(workspace);
  gram::gram_kernel<<<unsigned(size_t(pl.S) * pl.npairs), gram::NT, smem, s>>>(T, y, mean_const, N, view(basis), pl,
                                                                               ws, flags);
  FAGP_LAUNCH_CHECK();
  const int64_t me = basis->m + 1;
  dim3 grid(unsigned(ceil_div(me, 256)), unsigned(me));
  gram::gram_reduce_kernel<<<grid, 256, 0, s>>>(ws, basis->m, pl, gram_ext_packed);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // extern "C"
