// Fused modal Gram and fused modal predict: the two FP64 tensor-core kernels of the C3 step,
// evaluated straight from the input points (no basis table in HBM).
//
// The algebra is modal.cu's (Hermite linearisation, exact): with g_{d,k} the L = 2M-1 modal
// functions of dimension d,
//   K[kappa] = sum_r prod_d g_{d,kappa_d}(x_rd)                        (L^p entries; -> G = Phi^T Phi)
//   t[a]     = sum_r (y_r - c) prod_d phi_{d,a_d}(x_rd)                 (posterior.py:229-233)
//   var_i    = sigma2 sum_kappa C''[kappa] prod_d g_{d,kappa_d}(x*_i)   (posterior.py:249-263, diagonal)
//   mean_i   = c + sum_a w[a] prod_d phi_{d,a_d}(x*_i)                  (posterior.py:247)
// What changes here is the B200 mapping:
//
//  * Producer/consumer CTAs.  Two producer warps evaluate the 1-D eigenfunctions of the next
//    64-row block (mercer.py:122-143, 276-281, bit-faithful op order, eigfun.cuh) into a
//    double-buffered shared-memory row slab while the consumer warps run the DMMA contraction
//    on the current block; one __syncthreads per block flips the buffers.  Nothing but X (and
//    y) is read from HBM: 24 B per row at p = 3 instead of the 752 B table row.
//  * Register-generated DMMA fragments.  Every mma.m8n8k4.f64 operand that is a product of
//    basis values (g g, phi phi, r phi) is formed in the thread that feeds it to the tensor
//    core (FA/FB/FK LDS.64 + DMULs, conflict-free thanks to a row stride == 4 mod 16 doubles),
//    so generated operands never round-trip through shared memory.
//  * Gram: each CTA owns a contiguous row range and accumulates the WHOLE output ([K | t]:
//    46 x 3 + 13 x 2 8x8 fragments at C3) in registers of 14 consumer warps; one CTA per SM,
//    persistent; per-CTA partials are summed in a fixed order by a second small kernel
//    (deterministic, no float atomics) -- the same buffer the multi-GPU path all-reduces.
//  * Predict: the variance operand C'' and the mean weights are staged once per CTA into
//    shared memory in fragment-major order (one conflict-free LDS.64 per B fragment); 8
//    consumer warps = 4 row groups x 2 K-halves (split-K reduced through shared memory);
//    the g / phi epilogue products and the 4-lane row reductions stay in registers; mean and
//    variance come out of the same pass.
// Shapes whose output does not fit these layouts use the tiled table kernels (modal.cu,
// gram.cu, predict.cu) -- see fagp_gram_x / fagp_predict_x.
#include <cstring>

#include "common.cuh"
#include "eigfun.cuh"
#include "modal.cuh"

namespace fagp {
namespace fused {

// ---------------------------------------------------------------------------------------
// Shared-memory row slab: [g_{d,k} (p L) | phi_{d,a} (p M) | r | 1.0 | 0.0 | pad], stride BW
// with BW % 16 == 4 so 4 rows x 4 consecutive doubles hit 16 distinct bank pairs.
struct RowLayout {
  int goff, poff, roff, one, zero, bw;
};
__host__ __device__ inline RowLayout row_layout(int p, int M) {
  const int L = modal_L(M);
  RowLayout r;
  r.goff = 0;
  r.poff = p * L;
  r.roff = p * L + p * M;
  r.one = r.roff + 1;
  r.zero = r.roff + 2;
  int w = r.zero + 1;
  while (w % 16 != 4) ++w;
  r.bw = w;
  return r;
}

constexpr int kRows = 64;      // rows per block (16 DMMA k-steps of 4 rows)
constexpr int kProdWarps = 2;  // producer warps per CTA
constexpr int kMaxTasks = 4;   // (row, dim) tasks per producer thread: kRows * p / 64 <= 4
constexpr int kMaxF = 4;       // factors per generated column (p <= 4 on the fused path)

// Producer: rows [0, kRows) of `slab` <- basis of points row0 + i (i < nvalid; the rest zero).
__device__ __forceinline__ void produce_rows(const double* __restrict__ X, const double* __restrict__ y, double c,
                                             int64_t row0, int nvalid, const BasisView& b, const RowLayout& rl,
                                             const double* c1, const double* c2, double* slab, int ptid,
                                             bool want_phi, bool want_g, bool& bad_x) {
  const int p = b.p, M = b.M, L = modal_L(M);
  constexpr int NTH = kProdWarps * 32;
  const int tasks = kRows * p;
  double xs[kMaxTasks];
#pragma unroll
  for (int i = 0; i < kMaxTasks; ++i) {  // all loads first: one HBM round trip per block
    const int t = ptid + i * NTH;
    xs[i] = 0.0;
    if (t < tasks) {
      const int r = t / p;
      if (r < nvalid) xs[i] = X[row0 * p + t];
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxTasks; ++i) {
    const int t = ptid + i * NTH;
    if (t < tasks) {
      const int r = t / p, d = t - r * p;
      double* row = slab + r * rl.bw;
      if (r < nvalid) {
        bad_x |= not_finite(xs[i]);
        if (want_phi) eval_phi_dim(xs[i], b, d, c1, c2, row + rl.poff + d * M);
        if (want_g) eval_g_dim(xs[i], b, d, c1, c2, row + rl.goff + d * L);
      } else {
        if (want_phi)
          for (int k = 0; k < M; ++k) row[rl.poff + d * M + k] = 0.0;
        if (want_g)
          for (int k = 0; k < L; ++k) row[rl.goff + d * L + k] = 0.0;
      }
    }
  }
  for (int r = ptid; r < kRows; r += NTH) {
    double* row = slab + r * rl.bw;
    row[rl.roff] = (y != nullptr && r < nvalid) ? __dsub_rn(y[row0 + r], c) : 0.0;  // r = y - c (posterior.py:229)
    row[rl.one] = 1.0;
    row[rl.zero] = 0.0;
  }
}

// Offsets of the F factors of generated column `col` (< ncols valid): nd digits in `radix`
// (first dimension slowest) over dims [d0, d0 + nd) of the section at `base`; slot nd takes
// `extra` (e.g. the residual) when extra >= 0; remaining slots -> 1.0; invalid columns -> 0.
template <int F>
__device__ __forceinline__ void col_offsets(int col, int ncols, int base, int d0, int nd, int radix, int extra,
                                            const RowLayout& rl, int (&off)[F]) {
  unsigned q = col < ncols ? unsigned(col) : 0u;
#pragma unroll
  for (int e = F - 1; e >= 0; --e) {
    if (e < nd) {
      off[e] = base + (d0 + e) * radix + int(q % unsigned(radix));
      q /= unsigned(radix);
    } else {
      off[e] = (e == nd && extra >= 0) ? extra : rl.one;
    }
  }
  if (col >= ncols) {
    off[0] = rl.zero;
#pragma unroll
    for (int f = 1; f < F; ++f) off[f] = rl.one;
  }
}

template <int F>
__device__ __forceinline__ double gather_prod(const double* row, const int (&off)[F]) {
  double v = row[off[0]];
#pragma unroll
  for (int f = 1; f < F; ++f) v = __dmul_rn(v, row[off[f]]);
  return v;
}

// ---------------------------------------------------------------------------------------
// Fused Gram
// 16 warps = 4 per SM sub-partition: the most that still leaves each thread 128 registers
// (every sub-partition owns a quarter of the register file)
constexpr int kGramCW = 14;                                // consumer warps
constexpr int kGramNT = (kGramCW + kProdWarps) * 32;       // 512 threads
constexpr int kGramJobs = 5;                               // job slots per consumer warp
constexpr int kNF = 3;                                     // n-fragments per job (<= 24 columns)

struct GPlan {
  int p, M, L, LC;
  int pA, pT;          // K: A = dims [0,pA) x B = dims [pA,p) (g, radix L); t: A = [0,pT) x B = [pT,p) * r (phi)
  int KA, KB, TA, TB;  // section extents
  int kmf, knf, tmf, tnf;
  int G;               // row groups per CTA (each covers every job on k-steps kk = g mod G)
  int64_t Klen, len;   // partial / output layout [K (KA*KB) | t (TA*TB = m)]
  int64_t rows_per_cta;
  int grid, nparts;
  signed char job[kGramCW][kGramJobs];  // per warp-in-group: -1, K m-frag id, or kmf + t m-frag id
};

template <int FA, int FB>
__global__ void __launch_bounds__(kGramNT, 1)
fused_gram_kernel(const double* __restrict__ X, const double* __restrict__ y, double c, int64_t N, BasisView b,
                  const GPlan pl, double* __restrict__ ws, uint32_t* flags) {
  extern __shared__ double sm[];
  const RowLayout rl = row_layout(pl.p, pl.M);
  double* c1 = sm;
  double* c2 = sm + pl.LC;
  double* slabs = sm + 2 * pl.LC;  // [2][kRows * bw]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int k = tid; k < pl.LC; k += kGramNT) {
    c1[k] = herm_c1(k);
    c2[k] = herm_c2(k);
  }
  const int64_t r0 = int64_t(blockIdx.x) * pl.rows_per_cta;
  const int64_t r1 = tmin<int64_t>(N, r0 + pl.rows_per_cta);
  const int nblk = r1 > r0 ? int(ceil_div(r1 - r0, kRows)) : 0;
  const bool producer = warp >= kGramCW;
  const int ptid = tid - kGramCW * 32;
  bool bad_x = false;
  __syncthreads();
  if (producer && nblk > 0)
    produce_rows(X, y, c, r0, int(tmin<int64_t>(kRows, r1 - r0)), b, rl, c1, c2, slabs, ptid, true, true, bad_x);

  // consumer job setup (all warp-uniform except the lane's column)
  const int WG = kGramCW / pl.G;
  const int grp = warp / WG, wi = warp - grp * WG;
  int jid[kGramJobs];
  bool jK[kGramJobs];
  int offA[kGramJobs][FA];
  bool hasK = false, hasT = false;
#pragma unroll
  for (int j = 0; j < kGramJobs; ++j) {
    jid[j] = producer ? -1 : int(pl.job[wi][j]);
    jK[j] = jid[j] >= 0 && jid[j] < pl.kmf;
    hasK |= jK[j];
    hasT |= jid[j] >= pl.kmf;
    if (jK[j])
      col_offsets<FA>(jid[j] * 8 + (lane >> 2), pl.KA, rl.goff, 0, pl.pA, pl.L, -1, rl, offA[j]);
    else
      col_offsets<FA>((jid[j] - pl.kmf) * 8 + (lane >> 2), pl.TA, rl.poff, 0, pl.pT, pl.M, -1, rl, offA[j]);
  }
  int offBK[kNF][FB], offBT[kNF][FB];
#pragma unroll
  for (int nf = 0; nf < kNF; ++nf) {
    col_offsets<FB>(nf * 8 + (lane >> 2), pl.KB, rl.goff, pl.pA, pl.p - pl.pA, pl.L, -1, rl, offBK[nf]);
    col_offsets<FB>(nf * 8 + (lane >> 2), pl.TB, rl.poff, pl.pT, pl.p - pl.pT, pl.M, rl.roff, rl, offBT[nf]);
  }
  double acc[kGramJobs][kNF][2];
#pragma unroll
  for (int j = 0; j < kGramJobs; ++j)
#pragma unroll
    for (int nf = 0; nf < kNF; ++nf) acc[j][nf][0] = acc[j][nf][1] = 0.0;
  __syncthreads();

  for (int n = 0; n < nblk; ++n) {
    const double* cur = slabs + (n & 1) * (kRows * rl.bw);
    if (producer) {
      if (n + 1 < nblk) {
        const int64_t rn = r0 + int64_t(n + 1) * kRows;
        produce_rows(X, y, c, rn, int(tmin<int64_t>(kRows, r1 - rn)), b, rl, c1, c2,
                     slabs + ((n + 1) & 1) * (kRows * rl.bw), ptid, true, true, bad_x);
      }
    } else {
      for (int kk = grp; kk < kRows / 4; kk += pl.G) {
        const double* row = cur + (kk * 4 + (lane & 3)) * rl.bw;
        double bK[kNF], bT[kNF];
#pragma unroll
        for (int nf = 0; nf < kNF; ++nf) {
          bK[nf] = (hasK && nf < pl.knf) ? gather_prod<FB>(row, offBK[nf]) : 0.0;
          bT[nf] = (hasT && nf < pl.tnf) ? gather_prod<FB>(row, offBT[nf]) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < kGramJobs; ++j) {
          if (jid[j] >= 0) {
            const double a = gather_prod<FA>(row, offA[j]);
            const int nfs = jK[j] ? pl.knf : pl.tnf;
#pragma unroll
            for (int nf = 0; nf < kNF; ++nf)
              if (nf < nfs) dmma_8x8x4(acc[j][nf][0], acc[j][nf][1], a, jK[j] ? bK[nf] : bT[nf]);
          }
        }
      }
    }
    __syncthreads();
  }

  if (!producer) {
    double* out = ws + (int64_t(blockIdx.x) * pl.G + grp) * pl.len;
#pragma unroll
    for (int j = 0; j < kGramJobs; ++j) {
      if (jid[j] < 0) continue;
      const int mrow = (jK[j] ? jid[j] : jid[j] - pl.kmf) * 8 + (lane >> 2);
#pragma unroll
      for (int nf = 0; nf < kNF; ++nf)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int ncol = nf * 8 + 2 * (lane & 3) + e;
          if (jK[j]) {
            if (mrow < pl.KA && ncol < pl.KB && nf < pl.knf) out[int64_t(mrow) * pl.KB + ncol] = acc[j][nf][e];
          } else {
            if (mrow < pl.TA && ncol < pl.TB && nf < pl.tnf) out[pl.Klen + int64_t(mrow) * pl.TB + ncol] = acc[j][nf][e];
          }
        }
    }
  }
  if (bad_x) raise_flag(flags, FAGP_FLAG_X_NONFINITE);
}

// out[e] = sum over partials (fixed order: deterministic); non-finite -> PHI flag
__global__ void partial_sum_kernel(const double* __restrict__ ws, int nparts, int64_t len, double* __restrict__ out,
                                   uint32_t* flags) {
  bool bad = false;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < len; e += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nparts; ++q) s += ws[int64_t(q) * len + e];
    out[e] = s;
    bad |= not_finite(s);
  }
  if (bad) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
}

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// Plan for N rows; ok = false when the shape needs the tiled table path.
static bool make_gplan(int64_t N, int p, int M, GPlan& pl) {
  std::memset(&pl, 0, sizeof(pl));
  if (!modal_on(p, M) || p > kMaxF) return false;
  pl.p = p;
  pl.M = M;
  pl.L = modal_L(M);
  pl.LC = (pl.L + 1) & ~1;
  int64_t best = -1;
  for (int pA = 1; pA < p; ++pA) {
    const int64_t KA = ipow(pl.L, pA), KB = ipow(pl.L, p - pA);
    if (ceil_div(KB, 8) > kNF || pA > kMaxF || p - pA > kMaxF) continue;
    const int64_t cost = ceil_div(KA, 8) * ceil_div(KB, 8);
    if (best < 0 || cost < best) {
      best = cost;
      pl.pA = pA;
    }
  }
  if (best < 0) return false;
  best = -1;
  for (int pT = 1; pT < p; ++pT) {
    const int64_t TA = ipow(M, pT), TB = ipow(M, p - pT);
    if (ceil_div(TB, 8) > kNF || pT > kMaxF || p - pT + 1 > kMaxF) continue;
    const int64_t cost = ceil_div(TA, 8) * ceil_div(TB, 8);
    if (best < 0 || cost < best) {
      best = cost;
      pl.pT = pT;
    }
  }
  if (best < 0) return false;
  pl.KA = int(ipow(pl.L, pl.pA));
  pl.KB = int(ipow(pl.L, p - pl.pA));
  pl.TA = int(ipow(M, pl.pT));
  pl.TB = int(ipow(M, p - pl.pT));
  pl.kmf = int(ceil_div(pl.KA, 8));
  pl.knf = int(ceil_div(pl.KB, 8));
  pl.tmf = int(ceil_div(pl.TA, 8));
  pl.tnf = int(ceil_div(pl.TB, 8));
  // Row groups G (each group of kGramCW/G warps covers every job on k-steps kk = g mod G) and
  // the job -> warp assignment (longest processing time first, cost = n-frags): choose the G
  // with the smallest per-block critical path (ceil(16/G) k-steps x the busiest warp's DMMAs).
  int bestG = -1;
  double bestc = 0.0;
  signed char bestjob[kGramCW][kGramJobs];
  for (int G = 1; G <= kGramCW; ++G) {
    if (kGramCW % G) continue;
    const int WG = kGramCW / G;
    signed char job[kGramCW][kGramJobs];
    std::memset(job, -1, sizeof(job));
    int load[kGramCW] = {0}, cnt[kGramCW] = {0};
    bool fits = true;
    for (int pass = 0; pass < 2 && fits; ++pass) {
      const bool kpass = (pl.knf >= pl.tnf) ? pass == 0 : pass == 1;
      const int nj = kpass ? pl.kmf : pl.tmf, cost = kpass ? pl.knf : pl.tnf;
      for (int j = 0; j < nj && fits; ++j) {
        int w = -1;
        for (int q = 0; q < WG; ++q)
          if (cnt[q] < kGramJobs && (w < 0 || load[q] < load[w])) w = q;
        if (w < 0) {
          fits = false;
          break;
        }
        job[w][cnt[w]++] = static_cast<signed char>(kpass ? j : pl.kmf + j);
        load[w] += cost;
      }
    }
    if (!fits) continue;
    int mx = 0;
    for (int q = 0; q < WG; ++q) mx = tmax(mx, load[q]);
    const double crit = double(mx) * double((kRows / 4 + G - 1) / G);
    if (bestG < 0 || crit < bestc - 1e-9) {
      bestG = G;
      bestc = crit;
      std::memcpy(bestjob, job, sizeof(job));
    }
  }
  if (bestG < 0) return false;
  pl.G = bestG;
  std::memcpy(pl.job, bestjob, sizeof(bestjob));
  pl.Klen = int64_t(pl.KA) * pl.KB;
  pl.len = pl.Klen + int64_t(pl.TA) * pl.TB;
  const RowLayout rl = row_layout(p, M);
  const size_t smem = (size_t(2) * pl.LC + size_t(2) * kRows * rl.bw) * sizeof(double);
  if (smem > 220 * 1024) return false;
  const int64_t blocks = tmax<int64_t>(1, ceil_div(N, kRows));
  pl.grid = int(tmin<int64_t>(num_sms(), blocks));
  pl.rows_per_cta = ceil_div(blocks, pl.grid) * kRows;
  pl.grid = int(tmax<int64_t>(1, ceil_div(tmax<int64_t>(N, 1), pl.rows_per_cta)));
  pl.nparts = pl.grid * pl.G;
  return true;
}

static size_t gram_smem(const GPlan& pl) {
  return (size_t(2) * pl.LC + size_t(2) * kRows * row_layout(pl.p, pl.M).bw) * sizeof(double);
}

template <int FA>
static int launch_gram_fb(int FB, const double* X, const double* y, double c, int64_t N, const fagp_basis* b,
                          const GPlan& pl, double* ws, uint32_t* flags, cudaStream_t s) {
  const size_t smem = gram_smem(pl);
  auto go = [&](auto kern) -> int {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const char* dbg = getenv("FAGP_DEBUG");
    if (dbg && dbg[0] == '1') {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, kern);
      fprintf(stderr, "[fagp] fused_gram: regs %d maxthreads %d static smem %zu dyn %zu local %zu grid %d block %d\n",
              fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes, smem, fa.localSizeBytes, pl.grid, kGramNT);
    }
    kern<<<pl.grid, kGramNT, smem, s>>>(X, y, c, N, view(b), pl, ws, flags);
    return FAGP_OK;
  };
  switch (FB) {
    case 1: return go(fused_gram_kernel<FA, 1>);
    case 2: return go(fused_gram_kernel<FA, 2>);
    case 3: return go(fused_gram_kernel<FA, 3>);
    case 4: return go(fused_gram_kernel<FA, 4>);
    default: return FAGP_EUNSUPPORTED;
  }
}

bool gram_eligible(int64_t N, int p, int M) {
  GPlan pl;
  return make_gplan(N, p, M, pl);
}

size_t gram_workspace(int64_t N, int p, int M) {
  GPlan pl;
  if (!make_gplan(N, p, M, pl)) return 0;
  return size_t(pl.nparts) * size_t(pl.len) * sizeof(double);
}

int gram(const double* X, const double* y, double c, int64_t N, const fagp_basis* b, double* out, void* ws,
         size_t ws_bytes, uint32_t* flags, cudaStream_t s) {
  GPlan pl;
  if (!make_gplan(N, b->p, b->M, pl)) return FAGP_EUNSUPPORTED;
  if (ws == nullptr || ws_bytes < size_t(pl.nparts) * size_t(pl.len) * sizeof(double)) return FAGP_EWORKSPACE;
  double* w = static_cast<double*>(ws);
  const int FA = tmax(pl.pA, pl.pT), FB = tmax(b->p - pl.pA, b->p - pl.pT + 1);
  int rc;
  switch (FA) {
    case 1: rc = launch_gram_fb<1>(FB, X, y, c, N, b, pl, w, flags, s); break;
    case 2: rc = launch_gram_fb<2>(FB, X, y, c, N, b, pl, w, flags, s); break;
    case 3: rc = launch_gram_fb<3>(FB, X, y, c, N, b, pl, w, flags, s); break;
    case 4: rc = launch_gram_fb<4>(FB, X, y, c, N, b, pl, w, flags, s); break;
    default: rc = FAGP_EUNSUPPORTED;
  }
  if (rc) return rc;
  FAGP_LAUNCH_CHECK();
  const int grid = int(tmax<int64_t>(1, tmin<int64_t>(ceil_div(pl.len, 256), 4 * num_sms())));
  partial_sum_kernel<<<grid, 256, 0, s>>>(w, pl.nparts, pl.len, out, flags);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

// ---------------------------------------------------------------------------------------
// Fused predict (variance + mean)
constexpr int kPredCW = 8;                              // 4 row groups x 2 K-halves
constexpr int kPredNT = (kPredCW + kProdWarps) * 32;    // 320 threads

struct VPlan {
  int p, M, L, LC;
  int pN;                  // variance: N side dims [0,pN) (epilogue), K side [pN,p), radix L
  int NR, KR, vnf, vks;    // N extent (<= 24), K extent, n-frags, k-steps of 4
  int NM, KM, mnf, mks;    // mean: N side dim 0 (M), K side dims [1,p) (M^(p-1))
  int64_t KP, NP;          // predict_op layout (modal::Plan): C'' [KP][NP], then w (m)
  int64_t nblocks;
  int grid;
  size_t smem;
};

// byte-packed factor offsets of K column kappa (FK factors, 8 bits each; offsets < 256)
template <int F>
__device__ __forceinline__ void unpack_off(uint32_t v, int (&off)[F]) {
#pragma unroll
  for (int f = 0; f < F; ++f) off[f] = int((v >> (8 * f)) & 0xffu);
}

template <int FK, int FE, int FKM>
__global__ void __launch_bounds__(kPredNT, 1)
fused_predict_kernel(const double* __restrict__ Xs, int64_t Ns, BasisView b, const VPlan pl,
                     const double* __restrict__ op, double sigma2, double c, double* __restrict__ mean,
                     double* __restrict__ var, uint32_t* flags) {
  extern __shared__ double sm[];
  const RowLayout rl = row_layout(pl.p, pl.M);
  const bool want_var = var != nullptr;
  double* c1 = sm;
  double* c2 = sm + pl.LC;
  double* Bv = c2 + pl.LC;                          // [vks][vnf][32]
  double* Bm = Bv + pl.vks * pl.vnf * 32;           // [mks][mnf][32]
  double* red = Bm + pl.mks * pl.mnf * 32;          // [4 mg][2 mf][kNF][2][2 (var, mean)][32]
  double* slabs = red + 4 * 2 * kNF * 2 * 2 * 32;   // [2][kRows * bw]
  uint32_t* offV = reinterpret_cast<uint32_t*>(slabs + 2 * kRows * rl.bw);  // [vks * 4]
  uint32_t* offM = offV + pl.vks * 4;                                       // [mks * 4]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* w = op + pl.KP * pl.NP;
  for (int k = tid; k < pl.LC; k += kPredNT) {
    c1[k] = herm_c1(k);
    c2[k] = herm_c2(k);
  }
  // operands, fragment-major: B[ks][nf][lane] = Op[4 ks + (lane & 3)][8 nf + (lane >> 2)]
  if (want_var)
    for (int i = tid; i < pl.vks * pl.vnf * 32; i += kPredNT) {
      const int ln = i & 31, q = i >> 5, nf = q % pl.vnf, ks = q / pl.vnf;
      const int kap = 4 * ks + (ln & 3), nu = 8 * nf + (ln >> 2);
      Bv[i] = (kap < pl.KR && nu < pl.NR) ? op[int64_t(kap) * pl.NP + nu] : 0.0;
    }
  for (int i = tid; i < pl.mks * pl.mnf * 32; i += kPredNT) {
    const int ln = i & 31, q = i >> 5, nf = q % pl.mnf, ks = q / pl.mnf;
    const int kap = 4 * ks + (ln & 3), nu = 8 * nf + (ln >> 2);
    Bm[i] = (kap < pl.KM && nu < pl.NM) ? w[int64_t(nu) * pl.KM + kap] : 0.0;
  }
  // K-column factor offsets (variance: g of dims [pN,p); mean: phi of dims [1,p))
  for (int kap = tid; kap < pl.vks * 4; kap += kPredNT) {
    int off[FK];
    col_offsets<FK>(kap, pl.KR, rl.goff, pl.pN, pl.p - pl.pN, pl.L, -1, rl, off);
    uint32_t v = 0;
#pragma unroll
    for (int f = 0; f < FK; ++f) v |= uint32_t(off[f]) << (8 * f);
    offV[kap] = v;
  }
  for (int kap = tid; kap < pl.mks * 4; kap += kPredNT) {
    int off[FKM];
    col_offsets<FKM>(kap, pl.KM, rl.poff, 1, pl.p - 1, pl.M, -1, rl, off);
    uint32_t v = 0;
#pragma unroll
    for (int f = 0; f < FKM; ++f) v |= uint32_t(off[f]) << (8 * f);
    offM[kap] = v;
  }
  const bool producer = warp >= kPredCW;
  const int ptid = tid - kPredCW * 32;
  bool bad_x = false, bad = false;
  __syncthreads();
  const int64_t blk0 = blockIdx.x;
  const int64_t stride = gridDim.x;
  if (producer && blk0 < pl.nblocks) {
    const int64_t rr = blk0 * kRows;
    produce_rows(Xs, nullptr, 0.0, rr, int(tmin<int64_t>(kRows, Ns - rr)), b, rl, c1, c2, slabs, ptid, true,
                 want_var, bad_x);
  }
  // consumer roles
  const int mg = warp & 3, kh = (warp >> 2) & 1;
  const int vk0 = kh ? (pl.vks + 1) / 2 : 0, vk1 = kh ? pl.vks : (pl.vks + 1) / 2;
  const int mk0 = kh ? (pl.mks + 1) / 2 : 0, mk1 = kh ? pl.mks : (pl.mks + 1) / 2;
  // epilogue factor offsets: variance E[i, nu] = prod_{d < pN} g_d; mean phi_0[i, nu]
  int offE[kNF][2][FE], offEm[kNF][2];
#pragma unroll
  for (int nf = 0; nf < kNF; ++nf)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int nu = nf * 8 + 2 * (lane & 3) + e;
      col_offsets<FE>(nu, pl.NR, rl.goff, 0, pl.pN, pl.L, -1, rl, offE[nf][e]);
      offEm[nf][e] = nu < pl.NM ? rl.poff + nu : rl.zero;
    }
  __syncthreads();

  int it = 0;
  for (int64_t blk = blk0; blk < pl.nblocks; blk += stride, ++it) {
    const double* cur = slabs + (it & 1) * (kRows * rl.bw);
    if (producer) {
      const int64_t nb = blk + stride;
      if (nb < pl.nblocks) {
        const int64_t rr = nb * kRows;
        produce_rows(Xs, nullptr, 0.0, rr, int(tmin<int64_t>(kRows, Ns - rr)), b, rl, c1, c2,
                     slabs + ((it + 1) & 1) * (kRows * rl.bw), ptid, true, want_var, bad_x);
      }
    } else {
      const double* rowA = cur + (mg * 16 + (lane >> 2)) * rl.bw;  // m-frag 0 row; m-frag 1 = +8 rows
      const double* rowB = rowA + 8 * rl.bw;
      double accV[2][kNF][2], accM[2][kNF][2];
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int nf = 0; nf < kNF; ++nf) accV[f][nf][0] = accV[f][nf][1] = accM[f][nf][0] = accM[f][nf][1] = 0.0;
      if (want_var) {
        for (int ks = vk0; ks < vk1; ++ks) {
          int off[FK];
          unpack_off<FK>(offV[4 * ks + (lane & 3)], off);
          const double a0 = gather_prod<FK>(rowA, off), a1 = gather_prod<FK>(rowB, off);
          const double* bp = Bv + (ks * pl.vnf) * 32 + lane;
#pragma unroll
          for (int nf = 0; nf < kNF; ++nf)
            if (nf < pl.vnf) {
              const double bb = bp[nf * 32];
              dmma_8x8x4(accV[0][nf][0], accV[0][nf][1], a0, bb);
              dmma_8x8x4(accV[1][nf][0], accV[1][nf][1], a1, bb);
            }
        }
      }
      for (int ks = mk0; ks < mk1; ++ks) {
        int off[FKM];
        unpack_off<FKM>(offM[4 * ks + (lane & 3)], off);
        const double a0 = gather_prod<FKM>(rowA, off), a1 = gather_prod<FKM>(rowB, off);
        const double* bp = Bm + (ks * pl.mnf) * 32 + lane;
#pragma unroll
        for (int nf = 0; nf < kNF; ++nf)
          if (nf < pl.mnf) {
            const double bb = bp[nf * 32];
            dmma_8x8x4(accM[0][nf][0], accM[0][nf][1], a0, bb);
            dmma_8x8x4(accM[1][nf][0], accM[1][nf][1], a1, bb);
          }
      }
      // split-K: the upper K-half hands its partial sums to the lower one (fixed order)
      double* rp = red + mg * (2 * kNF * 2 * 2 * 32);
      if (kh) {
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int nf = 0; nf < kNF; ++nf)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              rp[(((f * kNF + nf) * 2 + e) * 2 + 0) * 32 + lane] = accV[f][nf][e];
              rp[(((f * kNF + nf) * 2 + e) * 2 + 1) * 32 + lane] = accM[f][nf][e];
            }
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(kPredCW * 32));
      if (!kh) {
        const int64_t rbase = blk * kRows + mg * 16 + (lane >> 2);
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const double* row = f ? rowB : rowA;
          double vs = 0.0, ms = 0.0;
#pragma unroll
          for (int nf = 0; nf < kNF; ++nf)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const double yv = accV[f][nf][e] + rp[(((f * kNF + nf) * 2 + e) * 2 + 0) * 32 + lane];
              const double zv = accM[f][nf][e] + rp[(((f * kNF + nf) * 2 + e) * 2 + 1) * 32 + lane];
              if (nf < pl.vnf && want_var) vs = fma(yv, gather_prod<FE>(row, offE[nf][e]), vs);
              if (nf < pl.mnf) ms = fma(zv, row[offEm[nf][e]], ms);
            }
          // the 4 lanes of a row hold disjoint columns: fixed-order xor reduction
          vs += __shfl_xor_sync(0xffffffffu, vs, 1);
          vs += __shfl_xor_sync(0xffffffffu, vs, 2);
          ms += __shfl_xor_sync(0xffffffffu, ms, 1);
          ms += __shfl_xor_sync(0xffffffffu, ms, 2);
          const int64_t row_i = rbase + 8 * f;
          if ((lane & 3) == 0 && row_i < Ns) {
            const double mm = c + ms;  // posterior.py:247
            mean[row_i] = mm;
            bad |= not_finite(mm);
            if (want_var) {
              const double vv = sigma2 * vs;
              var[row_i] = vv;
              bad |= not_finite(vv);
            }
          }
        }
      }
    }
    __syncthreads();
  }
  if (bad_x) raise_flag(flags, FAGP_FLAG_X_NONFINITE);
  if (bad) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
}

static bool make_vplan(int64_t Ns, int p, int M, VPlan& pl) {
  std::memset(&pl, 0, sizeof(pl));
  if (!modal_on(p, M) || p > kMaxF || M > 24) return false;
  const modal::Plan mp = modal::make_plan(0, p, M);
  pl.p = p;
  pl.M = M;
  pl.L = modal_L(M);
  pl.LC = (pl.L + 1) & ~1;
  pl.pN = mp.pN;
  pl.NR = int(mp.NR);
  pl.KR = int(mp.KR);
  pl.KP = mp.KP;
  pl.NP = mp.NP;
  if (pl.NR > 8 * kNF || p - pl.pN > kMaxF || pl.pN > 2) return false;
  pl.vnf = int(ceil_div(pl.NR, 8));
  pl.vks = int(ceil_div(pl.KR, 4));
  pl.NM = M;
  pl.KM = int(ipow(M, p - 1));
  pl.mnf = int(ceil_div(pl.NM, 8));
  pl.mks = int(ceil_div(pl.KM, 4));
  const RowLayout rl = row_layout(p, M);
  if (rl.bw > 256) return false;  // byte-packed offsets
  pl.smem = (size_t(2) * pl.LC + size_t(pl.vks) * pl.vnf * 32 + size_t(pl.mks) * pl.mnf * 32 +
             size_t(4) * 2 * kNF * 2 * 2 * 32 + size_t(2) * kRows * rl.bw) * sizeof(double) +
            size_t(pl.vks + pl.mks) * 4 * sizeof(uint32_t);
  if (pl.smem > 225 * 1024) return false;
  pl.nblocks = ceil_div(tmax<int64_t>(Ns, 0), kRows);
  pl.grid = int(tmax<int64_t>(1, tmin<int64_t>(num_sms(), pl.nblocks)));
  return true;
}

template <int FK>
static int launch_pred_fe(int FE, const double* Xs, int64_t Ns, const fagp_basis* b, const VPlan& pl, const double* op,
                          double sigma2, double c, double* mean, double* var, uint32_t* flags, cudaStream_t s) {
  auto go = [&](auto kern) -> int {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem)));
    kern<<<pl.grid, kPredNT, pl.smem, s>>>(Xs, Ns, view(b), pl, op, sigma2, c, mean, var, flags);
    return FAGP_OK;
  };
  // FKM = p - 1 = FK + FE - 1
  switch (FE) {
    case 1:
      return go(fused_predict_kernel<FK, 1, FK>);
    case 2:
      if constexpr (FK + 1 <= kMaxF) return go(fused_predict_kernel<FK, 2, FK + 1>);
      return FAGP_EUNSUPPORTED;
    default:
      return FAGP_EUNSUPPORTED;
  }
}

bool predict_eligible(int p, int M) {
  VPlan pl;
  return make_vplan(1, p, M, pl);
}

int predict(const double* Xs, int64_t Ns, const fagp_basis* b, const double* op, double sigma2, double c,
            double* mean, double* var, uint32_t* flags, cudaStream_t s) {
  VPlan pl;
  if (!make_vplan(Ns, b->p, b->M, pl)) return FAGP_EUNSUPPORTED;
  if (Ns == 0) return FAGP_OK;
  const int FK = b->p - pl.pN, FE = pl.pN;
  int rc;
  switch (FK) {
    case 1: rc = launch_pred_fe<1>(FE, Xs, Ns, b, pl, op, sigma2, c, mean, var, flags, s); break;
    case 2: rc = launch_pred_fe<2>(FE, Xs, Ns, b, pl, op, sigma2, c, mean, var, flags, s); break;
    case 3: rc = launch_pred_fe<3>(FE, Xs, Ns, b, pl, op, sigma2, c, mean, var, flags, s); break;
    default: rc = FAGP_EUNSUPPORTED;
  }
  if (rc) return rc;
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // namespace fused
}  // namespace fagp

// =======================================================================================
// C ABI: the point-input entry points (tables only where the fused layouts do not apply)
using namespace fagp;

extern "C" {

size_t fagp_gram_x_workspace_size(int64_t N, const fagp_basis* basis) {
  if (check_basis(basis) || N < 0) return 0;
  if (fused::gram_eligible(N, basis->p, basis->M)) return fused::gram_workspace(N, basis->p, basis->M);
  const size_t table = size_t(N) * table_width(basis->p, basis->M) * sizeof(double);
  return round_up(table, 256) + fagp_gram_workspace_size(N, basis);
}

int fagp_gram_x(const double* X, int64_t N, const fagp_basis* basis, const double* y, double mean_const,
                double* gram, void* workspace, size_t workspace_bytes, uint32_t* flags, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || gram == nullptr || (N > 0 && X == nullptr)) return FAGP_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (fused::gram_eligible(N, basis->p, basis->M))
    return fused::gram(X, y, mean_const, N, basis, gram, workspace, workspace_bytes, flags, s);
  const size_t table = round_up(size_t(N) * table_width(basis->p, basis->M) * sizeof(double), 256);
  if (workspace == nullptr || workspace_bytes < table + fagp_gram_workspace_size(N, basis)) return FAGP_EWORKSPACE;
  double* T = static_cast<double*>(workspace);
  if (N > 0) {
    st = fagp_basis_eval(X, N, basis, y, mean_const, T, flags, stream);
    if (st) return st;
  }
  return fagp_gram(T, N, basis, gram, static_cast<char*>(workspace) + table, workspace_bytes - table, flags, stream);
}

size_t fagp_predict_x_workspace_size(int64_t Ns, const fagp_basis* basis) {
  if (check_basis(basis) || Ns < 0) return 0;
  if (fused::predict_eligible(basis->p, basis->M)) return 0;
  return size_t(Ns) * table_width(basis->p, basis->M) * sizeof(double);
}

int fagp_predict_x(const double* Xs, int64_t Ns, const fagp_basis* basis, const double* predict_op, double sigma2,
                   double mean_const, double* mean, double* var, uint32_t* flags, void* workspace,
                   size_t workspace_bytes, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (Ns < 0 || predict_op == nullptr || (Ns > 0 && (Xs == nullptr || mean == nullptr))) return FAGP_EINVAL;
  if (Ns == 0) return FAGP_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (fused::predict_eligible(basis->p, basis->M))
    return fused::predict(Xs, Ns, basis, predict_op, sigma2, mean_const, mean, var, flags, s);
  const size_t table = size_t(Ns) * table_width(basis->p, basis->M) * sizeof(double);
  if (workspace == nullptr || workspace_bytes < table) return FAGP_EWORKSPACE;
  double* Ts = static_cast<double*>(workspace);
  st = fagp_basis_eval(Xs, Ns, basis, nullptr, 0.0, Ts, flags, stream);
  if (st) return st;
  return fagp_predict(Ts, Ns, basis, predict_op, sigma2, mean_const, mean, var, flags, stream);
}

}  // extern "C"
