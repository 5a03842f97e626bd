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
//  * Production / contraction phases.  Every block of rows (128 rows, 256 in the split Gram) starts
//    with a production phase in which all warps evaluate the 1-D eigenfunctions (one or two
//    (row, dimension) items per thread; mercer.py:122-143, 276-281, bit-faithful op order,
//    eigfun.cuh) into a shared-memory row slab, then all warps run the DMMA contraction over it.
//    (A dedicated producer warp group overlapping the contraction was measured slower: its
//    dependent FP64 recurrence chains starve behind the DMMAs in the shared FP64 pipe.)  Nothing
//    but X (and y) is read from HBM: 24 B per row at p = 3 instead of the 752 B table row.
//  * Register-generated DMMA fragments.  Every mma.m8n8k4.f64 operand that is a product of
//    basis values (g g, phi phi, r phi) is formed in the thread that feeds it to the tensor
//    core (FA/FB/FK LDS.64 + DMULs, conflict-free thanks to a row stride == 4 mod 16 doubles),
//    so generated operands never round-trip through shared memory.
//  * Gram: each CTA owns a contiguous row range and accumulates the WHOLE output ([K | t]:
//    46 x 3 + 13 x 2 8x8 fragments at C3) in registers of its 16 warps; one CTA per SM,
//    persistent; per-CTA partials are summed in a fixed order by a second small kernel
//    (deterministic, no float atomics) -- the same buffer the multi-GPU path all-reduces.
//  * Predict: the variance operand C'' and the mean weights are staged once per CTA into
//    shared memory in fragment-major order (one conflict-free LDS.64 per B fragment); 16
//    warps = 8 row groups (16 rows each) x 2 K-halves (split-K reduced through shared memory);
//    the g / phi epilogue products and the 4-lane row reductions stay in registers; mean and
//    variance come out of the same pass.
// Shapes whose output does not fit these layouts use the tiled table kernels (modal.cu,
// gram.cu, predict.cu) -- see fagp_gram_x / fagp_predict_x.
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "eigfun.cuh"
#include "modal.cuh"

namespace fagp {
namespace fused {

// ---------------------------------------------------------------------------------------
// Shared-memory row slab: [g_{d,k} (p L) | phi_{d,a} (p M) | r phi_{p-1,a} (M) | r | 1.0 | 0.0 | pad],
// stride BW with BW % 16 == 4 so 4 rows x 4 consecutive doubles hit 16 distinct bank pairs.
struct RowLayout {
  int goff, poff, rpoff, roff, one, zero, bw;
};
__host__ __device__ inline RowLayout row_layout(int p, int M) {
  const int L = modal_L(M);
  RowLayout r;
  r.goff = 0;
  r.poff = p * L;
  r.rpoff = p * L + p * M;
  r.roff = r.rpoff + M;
  r.one = r.roff + 1;
  r.zero = r.roff + 2;
  int w = r.zero + 1;
  while (w % 16 != 4) ++w;
  r.bw = w;
  return r;
}

constexpr int kRows = 64;      // rows per block (16 DMMA k-steps of 4 rows)
constexpr int kMaxF = 4;       // factors per generated column (p <= 4 on the fused path)

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
// Fused Gram.  16 warps = 4 per SM sub-partition (each sub-partition owns a quarter of the
// register file, so this is the most warps that keep 128 registers per thread) and no
// dedicated producer: warp w evaluates the eigenfunctions of rows [4w, 4w + 4) of the NEXT
// 64-row block at a point of its k-loop staggered against the other three warps of its
// sub-partition, which keep the DMMA pipe busy meanwhile.
// Output columns (first dimension slowest, A side = dims [0, p-1), B side = dim p-1):
//   K: A = g-products (L^(p-1)) x B = g (L)          t: A = phi-products (M^(p-1)) x B = phi * r (M)
// Warp wi of a row group owns K m-fragments wi + WG j (j < JK) and t m-fragments wi + WG j
// (j < JT), each against every B fragment: all counts compile-time, no predication.
constexpr int kGramW = 16;
constexpr int kGramNT = kGramW * 32;
constexpr int kGR = 128;                // rows per block (32 k-steps): one barrier per 128 rows
constexpr int kSR = 256;                // rows per block of the split kernel (one slab, 2 rows per producer)

struct GPlan {
  int p, M, L, LC;
  int KA, KB, TA, TB;  // KA = L^(p-1), KB = L, TA = M^(p-1), TB = M
  int kmf, tmf;        // A-side m-fragments of K and t
  int G, WG;           // row groups per CTA (k-steps kk = g mod G) and warps per group
  int JK, JT;          // m-fragments per warp
  int64_t Klen, len;   // output layout [K (KA*KB) | t (TA*TB = m)]
  int64_t plen;        // one partial: (kmf NFK + tmf NFT) fragments of 64 doubles
  int br;                // rows per block (kGR, or kSR for the split kernel)
  int64_t rows_per_cta;  // rows of one CTA (a multiple of 4; the last block of a CTA may be partial)
  int bpc;               // blocks per CTA = ceil(rows_per_cta / br)
  int S;                 // sub-ranges per CTA = chunks a host pipeline may launch separately
  int grid, nparts;      // nparts = grid * S * G partials
  HermCoef hc;           // recurrence coefficients (constant-bank operands)
  // split layout (p = 3, M = 10): the ragged last n-fragment of K / t contracted with the
  // roles of the last two dimensions swapped (see fused_gram_split_kernel)
  int split, W1, R, R2;          // warps in role 1; L - 16; M - 8
  int kmf1, kmf2, tmf1, tmf2;    // m-fragments of K1, K2, T1, T2
  int baseK2, baseT1, baseT2;    // fragment offsets of the sections in a partial
  // physical warp -> slot (slot < W1: role-1 warp index, else W1 + role-2 index): warp w issues on
  // SM sub-partition w % 4, and the slots' useful DMMA counts differ (reduced classes), so the
  // slots are dealt to balance the sub-partitions (C3: 36 -> 34 DMMA per k-step on the busiest)
  unsigned char wslot[kGramW];
  // launch mode: once = one partial per (CTA, row group) flushed at the end of the launch
  // (slot cta G + grp) instead of one per sub-range; ready (nullable) = per-sub-range words a
  // host pipeline sets non-zero (by a stream-ordered H2D copy) once the sub-range's rows landed
  int once;
  const unsigned* ready;
};

// Wait until *r != 0 (acquire).  Bounded: after ~2 s the STALLED flag is raised and the kernel
// carries on (garbage results, reported), so a lost signal cannot hang the device.
__device__ __noinline__ void wait_ready(const unsigned* r, uint32_t* flags) {
  const long long t0 = clock64();
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(r) : "memory");
    if (v) return;
    if (clock64() - t0 > (4ll << 30)) {
      raise_flag(flags, FAGP_FLAG_STALLED);
      return;
    }
    __nanosleep(500);
  }
}

#ifdef FAGP_GRAM_PROFILE
__device__ long long g_gram_prof[4];
extern "C" int fagp_debug_gram_profile(long long* out) {  // diagnostics build only
  return cudaMemcpyFromSymbol(out, g_gram_prof, sizeof(g_gram_prof)) == cudaSuccess ? 0 : 5;
}
#endif

template <int FA, int NFK, int NFT, int JK, int JT>
__global__ void __launch_bounds__(kGramNT, 1)
fused_gram_kernel(const double* __restrict__ X, const double* __restrict__ y, double c, int64_t N, BasisView b,
                  const GPlan pl, int k0, int k1, double* __restrict__ ws, uint32_t* flags) {
  extern __shared__ double sm[];
  const RowLayout rl = row_layout(pl.p, pl.M);
  double* c1 = sm;
  double* c2 = sm + pl.LC;
  double* slabs = sm + 2 * pl.LC;  // [2][kGR * bw]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int p = pl.p, M = pl.M, L = pl.L;
  for (int k = tid; k < pl.LC; k += kGramNT) {
    c1[k] = herm_c1(k);
    c2[k] = herm_c2(k);
  }
  // CTA rows [cta rpc, (cta + 1) rpc) = blocks [0, bpc) of kGR rows, cut into pl.S sub-ranges
  // (sub-range k = blocks [k bpc / S, (k + 1) bpc / S)); this launch covers sub-ranges [k0, k1)
  // and writes one partial per (CTA, sub-range, row group)
  const int cta = int(blockIdx.x);
  const int bpc = pl.bpc;
  auto sb = [&](int k) { return int(int64_t(k) * bpc / pl.S); };
  const int g0 = sb(k0);
  const int nblk = sb(k1) - g0;
  const int64_t cta_end = tmin<int64_t>(N, int64_t(cta + 1) * pl.rows_per_cta);
  auto blk_base = [&](int j) -> int64_t { return int64_t(cta) * pl.rows_per_cta + int64_t(g0 + j) * kGR; };
  auto blk_end = [&](int j) -> int64_t { return tmin<int64_t>(cta_end, blk_base(j) + kGR); };
  bool bad_x = false;

  // production: thread t < kGR p evaluates phi and g (one shared exponential, two independent
  // recurrences) of row t / p, dimension t % p; the last dimension also writes r phi.  x and y of
  // the next block are loaded one block ahead.
  const bool plane = tid < kGR * p;
  const int prow = tid / p, pdim = tid - (tid / p) * p;
  struct Pre {
    double x, y;
  };
  // pipelined launch: block j's rows may only be read once its sub-range's ready word is set.
  // The look-ahead load probes the word; if it is not set yet the load is deferred (pend = j)
  // and done, waiting, right before block j is produced -- never stalling the contraction of
  // the block already staged.
  int seen = k0 - 1;  // last sub-range whose ready word this thread has observed
  int pend = -1;
  auto load_pre = [&](int j, Pre& pr, bool block = false) {
    if (pl.ready && plane) {
      int k = k0;
      while (k + 1 < k1 && g0 + j >= sb(k + 1)) ++k;
      if (k > seen) {
        if (block) {
          wait_ready(pl.ready + k, flags);
        } else {
          unsigned v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(pl.ready + k) : "memory");
          if (!v) {
            pend = j;
            return;
          }
        }
        seen = k;
      }
    }
    const int64_t r = blk_base(j) + prow;
    const bool ok = plane && r < blk_end(j);
    pr.x = ok ? X[r * p + pdim] : 0.0;
    pr.y = (ok && y != nullptr && pdim == p - 1) ? y[r] : c;
  };
  auto produce = [&](const Pre& pr, int j, double* slab) {
    if (!plane) return;
    double* row = slab + prow * rl.bw;
    const bool valid = blk_base(j) + prow < blk_end(j);
    if (valid) {
      bad_x |= not_finite(pr.x);
      const double rr = __dsub_rn(pr.y, c);  // r = y - c (posterior.py:229)
      eval_phi_g_dim_u(pr.x, rr, b, pdim, pl.hc, row + rl.poff + pdim * M, row + rl.goff + pdim * L,
                       pdim == p - 1 ? row + rl.rpoff : nullptr);
    } else {
      for (int k = 0; k < M; ++k) row[rl.poff + pdim * M + k] = 0.0;
      for (int k = 0; k < L; ++k) row[rl.goff + pdim * L + k] = 0.0;
      if (pdim == p - 1)
        for (int k = 0; k < M; ++k) row[rl.rpoff + k] = 0.0;
    }
    if (pdim == 0) {
      row[rl.one] = 1.0;
      row[rl.zero] = 0.0;
    }
  };
  __syncthreads();
  Pre pre;
  if (nblk > 0) {
    load_pre(0, pre, true);
    produce(pre, 0, slabs);
  }
  if (nblk > 1) load_pre(1, pre);

  const int grp = warp / pl.WG, wi = warp - grp * pl.WG;
  int offAK[JK][FA], offAT[JT][FA], offBK[NFK], offBT[NFT];
#pragma unroll
  for (int j = 0; j < JK; ++j)
    col_offsets<FA>((wi + pl.WG * j) * 8 + (lane >> 2), pl.KA, rl.goff, 0, p - 1, L, -1, rl, offAK[j]);
#pragma unroll
  for (int j = 0; j < JT; ++j)
    col_offsets<FA>((wi + pl.WG * j) * 8 + (lane >> 2), pl.TA, rl.poff, 0, p - 1, M, -1, rl, offAT[j]);
#pragma unroll
  for (int nf = 0; nf < NFK; ++nf) {
    int o[1];
    col_offsets<1>(nf * 8 + (lane >> 2), pl.KB, rl.goff, p - 1, 1, L, -1, rl, o);
    offBK[nf] = o[0];
  }
#pragma unroll
  for (int nf = 0; nf < NFT; ++nf) {
    int o[1];
    col_offsets<1>(nf * 8 + (lane >> 2), pl.TB, rl.rpoff, 0, 1, M, -1, rl, o);
    offBT[nf] = o[0];
  }
  double accK[JK][NFK][2], accT[JT][NFT][2];
#pragma unroll
  for (int j = 0; j < JK; ++j)
#pragma unroll
    for (int nf = 0; nf < NFK; ++nf) accK[j][nf][0] = accK[j][nf][1] = 0.0;
#pragma unroll
  for (int j = 0; j < JT; ++j)
#pragma unroll
    for (int nf = 0; nf < NFT; ++nf) accT[j][nf][0] = accT[j][nf][1] = 0.0;
  const int nloc = (kGR / 4 - grp + pl.G - 1) / pl.G;  // k-steps of this warp per block
  __syncthreads();

  // one k-step = 4 rows: operands (B: K g-values, t r*phi-values; A: products over the first p-1
  // dims) then the DMMAs.  kloop software-pipelines: operands of step i + 1 are formed in program
  // order before the DMMAs of step i.
  struct Ops {
    double bK[NFK], bT[NFT], aK[JK], aT[JT];
  };
  auto load_ops = [&](const double* cur, int i, Ops& o) {
    const double* row = cur + ((grp + i * pl.G) * 4 + (lane & 3)) * rl.bw;
#pragma unroll
    for (int nf = 0; nf < NFK; ++nf) o.bK[nf] = row[offBK[nf]];
#pragma unroll
    for (int nf = 0; nf < NFT; ++nf) o.bT[nf] = row[offBT[nf]];
#pragma unroll
    for (int j = 0; j < JK; ++j) o.aK[j] = gather_prod<FA>(row, offAK[j]);
#pragma unroll
    for (int j = 0; j < JT; ++j) o.aT[j] = gather_prod<FA>(row, offAT[j]);
  };
  auto mma_ops = [&](const Ops& o) {
#pragma unroll
    for (int j = 0; j < JK; ++j)
#pragma unroll
      for (int nf = 0; nf < NFK; ++nf) dmma_8x8x4(accK[j][nf][0], accK[j][nf][1], o.aK[j], o.bK[nf]);
#pragma unroll
    for (int j = 0; j < JT; ++j)
#pragma unroll
      for (int nf = 0; nf < NFT; ++nf) dmma_8x8x4(accT[j][nf][0], accT[j][nf][1], o.aT[j], o.bT[nf]);
  };
  auto kloop = [&](const double* cur, int i0, int i1) {
    if (i0 >= i1) return;
    Ops o;
    load_ops(cur, i0, o);
    for (int i = i0; i < i1; ++i) {
      Ops on;
      load_ops(cur, i + 1 < i1 ? i + 1 : i, on);
      mma_ops(o);
      o = on;
    }
  };
  // partial of sub-range k in fragment-major order (coalesced: one 256 B store per fragment
  // half), then restart the accumulators; partial_sum_kernel maps it back to [K | t]
  auto flush = [&](int k) {
    double* out = ws + ((pl.once ? int64_t(cta) : int64_t(cta) * pl.S + k) * pl.G + grp) * pl.plen;
#pragma unroll
    for (int j = 0; j < JK; ++j) {
      const int mf = wi + pl.WG * j;
#pragma unroll
      for (int nf = 0; nf < NFK; ++nf) {
        if (mf < pl.kmf)
          *reinterpret_cast<double2*>(out + (int64_t(mf) * NFK + nf) * 64 + 2 * lane) =
              make_double2(accK[j][nf][0], accK[j][nf][1]);
        accK[j][nf][0] = accK[j][nf][1] = 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < JT; ++j) {
      const int mf = wi + pl.WG * j;
#pragma unroll
      for (int nf = 0; nf < NFT; ++nf) {
        if (mf < pl.tmf)
          *reinterpret_cast<double2*>(out + (int64_t(pl.kmf) * NFK + int64_t(mf) * NFT + nf) * 64 + 2 * lane) =
              make_double2(accT[j][nf][0], accT[j][nf][1]);
        accT[j][nf][0] = accT[j][nf][1] = 0.0;
      }
    }
  };
#ifdef FAGP_GRAM_PROFILE
  long long tp[4] = {0, 0, 0, 0};  // kloop, produce, flush, barrier (clock64 cycles)
#define GPROF(i, stmt)              \
  {                                 \
    const long long t_ = clock64(); \
    stmt;                           \
    tp[i] += clock64() - t_;        \
  }
#else
#define GPROF(i, stmt) stmt;
#endif
  // Production of block n + 1 runs as its own phase at the top of block n, all warps together:
  // overlapped with other warps' DMMAs its FP64 chains starve (DMUL and DMMA share one pipe and
  // the dependent recurrence waits behind every DMMA), costing ~40% of each warp's time; alone it
  // is ~1.5k cycles against ~22k of DMMA per block.
  for (int n = 0; n < nblk; ++n) {
    const double* cur = slabs + (n & 1) * (kGR * rl.bw);
    if (n + 1 < nblk) {
      if (pend == n + 1) {
        load_pre(n + 1, pre, true);
        pend = -1;
      }
      GPROF(1, produce(pre, n + 1, slabs + ((n + 1) & 1) * (kGR * rl.bw)); if (n + 2 < nblk) load_pre(n + 2, pre))
    }
    GPROF(0, kloop(cur, 0, nloc))
    if (pl.once) {
      if (n + 1 == nblk) flush(0);
    } else {
      GPROF(2, for (int k = k0; k < k1; ++k) if (g0 + n + 1 == sb(k + 1)) flush(k))
    }
    GPROF(3, __syncthreads())
  }
#ifdef FAGP_GRAM_PROFILE
  if (lane == 0)
    for (int i = 0; i < 4; ++i) atomicAdd(reinterpret_cast<unsigned long long*>(&g_gram_prof[i]), (unsigned long long)tp[i]);
#endif
#undef GPROF
  if (bad_x) raise_flag(flags, FAGP_FLAG_X_NONFINITE);
}

// ---------------------------------------------------------------------------------------
// Split-layout fused Gram for p = 3 (M = 10: L = 19 = 16 + 3, M = 8 + 2).  The last dimension's
// 8-column fragments leave 3 of L (2 of M) columns ragged; instead of padding them to a full
// fragment against all L^2 (M^2) A columns, they are contracted with the roles of dims 1 and 2
// swapped:
//   K1: A = g0 g1 (L^2 columns) x B = g2[0, 16)            K2: A = (g0, g2[16, L)) x B = g1
//   T1: A = phi0 phi1 (M^2)     x B = r phi2[0, 8)         T2: A = (phi0, r phi2[8, M)) x B = phi1
// 135 DMMA per 4-row k-step at C3 instead of 164.  Role 1 warps (w < W1) own JK1 K1 and JT1A T1
// m-fragments, role 2 warps JK2 K2, JT2 T2 and JT1B T1 m-fragments (fragment ids strided by the
// role's warp count), 9 DMMA per warp per k-step each.  Production, blocks, sub-ranges and the
// partial flush are those of fused_gram_kernel.
constexpr int kSplitGramBW = 100;  // row_layout(3, 10).bw
#ifndef FAGP_GRAM_UNROLL
#define FAGP_GRAM_UNROLL 8  // split Gram k-loop unroll per 64-k-step block (measured 4 / 8 / 16 / 32: 0.689 / 0.679 / 0.687 / 0.712 ms at C3: the 5 warp classes run different straight-line k-steps at once, so longer unrolls spill out of the instruction cache)
#endif
constexpr int kGramUnroll = FAGP_GRAM_UNROLL;
template <int JK1, int JT1A, int JK2, int JT2, int JT1B, int BR>
__global__ void __launch_bounds__(kGramNT, 1)
fused_gram_split_kernel(const double* __restrict__ X, const double* __restrict__ y, double c, int64_t N,
                        BasisView b, const GPlan pl, int k0, int k1, double* __restrict__ ws, uint32_t* flags) {
  extern __shared__ double sm[];
  constexpr int p = 3;
  // BR = kGR: two slabs, block n + 1 produced while block n is contracted; BR = kSR: one slab of
  // 256 rows, each producer thread evaluating two rows in lockstep (two independent recurrence
  // chains hide each other's FP64 latency), then a barrier, then 64 k-steps
  constexpr int PR = BR / kGR;
  constexpr int NSLAB = PR == 1 ? 2 : 1;
  const RowLayout rl = row_layout(p, pl.M);
  // the row stride as a compile-time constant (row_layout(3, 10).bw, checked on the host): every
  // operand address of a k-step is then a loop-invariant register plus an immediate -- no
  // per-load address arithmetic in the k-loop
  constexpr int SBW = kSplitGramBW;
  double* slabs = sm;  // [NSLAB][BR * bw]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = pl.M, L = pl.L;
  const int cta = int(blockIdx.x);
  const int bpc = pl.bpc;
  auto sb = [&](int k) { return int(int64_t(k) * bpc / pl.S); };
  const int g0 = sb(k0);
  const int nblk = sb(k1) - g0;
  const int64_t cta_end = tmin<int64_t>(N, int64_t(cta + 1) * pl.rows_per_cta);
  auto blk_base = [&](int j) -> int64_t { return int64_t(cta) * pl.rows_per_cta + int64_t(g0 + j) * BR; };
  auto blk_end = [&](int j) -> int64_t { return tmin<int64_t>(cta_end, blk_base(j) + BR); };
  bool bad_x = false;
  const bool plane = tid < kGR * p;
  const int prow = tid / p, pdim = tid - (tid / p) * p;
  struct Pre {
    double x[PR], y[PR];
  };
  // pipelined launch: block j's rows may only be read once its sub-range's ready word is set.
  // The look-ahead load probes the word; if it is not set yet the load is deferred (pend = j)
  // and done, waiting, right before block j is produced -- never stalling the contraction of
  // the block already staged.
  int seen = k0 - 1;  // last sub-range whose ready word this thread has observed
  int pend = -1;
  auto load_pre = [&](int j, Pre& pr, bool block = false) {
    if (pl.ready && plane) {
      int k = k0;
      while (k + 1 < k1 && g0 + j >= sb(k + 1)) ++k;
      if (k > seen) {
        if (block) {
          wait_ready(pl.ready + k, flags);
        } else {
          unsigned v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(pl.ready + k) : "memory");
          if (!v) {
            pend = j;
            return;
          }
        }
        seen = k;
      }
    }
#pragma unroll
    for (int t = 0; t < PR; ++t) {
      const int64_t r = blk_base(j) + prow + t * kGR;
      const bool ok = plane && r < blk_end(j);
      pr.x[t] = ok ? X[r * p + pdim] : 0.0;
      pr.y[t] = (ok && y != nullptr && pdim == p - 1) ? y[r] : c;
    }
  };
  auto produce = [&](const Pre& pr, int j, double* slab) {
    if (!plane) return;
    double rr[PR];
    int dd[PR];
    double *ophi[PR], *og[PR];
    bool valid[PR];
    // the split Gram reads phi of the last dimension only as r*phi: those tasks write r*phi into
    // the rphi slot and no bare phi, the others phi (scale 1) -- 29 stores per task at C3
    const bool last = pdim == p - 1;
#pragma unroll
    for (int t = 0; t < PR; ++t) {
      double* row = slab + (prow + t * kGR) * rl.bw;
      valid[t] = blk_base(j) + prow + t * kGR < blk_end(j);
      if (valid[t]) bad_x |= not_finite(pr.x[t]);
      rr[t] = last ? __dsub_rn(pr.y[t], c) : 1.0;  // r = y - c (posterior.py:229)
      dd[t] = pdim;
      ophi[t] = last ? row + rl.rpoff : row + rl.poff + pdim * M;
      og[t] = row + rl.goff + pdim * L;
      if (pdim == 0) {
        row[rl.one] = 1.0;
        row[rl.zero] = 0.0;
      }
    }
    eval_phi_g_dim_uT<PR>(pr.x, rr, b, dd, pl.hc, ophi, og);  // padding rows: x = 0, then zeroed
#pragma unroll
    for (int t = 0; t < PR; ++t) {
      if (valid[t]) continue;
      for (int k = 0; k < M; ++k) ophi[t][k] = 0.0;
      for (int k = 0; k < L; ++k) og[t][k] = 0.0;
    }
  };
  __syncthreads();
  Pre pre;
  if constexpr (NSLAB == 2) {
    if (nblk > 0) {
      load_pre(0, pre, true);
      produce(pre, 0, slabs);
    }
    if (nblk > 1) load_pre(1, pre);
  } else {
    if (nblk > 0) load_pre(0, pre, true);
  }

  // A-operand offsets of an m-fragment: 2 factors; invalid columns -> (0, 1)
  const int col = lane >> 2;
  auto offs2 = [&](int m, int nvalid, int o0, int o1, int (&off)[2]) {
    if (m < nvalid) {
      off[0] = o0;
      off[1] = o1;
    } else {
      off[0] = rl.zero;
      off[1] = rl.one;
    }
  };
  const int slot = pl.wslot[warp];
  const bool role1 = slot < pl.W1;
  const int wi = role1 ? slot : slot - pl.W1, WR = role1 ? pl.W1 : kGramW - pl.W1;
  constexpr int NJ = (JK1 + JT1A) > (JK2 + JT2 + JT1B) ? (JK1 + JT1A) : (JK2 + JT2 + JT1B);
  constexpr int NACC = (2 * JK1 + JT1A) > (3 * JK2 + 2 * JT2 + JT1B) ? (2 * JK1 + JT1A) : (3 * JK2 + 2 * JT2 + JT1B);
  int offA[NJ][2], offB[5];
  int fragOf[NACC];  // partial fragment index of each accumulator (-1: dummy)
#pragma unroll
  for (int q = 0; q < NACC; ++q) fragOf[q] = -1;
  if (role1) {
#pragma unroll
    for (int j = 0; j < JK1; ++j) {
      const int mf = wi + WR * j, m = mf * 8 + col;
      offs2(m, L * L, rl.goff + m / L, rl.goff + L + m % L, offA[j]);
#pragma unroll
      for (int nf = 0; nf < 2; ++nf) fragOf[2 * j + nf] = mf < pl.kmf1 ? mf * 2 + nf : -1;
    }
#pragma unroll
    for (int j = 0; j < JT1A; ++j) {
      const int mf = wi + WR * j, m = mf * 8 + col;
      offs2(m, M * M, rl.poff + m / M, rl.poff + M + m % M, offA[JK1 + j]);
      fragOf[2 * JK1 + j] = mf < pl.tmf1 ? pl.baseT1 + mf : -1;
    }
    offB[0] = rl.goff + 2 * L + col;      // g2[0, 8)
    offB[1] = rl.goff + 2 * L + 8 + col;  // g2[8, 16)
    offB[2] = rl.rpoff + col;             // r phi2[0, 8)
  } else {
#pragma unroll
    for (int j = 0; j < JK2; ++j) {
      const int mf = wi + WR * j, m = mf * 8 + col;
      offs2(m, L * pl.R, rl.goff + m / pl.R, rl.goff + 2 * L + 16 + m % pl.R, offA[j]);
#pragma unroll
      for (int nf = 0; nf < 3; ++nf) fragOf[3 * j + nf] = mf < pl.kmf2 ? pl.baseK2 + mf * 3 + nf : -1;
    }
#pragma unroll
    for (int j = 0; j < JT2; ++j) {
      const int mf = wi + WR * j, m = mf * 8 + col;
      offs2(m, M * pl.R2, rl.poff + m / pl.R2, rl.rpoff + 8 + m % pl.R2, offA[JK2 + j]);
#pragma unroll
      for (int nf = 0; nf < 2; ++nf) fragOf[3 * JK2 + 2 * j + nf] = mf < pl.tmf2 ? pl.baseT2 + mf * 2 + nf : -1;
    }
#pragma unroll
    for (int j = 0; j < JT1B; ++j) {
      const int mf = pl.W1 * JT1A + wi + WR * j, m = mf * 8 + col;
      offs2(m, M * M, rl.poff + m / M, rl.poff + M + m % M, offA[JK2 + JT2 + j]);
      fragOf[3 * JK2 + 2 * JT2 + j] = mf < pl.tmf1 ? pl.baseT1 + mf : -1;
    }
#pragma unroll
    for (int nf = 0; nf < 3; ++nf) offB[nf] = nf * 8 + col < L ? rl.goff + L + nf * 8 + col : rl.zero;  // g1
#pragma unroll
    for (int nf = 0; nf < 2; ++nf) offB[3 + nf] = nf * 8 + col < M ? rl.poff + M + nf * 8 + col : rl.zero;  // phi1
  }
  if (role1) offB[3] = offB[4] = rl.zero;
  double acc[NACC][2];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc[q][0] = acc[q][1] = 0.0;
  __syncthreads();

  // one straight-line k-step per warp class, the class branch hoisted out of the k-loop below (a
  // branch inside every k-step kept the scheduler from overlapping k-step i + 1's loads with
  // k-step i's DMMAs).  Classes: role 1 with NK1 K1 m-fragments (+ JT1A T1), role 2 with JK2 K2,
  // NT2 T2 and NT1B T1 m-fragments.  At C3 the slots past the last fragment (9 of 144 DMMA per
  // k-step) belong to warps of the reduced classes, which skip them at no per-k-step cost.
  auto kstep1 = [&](const double* cur, int i, auto nk1) {
    constexpr int NK1 = decltype(nk1)::value;
    const double* row = cur + (i * 4 + (lane & 3)) * SBW;
    const double b0 = row[offB[0]], b1 = row[offB[1]], bt = row[offB[2]];
#pragma unroll
    for (int j = 0; j < NK1; ++j) {
      const double a = __dmul_rn(row[offA[j][0]], row[offA[j][1]]);
      dmma_8x8x4(acc[2 * j][0], acc[2 * j][1], a, b0);
      dmma_8x8x4(acc[2 * j + 1][0], acc[2 * j + 1][1], a, b1);
    }
#pragma unroll
    for (int j = 0; j < JT1A; ++j) {
      const double a = __dmul_rn(row[offA[JK1 + j][0]], row[offA[JK1 + j][1]]);
      dmma_8x8x4(acc[2 * JK1 + j][0], acc[2 * JK1 + j][1], a, bt);
    }
  };
  auto kstep2 = [&](const double* cur, int i, auto nt2, auto nt1b) {
    constexpr int NT2 = decltype(nt2)::value, NT1B = decltype(nt1b)::value;
    const double* row = cur + (i * 4 + (lane & 3)) * SBW;
    const double b0 = row[offB[0]], b1 = row[offB[1]], b2 = row[offB[2]];
#pragma unroll
    for (int j = 0; j < JK2; ++j) {
      const double a = __dmul_rn(row[offA[j][0]], row[offA[j][1]]);
      dmma_8x8x4(acc[3 * j][0], acc[3 * j][1], a, b0);
      dmma_8x8x4(acc[3 * j + 1][0], acc[3 * j + 1][1], a, b1);
      dmma_8x8x4(acc[3 * j + 2][0], acc[3 * j + 2][1], a, b2);
    }
    if constexpr (NT2 > 0) {
      const double p0 = row[offB[3]], p1 = row[offB[4]];
#pragma unroll
      for (int j = 0; j < NT2; ++j) {
        const double a = __dmul_rn(row[offA[JK2 + j][0]], row[offA[JK2 + j][1]]);
        dmma_8x8x4(acc[3 * JK2 + 2 * j][0], acc[3 * JK2 + 2 * j][1], a, p0);
        dmma_8x8x4(acc[3 * JK2 + 2 * j + 1][0], acc[3 * JK2 + 2 * j + 1][1], a, p1);
      }
    }
    if constexpr (NT1B > 0) {
      const double bt = row[rl.rpoff + col];
#pragma unroll
      for (int j = 0; j < NT1B; ++j) {
        const double a = __dmul_rn(row[offA[JK2 + JT2 + j][0]], row[offA[JK2 + JT2 + j][1]]);
        dmma_8x8x4(acc[3 * JK2 + 2 * JT2 + j][0], acc[3 * JK2 + 2 * JT2 + j][1], a, bt);
      }
    }
  };
  // this warp's class from its valid slots (prefixes): 0 role 1 full, 1 role 1 with JK1 - 1 K1
  // fragments, 2 role 2 full, 3 role 2 without its T1B fragment, 4 without T2 and T1B; any other
  // pattern runs the full class of its role (dummy slots compute discarded fragments)
  int cls;
  {
    int nk = 0, nt = 0, nb = 0;
    if (role1) {
#pragma unroll
      for (int j = 0; j < JK1; ++j) nk += fragOf[2 * j] >= 0;
#pragma unroll
      for (int j = 0; j < JT1A; ++j) nt += fragOf[2 * JK1 + j] >= 0;
      cls = (nk == JK1 - 1 && nt == JT1A) ? 1 : 0;
    } else {
#pragma unroll
      for (int j = 0; j < JK2; ++j) nk += fragOf[3 * j] >= 0;
#pragma unroll
      for (int j = 0; j < JT2; ++j) nt += fragOf[3 * JK2 + 2 * j] >= 0;
#pragma unroll
      for (int j = 0; j < JT1B; ++j) nb += fragOf[3 * JK2 + 2 * JT2 + j] >= 0;
      cls = (nk == JK2 && nt == JT2 && nb == 0) ? 3 : (nk == JK2 && nt == 0 && nb == 0) ? 4 : 2;
    }
  }
  using I0 = std::integral_constant<int, 0>;
  using IK1 = std::integral_constant<int, JK1>;
  using IK1m = std::integral_constant<int, (JK1 > 0 ? JK1 - 1 : 0)>;
  using IT2 = std::integral_constant<int, JT2>;
  using IT1B = std::integral_constant<int, JT1B>;
  auto kloop = [&](const double* cur, int nks, auto body) {
    if (nks == BR / 4) {
#pragma unroll kGramUnroll
      for (int i = 0; i < BR / 4; ++i) body(cur, i);
    } else {
      for (int i = 0; i < nks; ++i) body(cur, i);
    }
  };
  auto contract_block = [&](const double* cur, int nks) {
    switch (cls) {
      case 1: kloop(cur, nks, [&](const double* c, int i) { kstep1(c, i, IK1m{}); }); break;
      case 2: kloop(cur, nks, [&](const double* c, int i) { kstep2(c, i, IT2{}, IT1B{}); }); break;
      case 3: kloop(cur, nks, [&](const double* c, int i) { kstep2(c, i, IT2{}, I0{}); }); break;
      case 4: kloop(cur, nks, [&](const double* c, int i) { kstep2(c, i, I0{}, I0{}); }); break;
      default: kloop(cur, nks, [&](const double* c, int i) { kstep1(c, i, IK1{}); }); break;
    }
  };
  auto flush = [&](int k) {
    double* out = ws + (pl.once ? int64_t(cta) : int64_t(cta) * pl.S + k) * pl.plen;
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      if (fragOf[q] >= 0)
        *reinterpret_cast<double2*>(out + int64_t(fragOf[q]) * 64 + 2 * lane) = make_double2(acc[q][0], acc[q][1]);
      acc[q][0] = acc[q][1] = 0.0;
    }
  };
#ifdef FAGP_GRAM_PROFILE
  long long tp[4] = {0, 0, 0, 0};  // kloop, produce, flush, barrier (clock64 cycles)
#define SPROF(i, stmt)              \
  {                                 \
    const long long t_ = clock64(); \
    stmt;                           \
    tp[i] += clock64() - t_;        \
  }
#else
#define SPROF(i, stmt) stmt;
#endif
  for (int n = 0; n < nblk; ++n) {
    const double* cur;
    if constexpr (NSLAB == 2) {
      cur = slabs + (n & 1) * (BR * rl.bw);
      if (n + 1 < nblk) {
        if (pend == n + 1) {
          load_pre(n + 1, pre, true);
          pend = -1;
        }
        produce(pre, n + 1, slabs + ((n + 1) & 1) * (BR * rl.bw));
        if (n + 2 < nblk) load_pre(n + 2, pre);
      }
    } else {
      cur = slabs;
      SPROF(1, if (pend == n) {
        load_pre(n, pre, true);
        pend = -1;
      } produce(pre, n, slabs);
      if (n + 1 < nblk) load_pre(n + 1, pre))
      SPROF(3, __syncthreads())
    }
    // k-steps holding a valid row (a CTA's last block may be partial; padding rows are zero)
    const int nks = int(tmax<int64_t>(0, blk_end(n) - blk_base(n)) + 3) / 4;
    SPROF(0, contract_block(cur, nks))
    if (pl.once) {
      SPROF(2, if (n + 1 == nblk) flush(0))
    } else {
      SPROF(2, for (int k = k0; k < k1; ++k) if (g0 + n + 1 == sb(k + 1)) flush(k))
    }
    SPROF(3, __syncthreads())
  }
#ifdef FAGP_GRAM_PROFILE
  if (lane == 0)
    for (int i = 0; i < 4; ++i) atomicAdd(reinterpret_cast<unsigned long long*>(&g_gram_prof[i]), (unsigned long long)tp[i]);
#endif
#undef SPROF
  if (bad_x) raise_flag(flags, FAGP_FLAG_X_NONFINITE);
}

// out[e] = sum over the partials (fixed order: deterministic) of entry e of [K | t], read from
// the fragment-major partial layout; non-finite -> PHI flag
// partial_sum: PSE entries per CTA x PSG partial groups, 512 threads.  Many groups for the C2-size
// plans (~2400 partials per entry); few for the one-launch plans (C3: 148), whose CTAs then cover 64
// entries and the final group sum is 8 adds instead of a 64-long chain
constexpr int kPSE = 8, kPSG = 64;
template <int PSE, int PSG>
__global__ void __launch_bounds__(PSE * PSG) partial_sum_kernel(const double* __restrict__ ws, const GPlan pl,
                                                                double* __restrict__ out, uint32_t* flags) {
  constexpr int kPSE = PSE, kPSG = PSG;
  __shared__ double red[kPSG][kPSE];
  const int NFK = int(ceil_div(pl.KB, 8)), NFT = int(ceil_div(pl.TB, 8));
  const int grp = int(threadIdx.x) / kPSE, el = int(threadIdx.x) % kPSE;
  const int64_t e = int64_t(blockIdx.x) * kPSE + el;
  double s = 0.0;
  if (e < pl.len) {
    int64_t m, n, frag;
    if (pl.split) {
      if (e < pl.Klen) {
        const int64_t ka = e / pl.L, k2 = e - ka * pl.L;
        if (k2 < 16) {
          m = ka;
          n = k2;
          frag = (m >> 3) * 2 + (n >> 3);
        } else {
          m = (ka / pl.L) * pl.R + (k2 - 16);
          n = ka % pl.L;
          frag = pl.baseK2 + (m >> 3) * 3 + (n >> 3);
        }
      } else {
        const int64_t q = e - pl.Klen, aa = q / pl.M, a2 = q - aa * pl.M;
        if (a2 < 8) {
          m = aa;
          n = a2;
          frag = pl.baseT1 + (m >> 3);
        } else {
          m = (aa / pl.M) * pl.R2 + (a2 - 8);
          n = aa % pl.M;
          frag = pl.baseT2 + (m >> 3) * 2 + (n >> 3);
        }
      }
    } else if (e < pl.Klen) {
      m = e / pl.KB;
      n = e - m * pl.KB;
      frag = (m >> 3) * NFK + (n >> 3);
    } else {
      m = (e - pl.Klen) / pl.TB;
      n = (e - pl.Klen) - m * pl.TB;
      frag = int64_t(pl.kmf) * NFK + (m >> 3) * NFT + (n >> 3);
    }
    const int64_t idx = frag * 64 + ((m & 7) * 4 + ((n & 7) >> 1)) * 2 + (n & 1);
    // group grp sums partials [q0, q1) in order (loads batched 8 at a time: latency-bound
    // otherwise); the kPSG group sums are then added in group order -- a fixed order
    const int q0 = int(int64_t(grp) * pl.nparts / kPSG), q1 = int(int64_t(grp + 1) * pl.nparts / kPSG);
    int q = q0;
    for (; q + 8 <= q1; q += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ws[int64_t(q + u) * pl.plen + idx];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; q < q1; ++q) s += ws[int64_t(q) * pl.plen + idx];
  }
  red[grp][el] = s;
  if (pl.ready && blockIdx.x == 0 && threadIdx.x < unsigned(pl.S))
    const_cast<unsigned*>(pl.ready)[threadIdx.x] = 0u;  // re-arm for the next pipelined call
  __syncthreads();
  if (grp == 0 && e < pl.len) {
    double t = red[0][el];
#pragma unroll
    for (int g = 1; g < kPSG; ++g) t += red[g][el];
    out[e] = t;
    if (not_finite(t)) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
  }
}

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// (JK, JT) warp shapes compiled for the fused Gram
constexpr int kGramShapes[][2] = {{1, 1}, {3, 1}, {4, 2}};

// Plan for N rows; false when the shape needs the tiled table path.

// Useful DMMA per k-step of each split slot (template split <4, 1, 2, 1, 1>; a slot's skipped
// fragments are those of the reduced classes in fused_gram_split_kernel, others count in full),
// then slots placed on the 4 SM sub-partitions largest first, each onto the least-loaded
// sub-partition with a free warp slot (4 warps each).
static void split_warp_map(GPlan& pl) {
  constexpr int JK1 = 4, JT1A = 1, JK2 = 2, JT2 = 1, JT1B = 1;
  const int W2 = kGramW - pl.W1;
  int load[kGramW];
  for (int sl = 0; sl < kGramW; ++sl) {
    int nk = 0, nt = 0, nb = 0;
    if (sl < pl.W1) {
      for (int j = 0; j < JK1; ++j) nk += sl + pl.W1 * j < pl.kmf1;
      for (int j = 0; j < JT1A; ++j) nt += sl + pl.W1 * j < pl.tmf1;
      load[sl] = (nk == JK1 - 1 && nt == JT1A) ? 2 * (JK1 - 1) + JT1A : 2 * JK1 + JT1A;
    } else {
      const int wi = sl - pl.W1;
      for (int j = 0; j < JK2; ++j) nk += wi + W2 * j < pl.kmf2;
      for (int j = 0; j < JT2; ++j) nt += wi + W2 * j < pl.tmf2;
      for (int j = 0; j < JT1B; ++j) nb += pl.W1 * JT1A + wi + W2 * j < pl.tmf1;
      load[sl] = (nk == JK2 && nt == JT2 && nb == 0)  ? 3 * JK2 + 2 * JT2
                 : (nk == JK2 && nt == 0 && nb == 0) ? 3 * JK2
                                                      : 3 * JK2 + 2 * JT2 + JT1B;
    }
  }
  int order[kGramW];
  for (int sl = 0; sl < kGramW; ++sl) order[sl] = sl;
  std::stable_sort(order, order + kGramW, [&](int a, int b) { return load[a] > load[b]; });
  int sp_load[4] = {0, 0, 0, 0}, sp_used[4] = {0, 0, 0, 0};
  for (int k = 0; k < kGramW; ++k) {
    int best = -1;
    for (int q = 0; q < 4; ++q)
      if (sp_used[q] < kGramW / 4 && (best < 0 || sp_load[q] < sp_load[best])) best = q;
    pl.wslot[best + 4 * sp_used[best]] = static_cast<unsigned char>(order[k]);
    sp_load[best] += load[order[k]];
    ++sp_used[best];
  }
}

static bool make_gplan(int64_t N, int p, int M, GPlan& pl) {
  std::memset(&pl, 0, sizeof(pl));
  if (!modal_on(p, M) || p > kMaxF || M > 12 || kGR * p > kGramNT) return false;
  pl.p = p;
  pl.M = M;
  pl.L = modal_L(M);
  pl.LC = (pl.L + 1) & ~1;
  pl.KA = int(ipow(pl.L, p - 1));
  pl.KB = pl.L;
  pl.TA = int(ipow(M, p - 1));
  pl.TB = M;
  pl.kmf = int(ceil_div(pl.KA, 8));
  pl.tmf = int(ceil_div(pl.TA, 8));
  const int NFK = int(ceil_div(pl.KB, 8)), NFT = int(ceil_div(pl.TB, 8));
  // row groups and warp shape with the smallest per-block critical path:
  // ceil(16 / G) k-steps x (JK NFK + JT NFT) DMMAs per warp
  int best = -1;
  for (int G = 1; G <= kGramW; G *= 2) {
    const int WG = kGramW / G;
    for (const auto& sh : kGramShapes) {
      if (WG * sh[0] < pl.kmf || WG * sh[1] < pl.tmf) continue;
      const int cost = ((kGR / 4 + G - 1) / G) * (sh[0] * NFK + sh[1] * NFT);
      if (best < 0 || cost < best) {
        best = cost;
        pl.G = G;
        pl.WG = WG;
        pl.JK = sh[0];
        pl.JT = sh[1];
      }
    }
  }
  if (best < 0) return false;
  pl.Klen = int64_t(pl.KA) * pl.KB;
  pl.len = pl.Klen + int64_t(pl.TA) * pl.TB;
  pl.plen = (int64_t(pl.kmf) * NFK + int64_t(pl.tmf) * NFT) * 64;
  const RowLayout rl = row_layout(p, M);
  const size_t smem = (size_t(2) * pl.LC + size_t(2) * kGR * rl.bw) * sizeof(double);
  if (smem > 225 * 1024) return false;
  // split layout (fused_gram_split_kernel): p = 3, M = 10 (the BASELINE C3 shape)
  const char* se = getenv("FAGP_GRAM_SPLIT");
  const bool split = p == 3 && M == 10 && !(se && se[0] == '0') && row_layout(3, 10).bw == kSplitGramBW;
  pl.br = kGR;
  if (split) {
    const char* be = getenv("FAGP_GRAM_BR");  // tuning knob: 128 = double-buffered 128-row slabs
    pl.br = (be && atoi(be) == kGR) ? kGR : kSR;
    if (size_t(pl.br) * rl.bw * sizeof(double) > 225 * 1024) pl.br = kGR;
  }
  // rows: one CTA per SM, each a contiguous range of S sub-ranges (S = 4 / 8 once every
  // sub-range holds at least 2 blocks), so a host pipeline can upload sub-range k + 1 of every
  // CTA while the Gram contracts sub-range k -- the first chunk, the only upload not hidden
  // behind the contraction, is 1/S of the rows
  // The rows are cut evenly (in whole k-steps of 4) over the CTAs, so a CTA's last block may be
  // partial (the split kernel skips its empty k-steps): the makespan is N / grid rows, not a
  // whole number of blocks.
  const int64_t blocks = tmax<int64_t>(1, ceil_div(N, pl.br));
  pl.grid = int(tmin<int64_t>(num_sms(), blocks));
  pl.rows_per_cta = tmax<int64_t>(4, ceil_div(ceil_div(tmax<int64_t>(N, 1), pl.grid), 4) * 4);
  const int64_t bpc = ceil_div(pl.rows_per_cta, pl.br);  // blocks per CTA
  pl.bpc = int(bpc);
  pl.S = bpc >= 16 ? 8 : bpc >= 8 ? 4 : 1;
  if (const char* e = getenv("FAGP_GRAM_SUBRANGES")) pl.S = tmax(1, tmin<int>(int(bpc), atoi(e)));  // tuning knob
  pl.S = tmin(pl.S, 64);  // ready words re-armed by one partial_sum block (and a sane chunk count)
  pl.grid = int(tmax<int64_t>(1, ceil_div(tmax<int64_t>(N, 1), pl.rows_per_cta)));
  pl.nparts = pl.grid * pl.S * pl.G;
  pl.hc = herm_coef_host();
  if (split) {
    pl.split = 1;
    pl.W1 = 12;
    pl.R = pl.L - 16;
    pl.R2 = M - 8;
    pl.kmf1 = int(ceil_div(int64_t(pl.L) * pl.L, 8));
    pl.kmf2 = int(ceil_div(int64_t(pl.L) * pl.R, 8));
    pl.tmf1 = int(ceil_div(int64_t(M) * M, 8));
    pl.tmf2 = int(ceil_div(int64_t(M) * pl.R2, 8));
    pl.baseK2 = pl.kmf1 * 2;
    pl.baseT1 = pl.baseK2 + pl.kmf2 * 3;
    pl.baseT2 = pl.baseT1 + pl.tmf1;
    pl.plen = int64_t(pl.baseT2 + pl.tmf2 * 2) * 64;
    pl.G = 1;
    pl.WG = kGramW;
    pl.nparts = pl.grid * pl.S;
    split_warp_map(pl);
  }
  return true;
}

static size_t gram_smem(const GPlan& pl) {
  if (pl.split) return size_t(pl.br == kGR ? 2 : 1) * pl.br * row_layout(pl.p, pl.M).bw * sizeof(double);
  return (size_t(2) * pl.LC + size_t(2) * kGR * row_layout(pl.p, pl.M).bw) * sizeof(double);
}

template <int FA, int NFK, int NFT>
static int launch_gram_shape(const double* X, const double* y, double c, int64_t N, const fagp_basis* b,
                             const GPlan& pl, int k0, int k1, double* ws, uint32_t* flags, cudaStream_t s) {
  const size_t smem = gram_smem(pl);
  auto go = [&](auto kern) -> int {
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<pl.grid, kGramNT, smem, s>>>(X, y, c, N, view(b), pl, k0, k1, ws, flags);
    return FAGP_OK;
  };
  if (pl.JK == 1 && pl.JT == 1) return go(fused_gram_kernel<FA, NFK, NFT, 1, 1>);
  if (pl.JK == 3 && pl.JT == 1) return go(fused_gram_kernel<FA, NFK, NFT, 3, 1>);
  if (pl.JK == 4 && pl.JT == 2) return go(fused_gram_kernel<FA, NFK, NFT, 4, 2>);
  return FAGP_EUNSUPPORTED;
}

template <int FA>
static int launch_gram_fa(const double* X, const double* y, double c, int64_t N, const fagp_basis* b,
                          const GPlan& pl, int k0, int k1, double* ws, uint32_t* flags, cudaStream_t s) {
  // (n-frags of K, n-frags of t) from M: L = 2M - 1 <= 8 NFK, M <= 8 NFT
  if (pl.M <= 4) return launch_gram_shape<FA, 1, 1>(X, y, c, N, b, pl, k0, k1, ws, flags, s);
  if (pl.M <= 8) return launch_gram_shape<FA, 2, 1>(X, y, c, N, b, pl, k0, k1, ws, flags, s);
  return launch_gram_shape<FA, 3, 2>(X, y, c, N, b, pl, k0, k1, ws, flags, s);
}

bool gram_eligible(int64_t N, int p, int M) {
  GPlan pl;
  return make_gplan(N, p, M, pl);
}

size_t gram_workspace(int64_t N, int p, int M) {
  GPlan pl;
  if (!make_gplan(N, p, M, pl)) return 0;
  return size_t(pl.nparts) * size_t(pl.plen) * sizeof(double);
}

int gram_chunks(int64_t N, int p, int M) {
  GPlan pl;
  return make_gplan(N, p, M, pl) ? pl.S : 1;
}

// H2D of the rows chunk k reads: sub-range k of every CTA (one 2-D copy for the CTAs whose
// sub-range lies inside [0, N), one plain copy for the CTA that holds row N - 1)
int upload_chunk(const double* Xh, const double* yh, int64_t N, int p, int M, int k, double* Xd, double* yd,
                 cudaStream_t s) {
  GPlan pl;
  if (!make_gplan(N, p, M, pl)) {
    if (k != 0) return FAGP_EINVAL;
    if (N > 0) {
      FAGP_CUDA_TRY(cudaMemcpyAsync(Xd, Xh, size_t(N) * p * sizeof(double), cudaMemcpyHostToDevice, s));
      if (yh && yd) FAGP_CUDA_TRY(cudaMemcpyAsync(yd, yh, size_t(N) * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    return FAGP_OK;
  }
  if (k < 0 || k >= pl.S) return FAGP_EINVAL;
  const int64_t bpc = pl.bpc;
  const int64_t off = (int64_t(k) * bpc / pl.S) * pl.br;
  const int64_t sub_rows = tmin<int64_t>((int64_t(k + 1) * bpc / pl.S) * pl.br, pl.rows_per_cta) - off;
  // CTAs c with c rpc + off + sub_rows <= N
  const int64_t head = N - off - sub_rows;
  const int64_t full = head < 0 ? 0 : tmin<int64_t>(pl.grid, head / pl.rows_per_cta + 1);
  if (full > 0) {
    const size_t pitch = size_t(pl.rows_per_cta) * sizeof(double);
    FAGP_CUDA_TRY(cudaMemcpy2DAsync(Xd + off * p, pitch * p, Xh + off * p, pitch * p, size_t(sub_rows) * p * 8,
                                    size_t(full), cudaMemcpyHostToDevice, s));
    if (yh && yd)
      FAGP_CUDA_TRY(cudaMemcpy2DAsync(yd + off, pitch, yh + off, pitch, size_t(sub_rows) * 8, size_t(full),
                                      cudaMemcpyHostToDevice, s));
  }
  if (full < pl.grid) {
    const int64_t a = full * pl.rows_per_cta + off, e = tmin<int64_t>(N, a + sub_rows);
    if (e > a) {
      FAGP_CUDA_TRY(cudaMemcpyAsync(Xd + a * p, Xh + a * p, size_t(e - a) * p * 8, cudaMemcpyHostToDevice, s));
      if (yh && yd) FAGP_CUDA_TRY(cudaMemcpyAsync(yd + a, yh + a, size_t(e - a) * 8, cudaMemcpyHostToDevice, s));
    }
  }
  return FAGP_OK;
}

// host staging of the rows chunk k reads (the rows upload_chunk copies, the same geometry) from a
// caller's pageable arrays into pinned buffers laid out like the device ones
int stage_chunk(const double* Xsrc, const double* ysrc, int64_t N, int p, int M, int k, double* Xdst, double* ydst,
                int threads) {
  GPlan pl;
  if (!make_gplan(N, p, M, pl)) {
    if (k != 0) return FAGP_EINVAL;
    int rc = fagp_host_copy(Xdst, Xsrc, size_t(N) * p * sizeof(double), threads);
    if (rc == FAGP_OK && ysrc && ydst) rc = fagp_host_copy(ydst, ysrc, size_t(N) * sizeof(double), threads);
    return rc;
  }
  if (k < 0 || k >= pl.S) return FAGP_EINVAL;
  const int64_t bpc = pl.bpc;
  const int64_t off = (int64_t(k) * bpc / pl.S) * pl.br;
  const int64_t sub_rows = tmin<int64_t>((int64_t(k + 1) * bpc / pl.S) * pl.br, pl.rows_per_cta) - off;
  const int64_t head = N - off - sub_rows;
  const int64_t full = head < 0 ? 0 : tmin<int64_t>(pl.grid, head / pl.rows_per_cta + 1);
  int rc = FAGP_OK;
  if (full > 0) {
    const size_t pitch = size_t(pl.rows_per_cta) * sizeof(double);
    rc = fagp_host_copy_2d(Xdst + off * p, pitch * p, Xsrc + off * p, pitch * p, size_t(sub_rows) * p * 8, size_t(full),
                           threads);
    if (rc == FAGP_OK && ysrc && ydst)
      rc = fagp_host_copy_2d(ydst + off, pitch, ysrc + off, pitch, size_t(sub_rows) * 8, size_t(full), threads);
  }
  if (rc == FAGP_OK && full < pl.grid) {
    const int64_t a = full * pl.rows_per_cta + off, e = tmin<int64_t>(N, a + sub_rows);
    if (e > a) {
      rc = fagp_host_copy(Xdst + a * p, Xsrc + a * p, size_t(e - a) * p * 8, threads);
      if (rc == FAGP_OK && ysrc && ydst) rc = fagp_host_copy(ydst + a, ysrc + a, size_t(e - a) * 8, threads);
    }
  }
  return rc;
}

// chunks [k0, k1) of the plan; the last chunk also sums the partials into `out`
int gram(const double* X, const double* y, double c, int64_t N, const fagp_basis* b, int k0, int k1, double* out,
         void* ws, size_t ws_bytes, uint32_t* flags, cudaStream_t s, const unsigned* ready) {
  GPlan pl;
  if (!make_gplan(N, b->p, b->M, pl)) return FAGP_EUNSUPPORTED;
  if (k0 < 0 || k1 > pl.S || k0 >= k1) return FAGP_EINVAL;
  // one launch over every sub-range: one partial per CTA (and row group)
  pl.once = (k0 == 0 && k1 == pl.S) ? 1 : 0;
  const size_t parts = pl.once ? size_t(pl.grid) * pl.G : size_t(pl.nparts);
  if (ws == nullptr || ws_bytes < parts * size_t(pl.plen) * sizeof(double)) return FAGP_EWORKSPACE;
  pl.ready = pl.once ? ready : nullptr;
  if (pl.ready) {
    // load partial_sum_kernel now: with lazy module loading its first launch (queued behind a
    // Gram that is still waiting for its input signals) could block this thread until the
    // device is idle -- before the caller has issued the signals
    static bool loaded = false;
    if (!loaded) {
      cudaFuncAttributes fa;
      FAGP_CUDA_TRY(cudaFuncGetAttributes(&fa, partial_sum_kernel<64, 8>));
      FAGP_CUDA_TRY(cudaFuncGetAttributes(&fa, partial_sum_kernel<kPSE, kPSG>));
      loaded = true;
    }
  }
  double* w = static_cast<double*>(ws);
  int rc;
  if (pl.split) {
    const size_t smem = gram_smem(pl);
    auto kern = pl.br == kGR ? fused_gram_split_kernel<4, 1, 2, 1, 1, kGR> : fused_gram_split_kernel<4, 1, 2, 1, 1, kSR>;
    FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<pl.grid, kGramNT, smem, s>>>(X, y, c, N, view(b), pl, k0, k1, w, flags);
    rc = FAGP_OK;
  } else switch (b->p - 1) {
    case 1: rc = launch_gram_fa<1>(X, y, c, N, b, pl, k0, k1, w, flags, s); break;
    case 2: rc = launch_gram_fa<2>(X, y, c, N, b, pl, k0, k1, w, flags, s); break;
    case 3: rc = launch_gram_fa<3>(X, y, c, N, b, pl, k0, k1, w, flags, s); break;
    default: rc = FAGP_EUNSUPPORTED;
  }
  if (rc) return rc;
  FAGP_LAUNCH_CHECK();
  if (k1 == pl.S) {
    if (pl.once) pl.nparts = pl.grid * pl.G;
    if (pl.nparts <= 1024)
      partial_sum_kernel<64, 8><<<unsigned(ceil_div(pl.len, 64)), 512, 0, s>>>(w, pl, out, flags);
    else
      partial_sum_kernel<kPSE, kPSG><<<unsigned(ceil_div(pl.len, kPSE)), kPSE * kPSG, 0, s>>>(w, pl, out, flags);
    FAGP_LAUNCH_CHECK();
  }
  return FAGP_OK;
}

// ---------------------------------------------------------------------------------------
// Fused predict (variance + mean).  16 warps = 8 row groups (16 rows = 2 m-fragments) x 2
// K-halves.  Each 128-row block starts with a production phase in which all warps evaluate phi
// and g of the block (one (row, dim) per thread; kept apart from the DMMA phase, where the
// dependent FP64 chains would starve behind the shared pipe -- its cost is one chain latency
// per block, so blocks are as large as shared memory allows: one 128-row slab); then the DMMA
// phase.  The variance and mean epilogues are linear in the GEMM outputs, so every warp
// applies them to its own K-quarter partial (g / phi products gathered from the row slab, 4-lane
// shuffle reduction) and only one scalar per row and quarter meets in shared memory; the
// quarters are summed in fixed order.
constexpr int kPredW = 16;
constexpr int kPredNT = kPredW * 32;  // 512 threads
constexpr int kPMF = 2;               // m-fragments per warp
constexpr int kPR = 128;              // rows per block: 8 row groups of 16 x 2 K-halves
constexpr int kPKS = 2;               // K splits

struct VPlan {
  int p, M, L, LC;
  int pN;                // variance: N side dims [0,pN) (epilogue), K side [pN,p), radix L
  int NR, KR, vks;       // N extent (<= 8 NFV), K extent, k-steps of 4
  int NM, KM, mks;       // mean: N side dim 0 (M), K side dims [1,p) (M^(p-1))
  int64_t KP, NP;        // predict_op layout (modal::Plan): C'' [KP][NP], then w (m)
  int64_t nblocks;
  int grid;
  size_t smem;
  HermCoef hc;           // recurrence coefficients (constant-bank operands)
};

// byte-packed factor offsets of K column kappa (F factors, 8 bits each; offsets < 256)
template <int F>
__device__ __forceinline__ void unpack_off(uint32_t v, int (&off)[F]) {
#pragma unroll
  for (int f = 0; f < F; ++f) off[f] = int((v >> (8 * f)) & 0xffu);
}

// acc[f][nf] += A[rows 8 f + (lane >> 2)][kappa] B[kappa][nu] over the k-steps [k0, k1) of 4 kappa:
// A gathered from the row slab by the packed offsets of kappa = 4 ks + (lane & 3), B from the
// fragment-major operand.  Software-pipelined: the operands of k-step ks + 1 are loaded and
// multiplied in program order before the DMMAs of k-step ks, so they overlap.
template <int F, int NF, int BW = 0>
__device__ __forceinline__ void contract(const double* row0, int bw_rt, const uint32_t* offs, const double* B, int k0,
                                         int k1, int lane, double (&acc)[kPMF][NF][2]) {
  if (k0 >= k1) return;
  const int bw = BW ? BW : bw_rt;  // compile-time row stride where known: immediate load offsets
  auto load = [&](int ks, double (&ao)[kPMF], double (&bo)[NF]) {
    int off[F];
    unpack_off<F>(offs[4 * ks + (lane & 3)], off);
#pragma unroll
    for (int f = 0; f < kPMF; ++f) ao[f] = gather_prod<F>(row0 + 8 * f * bw, off);
#pragma unroll
    for (int nf = 0; nf < NF; ++nf) bo[nf] = B[(ks * NF + nf) * 32 + lane];
  };
  double a[kPMF], bb[NF];
  load(k0, a, bb);
  for (int ks = k0; ks < k1; ++ks) {
    double an[kPMF], bn[NF];
    load(ks + 1 < k1 ? ks + 1 : ks, an, bn);
#pragma unroll
    for (int f = 0; f < kPMF; ++f)
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[f][nf][0], acc[f][nf][1], a[f], bb[nf]);
#pragma unroll
    for (int f = 0; f < kPMF; ++f) a[f] = an[f];
#pragma unroll
    for (int nf = 0; nf < NF; ++nf) bb[nf] = bn[nf];
  }
}

// contract() with compile-time k-step bounds: a plain loop the compiler unrolls and schedules
// itself (loads of later k-steps hoisted over earlier DMMAs), as in the Gram's k-loop.
// UNR: the k-loop unroll.  One lockstep CTA: full (measured: 8 -> 0.750 ms, 4 / 16 -> 0.743, 64 =
// full -> 0.735 at C3).  Two warp groups: 16 -- the groups run different phases at once, so the
// fully unrolled kernel (97 KB of SASS) keeps its production and both contraction halves hot
// together and, behind the Gram's code in the step, runs out of the SM's instruction cache (0.720
// ms in the step, 0.682 alone; unroll 16: 0.682 in the step, profiles/predict_groups_r06.txt)
template <int F, int NF, int BW, int K0, int K1, int UNR>
__device__ __forceinline__ void contract_ct(const double* row0, const uint32_t* offs, const double* B, int lane,
                                            double (&acc)[kPMF][NF][2]) {
#pragma unroll UNR
  for (int ks = K0; ks < K1; ++ks) {
    int off[F];
    unpack_off<F>(offs[4 * ks + (lane & 3)], off);
    double a[kPMF], bb[NF];
#pragma unroll
    for (int f = 0; f < kPMF; ++f) a[f] = gather_prod<F>(row0 + 8 * f * BW, off);
#pragma unroll
    for (int nf = 0; nf < NF; ++nf) bb[nf] = B[(ks * NF + nf) * 32 + lane];
#pragma unroll
    for (int f = 0; f < kPMF; ++f)
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[f][nf][0], acc[f][nf][1], a[f], bb[nf]);
  }
}

#ifdef FAGP_GRAM_PROFILE
__device__ long long g_pred_prof[4];
extern "C" int fagp_debug_pred_profile(long long* out) {  // diagnostics build only
  return cudaMemcpyFromSymbol(out, g_pred_prof, sizeof(g_pred_prof)) == cudaSuccess ? 0 : 5;
}
#endif

template <int FK, int FE, int FKM, int NFV, int NFM>
__global__ void __launch_bounds__(kPredNT, 1)
fused_predict_kernel(const double* __restrict__ Xs, int64_t Ns, BasisView b, const VPlan pl,
                     const double* __restrict__ op, double sigma2, double c, double* __restrict__ mean,
                     double* __restrict__ var, uint32_t* flags) {
  constexpr int P = FK + FE;
  extern __shared__ double sm[];
  const RowLayout rl = row_layout(pl.p, pl.M);
  const bool want_var = var != nullptr;
  double* Bv = sm;                           // [vks][NFV][32]
  double* Bm = Bv + pl.vks * NFV * 32;       // [mks][NFM][32]
  double* red = Bm + pl.mks * NFM * 32;      // [kPKS][kPR][2 (var, mean)]
  double* slab = red + kPKS * kPR * 2;       // [kPR * bw]
  uint32_t* offV = reinterpret_cast<uint32_t*>(slab + kPR * rl.bw);  // [vks * 4]
  uint32_t* offM = offV + pl.vks * 4;                                       // [mks * 4]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = pl.M, L = pl.L;
  const double* w = op + pl.KP * pl.NP;
  // operands, fragment-major: B[ks][nf][lane] = Op[4 ks + (lane & 3)][8 nf + (lane >> 2)]
  if (want_var)
    for (int i = tid; i < pl.vks * NFV * 32; i += kPredNT) {
      const int ln = i & 31, q = i >> 5, nf = q % NFV, ks = q / NFV;
      const int kap = 4 * ks + (ln & 3), nu = 8 * nf + (ln >> 2);
      Bv[i] = (kap < pl.KR && nu < pl.NR) ? op[int64_t(kap) * pl.NP + nu] : 0.0;
    }
  for (int i = tid; i < pl.mks * NFM * 32; i += kPredNT) {
    const int ln = i & 31, q = i >> 5, nf = q % NFM, ks = q / NFM;
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
  bool bad_x = false, bad = false;
  // production: thread t < 128 P evaluates phi and g of row t / P, dimension t % P
  const bool plane = tid < kPR * P;
  const int prow = tid / P, pdim = tid - (tid / P) * P;
  auto load_x = [&](int64_t blk) -> double {
    const int64_t r = blk * kPR + prow;
    return (plane && blk < pl.nblocks && r < Ns) ? Xs[r * P + pdim] : 0.0;
  };
  auto produce = [&](double x, int64_t blk) {
    if (!plane) return;
    double* row = slab + prow * rl.bw;
    if (blk * kPR + prow < Ns) {
      bad_x |= not_finite(x);
      eval_phi_g_dim_u(x, 0.0, b, pdim, pl.hc, row + rl.poff + pdim * M, row + rl.goff + pdim * L, nullptr);
    } else {
      for (int k = 0; k < M; ++k) row[rl.poff + pdim * M + k] = 0.0;
      for (int k = 0; k < L; ++k) row[rl.goff + pdim * L + k] = 0.0;
    }
    if (pdim == 0) {
      row[rl.one] = 1.0;
      row[rl.zero] = 0.0;
    }
  };
  const int64_t blk0 = blockIdx.x, stride = gridDim.x;
  double xn = load_x(blk0);
  // consumer roles: rows [16 mg, 16 mg + 16), K-split kq
  const int mg = warp % (kPredW / kPKS), kq = warp / (kPredW / kPKS);
  const int v0 = kq * pl.vks / kPKS, v1 = (kq + 1) * pl.vks / kPKS;
  const int m0 = kq * pl.mks / kPKS, m1 = (kq + 1) * pl.mks / kPKS;
  // epilogue factor offsets: variance E[i, nu] = prod_{d < pN} g_d; mean phi_0[i, nu]
  int offE[NFV][2][FE], offEm[NFM][2];
#pragma unroll
  for (int nf = 0; nf < NFV; ++nf)
#pragma unroll
    for (int e = 0; e < 2; ++e)
      col_offsets<FE>(nf * 8 + 2 * (lane & 3) + e, pl.NR, rl.goff, 0, pl.pN, pl.L, -1, rl, offE[nf][e]);
#pragma unroll
  for (int nf = 0; nf < NFM; ++nf)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int nu = nf * 8 + 2 * (lane & 3) + e;
      offEm[nf][e] = nu < pl.NM ? rl.poff + nu : rl.zero;
    }
  __syncthreads();

#ifdef FAGP_GRAM_PROFILE
  long long tp[4] = {0, 0, 0, 0};  // produce, contract, epilogue+final, barrier (clock64 cycles)
  long long t_ = clock64();
#define PPROF(i)                    \
  {                                 \
    const long long n_ = clock64(); \
    tp[i] += n_ - t_;               \
    t_ = n_;                        \
  }
#else
#define PPROF(i)
#endif
  for (int64_t blk = blk0; blk < pl.nblocks; blk += stride) {
    // production phase
    produce(xn, blk);
    xn = load_x(blk + stride);
    __syncthreads();
    PPROF(0)
    // DMMA phase
    const double* row0 = slab + (mg * 16 + (lane >> 2)) * rl.bw;  // m-fragment f: + 8 f rows
    double accV[kPMF][NFV][2], accM[kPMF][NFM][2];
#pragma unroll
    for (int f = 0; f < kPMF; ++f) {
#pragma unroll
      for (int nf = 0; nf < NFV; ++nf) accV[f][nf][0] = accV[f][nf][1] = 0.0;
#pragma unroll
      for (int nf = 0; nf < NFM; ++nf) accM[f][nf][0] = accM[f][nf][1] = 0.0;
    }
    if (want_var) contract<FK, NFV>(row0, rl.bw, offV, Bv, v0, v1, lane, accV);
    contract<FKM, NFM>(row0, rl.bw, offM, Bm, m0, m1, lane, accM);
    PPROF(1)
    // this K-split's epilogue contribution per row: sum_nu Y[i, nu] E[i, nu] (var),
    // sum_nu Z[i, nu] phi_0[i, nu] (mean); the 4 lanes of a row hold disjoint columns
#pragma unroll
    for (int f = 0; f < kPMF; ++f) {
      const double* row = row0 + 8 * f * rl.bw;
      double vs = 0.0, ms = 0.0;
#pragma unroll
      for (int nf = 0; nf < NFV; ++nf)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (want_var) vs = fma(accV[f][nf][e], gather_prod<FE>(row, offE[nf][e]), vs);
#pragma unroll
      for (int nf = 0; nf < NFM; ++nf)
#pragma unroll
        for (int e = 0; e < 2; ++e) ms = fma(accM[f][nf][e], row[offEm[nf][e]], ms);
      vs += __shfl_xor_sync(0xffffffffu, vs, 1);
      vs += __shfl_xor_sync(0xffffffffu, vs, 2);
      ms += __shfl_xor_sync(0xffffffffu, ms, 1);
      ms += __shfl_xor_sync(0xffffffffu, ms, 2);
      if ((lane & 3) == 0) {
        const int r = mg * 16 + 8 * f + (lane >> 2);
        red[(kq * kPR + r) * 2 + 0] = vs;
        red[(kq * kPR + r) * 2 + 1] = ms;
      }
    }
    PPROF(2)
    __syncthreads();  // red complete; the slab is free for the next production
    PPROF(3)
    if (tid < kPR) {
      const int64_t row_i = blk * kPR + tid;
      if (row_i < Ns) {
        double vs = red[tid * 2], ms = red[tid * 2 + 1];
#pragma unroll
        for (int q = 1; q < kPKS; ++q) {
          vs += red[(q * kPR + tid) * 2];
          ms += red[(q * kPR + tid) * 2 + 1];
        }
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
    // red is next written after the next block's first barrier, which these threads pass only
    // after finishing here
    PPROF(2)
  }
#ifdef FAGP_GRAM_PROFILE
  if (lane == 0)
    for (int i = 0; i < 4; ++i) atomicAdd(reinterpret_cast<unsigned long long*>(&g_pred_prof[i]), (unsigned long long)tp[i]);
#endif
#undef PPROF
  if (bad_x) raise_flag(flags, FAGP_FLAG_X_NONFINITE);
  if (bad) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
}

// Split-layout fused predict for p = 3, M in [9, 12] (the C3 shape): the ragged last n-fragment of
// the variance (nu = kappa_0 in [16, L)) and of the mean (a_0 in [8, M)) is contracted with the
// roles of dims 0 and 1 swapped, as in fused_gram_split_kernel:
//   var1:  A = g1 g2 (L^2)            x B = C''[.][0, 16)       epilogue g0[nu]
//   var2:  A = (g0[16, L), g2) ((L-16) L)  x B = C''[(k1,k2)][16 + k0'] over k1   epilogue g1[k1]
//   mean1: A = phi1 phi2 (M^2)        x B = w[a0 < 8][.]        epilogue phi0[a0]
//   mean2: A = (phi0[8, M), phi2)     x B = w[8 + a0'][a1][a2] over a1            epilogue phi1[a1]
// (19% fewer DMMA at C3).  Same blocks, production, warp split and reduction as
// fused_predict_kernel.
template <int BW, int MM = 0, int G = 1>
__global__ void __launch_bounds__(kPredNT, 1)
fused_predict_split_kernel(const double* __restrict__ Xs, int64_t Ns, BasisView b, const VPlan pl,
                           const double* __restrict__ op, double sigma2, double c, double* __restrict__ mean,
                           double* __restrict__ var, uint32_t* flags) {
  constexpr int P = 3;
  extern __shared__ double sm[];
  RowLayout rl = row_layout(P, pl.M);
  rl.bw = BW;  // == row_layout(3, M).bw (the launcher picks BW by M)
  const bool want_var = var != nullptr;
  const int M = pl.M, L = pl.L, R = L - 16, R2 = M - 8;
  const int vk1 = (L * L + 3) / 4, vk2 = (R * L + 3) / 4, mk1 = (M * M + 3) / 4, mk2 = (R2 * M + 3) / 4;
  double* Bv1 = sm;                      // [vk1][2][32]
  double* Bv2 = Bv1 + vk1 * 2 * 32;      // [vk2][3][32]
  double* Bm1 = Bv2 + vk2 * 3 * 32;      // [mk1][1][32]
  double* Bm2 = Bm1 + mk1 * 32;          // [mk2][2][32]
  double* red = Bm2 + mk2 * 2 * 32;      // [kPKS][kPR][2]
  double* slab = red + kPKS * kPR * 2;   // [kPR * bw]
  uint32_t* offV1 = reinterpret_cast<uint32_t*>(slab + kPR * rl.bw);
  uint32_t* offV2 = offV1 + vk1 * 4;
  uint32_t* offM1 = offV2 + vk2 * 4;
  uint32_t* offM2 = offM1 + mk1 * 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // G independent warp groups (G = 2: two 8-warp halves on alternating 64-row blocks, one group's
  // production and epilogue overlapping the other's DMMA phase); each group has its own slab,
  // reduction buffer and named barrier
  constexpr int WG = kPredW / G, RB = kPR / G, GT = WG * 32;
  const int gid = warp / WG, gw = warp % WG, gt = tid % GT;
  auto gsync = [&]() {
    if constexpr (G == 1)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(1 + gid), "r"(GT) : "memory");
  };
  const double* w = op + pl.KP * pl.NP;
  const int64_t KM = int64_t(M) * M;
  auto pack2 = [&](int o0, int o1) { return uint32_t(o0) | (uint32_t(o1) << 8); };
  for (int i = tid; i < vk1 * 2 * 32; i += kPredNT) {  // C''[kappa = (k1, k2)][nu < 16]
    const int ln = i & 31, q = i >> 5, nf = q & 1, ks = q >> 1;
    const int kap = 4 * ks + (ln & 3), nu = 8 * nf + (ln >> 2);
    Bv1[i] = (want_var && kap < L * L) ? op[int64_t(kap) * pl.NP + nu] : 0.0;
  }
  for (int i = tid; i < vk2 * 3 * 32; i += kPredNT) {  // C''[(k1, k2)][16 + k0'], kappa' = k0' L + k2, column k1
    const int ln = i & 31, q = i >> 5, nf = q % 3, ks = q / 3;
    const int kap = 4 * ks + (ln & 3), k1 = 8 * nf + (ln >> 2);
    Bv2[i] = (want_var && kap < R * L && k1 < L) ? op[int64_t(k1 * L + kap % L) * pl.NP + 16 + kap / L] : 0.0;
  }
  for (int i = tid; i < mk1 * 32; i += kPredNT) {  // w[a0 < 8][(a1, a2)]
    const int ln = i & 31, ks = i >> 5;
    const int kap = 4 * ks + (ln & 3), a0 = ln >> 2;
    Bm1[i] = kap < M * M ? w[int64_t(a0) * KM + kap] : 0.0;
  }
  for (int i = tid; i < mk2 * 2 * 32; i += kPredNT) {  // w[8 + a0'][a1][a2], kappa' = a0' M + a2, column a1
    const int ln = i & 31, q = i >> 5, nf = q & 1, ks = q >> 1;
    const int kap = 4 * ks + (ln & 3), a1 = 8 * nf + (ln >> 2);
    Bm2[i] = (kap < R2 * M && a1 < M) ? w[int64_t(8 + kap / M) * KM + int64_t(a1) * M + kap % M] : 0.0;
  }
  for (int k = tid; k < vk1 * 4; k += kPredNT)
    offV1[k] = k < L * L ? pack2(rl.goff + L + k / L, rl.goff + 2 * L + k % L) : pack2(rl.zero, rl.one);
  for (int k = tid; k < vk2 * 4; k += kPredNT)
    offV2[k] = k < R * L ? pack2(rl.goff + 16 + k / L, rl.goff + 2 * L + k % L) : pack2(rl.zero, rl.one);
  for (int k = tid; k < mk1 * 4; k += kPredNT)
    offM1[k] = k < M * M ? pack2(rl.poff + M + k / M, rl.poff + 2 * M + k % M) : pack2(rl.zero, rl.one);
  for (int k = tid; k < mk2 * 4; k += kPredNT)
    offM2[k] = k < R2 * M ? pack2(rl.poff + 8 + k / M, rl.poff + 2 * M + k % M) : pack2(rl.zero, rl.one);
  bool bad_x = false, bad = false;
  const bool plane = gt < RB * P;
  const int prow = gt / P, pdim = gt - (gt / P) * P;
  const int64_t nb = (Ns + RB - 1) / RB;
  double* const gslab = slab + gid * RB * rl.bw;
  double* const gred = red + gid * kPKS * RB * 2;
  auto load_x = [&](int64_t blk) -> double {
    const int64_t r = blk * RB + prow;
    return (plane && blk < nb && r < Ns) ? Xs[r * P + pdim] : 0.0;
  };
  auto produce = [&](double x, int64_t blk) {
    if (!plane) return;
    double* row = gslab + prow * rl.bw;
    if (blk * RB + prow < Ns) {
      bad_x |= not_finite(x);
      eval_phi_g_dim_u(x, 0.0, b, pdim, pl.hc, row + rl.poff + pdim * M, row + rl.goff + pdim * L, nullptr);
    } else {
      for (int k = 0; k < M; ++k) row[rl.poff + pdim * M + k] = 0.0;
      for (int k = 0; k < L; ++k) row[rl.goff + pdim * L + k] = 0.0;
    }
    if (pdim == 0) {
      row[rl.one] = 1.0;
      row[rl.zero] = 0.0;
    }
  };
  const int64_t blk0 = int64_t(blockIdx.x) * G + gid, stride = int64_t(gridDim.x) * G;
  double xn = load_x(blk0);
  const int mg = gw % (WG / kPKS), kq = gw / (WG / kPKS);
  auto half = [&](int n, int q) { return q * n / kPKS; };
  // epilogue offsets: var1 g0[nu < 16], var2 g1[k1 < L], mean1 phi0[a0 < 8], mean2 phi1[a1 < M]
  int oE1[2][2], oE2[3][2], oM1[1][2], oM2[2][2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int cc = 2 * (lane & 3) + e;
#pragma unroll
    for (int nf = 0; nf < 2; ++nf) oE1[nf][e] = rl.goff + nf * 8 + cc;
#pragma unroll
    for (int nf = 0; nf < 3; ++nf) oE2[nf][e] = nf * 8 + cc < L ? rl.goff + L + nf * 8 + cc : rl.zero;
    oM1[0][e] = rl.poff + cc;
#pragma unroll
    for (int nf = 0; nf < 2; ++nf) oM2[nf][e] = nf * 8 + cc < M ? rl.poff + M + nf * 8 + cc : rl.zero;
  }
  __syncthreads();
  // stagger: group 1 starts producing once group 0 has produced its first block, so the groups'
  // DMMA phases are offset by a production phase from the start
  bool staggered = G == 1 || gid == 1;
  if constexpr (G == 2)
    if (gid == 1) asm volatile("bar.sync 3, %0;" ::"r"(kPredNT) : "memory");

  for (int64_t blk = blk0; blk < nb; blk += stride) {
    produce(xn, blk);
    xn = load_x(blk + stride);
    gsync();
    if constexpr (G == 2)
      if (!staggered) {
        asm volatile("bar.arrive 3, %0;" ::"r"(kPredNT) : "memory");
        staggered = true;
      }
    const double* row0 = gslab + (mg * 16 + (lane >> 2)) * rl.bw;
    double aV1[kPMF][2][2], aV2[kPMF][3][2], aM1[kPMF][1][2], aM2[kPMF][2][2];
#pragma unroll
    for (int f = 0; f < kPMF; ++f)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        aV1[f][0][e] = aV1[f][1][e] = aV2[f][0][e] = aV2[f][1][e] = aV2[f][2][e] = 0.0;
        aM1[f][0][e] = aM2[f][0][e] = aM2[f][1][e] = 0.0;
      }
    if constexpr (MM > 0) {
      // compile-time section bounds (M known): per K-half straight-line loops
      constexpr int cL = 2 * MM - 1, cR = cL - 16, cR2 = MM - 8;
      constexpr int cvk1 = (cL * cL + 3) / 4, cvk2 = (cR * cL + 3) / 4, cmk1 = (MM * MM + 3) / 4,
                    cmk2 = (cR2 * MM + 3) / 4;
      static_assert(kPKS == 2, "two K halves");
#ifdef FAGP_PRED_UNROLL
      constexpr int UNR = FAGP_PRED_UNROLL;
#else
      constexpr int UNR = G == 1 ? 64 : 16;
#endif
      auto sections = [&](auto q) {
        constexpr int Q = decltype(q)::value;
        if (want_var) {
          contract_ct<2, 2, BW, Q * cvk1 / 2, (Q + 1) * cvk1 / 2, UNR>(row0, offV1, Bv1, lane, aV1);
          contract_ct<2, 3, BW, Q * cvk2 / 2, (Q + 1) * cvk2 / 2, UNR>(row0, offV2, Bv2, lane, aV2);
        }
        contract_ct<2, 1, BW, Q * cmk1 / 2, (Q + 1) * cmk1 / 2, UNR>(row0, offM1, Bm1, lane, aM1);
        contract_ct<2, 2, BW, Q * cmk2 / 2, (Q + 1) * cmk2 / 2, UNR>(row0, offM2, Bm2, lane, aM2);
      };
      if (kq == 0)
        sections(std::integral_constant<int, 0>{});
      else
        sections(std::integral_constant<int, 1>{});
    } else {
      if (want_var) {
        contract<2, 2, BW>(row0, rl.bw, offV1, Bv1, half(vk1, kq), half(vk1, kq + 1), lane, aV1);
        contract<2, 3, BW>(row0, rl.bw, offV2, Bv2, half(vk2, kq), half(vk2, kq + 1), lane, aV2);
      }
      contract<2, 1, BW>(row0, rl.bw, offM1, Bm1, half(mk1, kq), half(mk1, kq + 1), lane, aM1);
      contract<2, 2, BW>(row0, rl.bw, offM2, Bm2, half(mk2, kq), half(mk2, kq + 1), lane, aM2);
    }
#pragma unroll
    for (int f = 0; f < kPMF; ++f) {
      const double* row = row0 + 8 * f * rl.bw;
      double vs = 0.0, ms = 0.0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (want_var) {
#pragma unroll
          for (int nf = 0; nf < 2; ++nf) vs = fma(aV1[f][nf][e], row[oE1[nf][e]], vs);
#pragma unroll
          for (int nf = 0; nf < 3; ++nf) vs = fma(aV2[f][nf][e], row[oE2[nf][e]], vs);
        }
        ms = fma(aM1[f][0][e], row[oM1[0][e]], ms);
#pragma unroll
        for (int nf = 0; nf < 2; ++nf) ms = fma(aM2[f][nf][e], row[oM2[nf][e]], ms);
      }
      vs += __shfl_xor_sync(0xffffffffu, vs, 1);
      vs += __shfl_xor_sync(0xffffffffu, vs, 2);
      ms += __shfl_xor_sync(0xffffffffu, ms, 1);
      ms += __shfl_xor_sync(0xffffffffu, ms, 2);
      if ((lane & 3) == 0) {
        const int r = mg * 16 + 8 * f + (lane >> 2);
        gred[(kq * RB + r) * 2 + 0] = vs;
        gred[(kq * RB + r) * 2 + 1] = ms;
      }
    }
    gsync();
    if (gt < RB) {
      const int64_t row_i = blk * RB + gt;
      if (row_i < Ns) {
        double vs = gred[gt * 2], ms = gred[gt * 2 + 1];
#pragma unroll
        for (int q = 1; q < kPKS; ++q) {
          vs += gred[(q * RB + gt) * 2];
          ms += gred[(q * RB + gt) * 2 + 1];
        }
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
  if constexpr (G == 2)
    if (!staggered) asm volatile("bar.arrive 3, %0;" ::"r"(kPredNT) : "memory");  // group 0 had no block
  if (bad_x) raise_flag(flags, FAGP_FLAG_X_NONFINITE);
  if (bad) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
}

static size_t split_predict_smem(int M) {
  const int L = 2 * M - 1, R = L - 16, R2 = M - 8;
  const int vk1 = (L * L + 3) / 4, vk2 = (R * L + 3) / 4, mk1 = (M * M + 3) / 4, mk2 = (R2 * M + 3) / 4;
  const RowLayout rl = row_layout(3, M);
  return (size_t(vk1) * 2 * 32 + size_t(vk2) * 3 * 32 + size_t(mk1) * 32 + size_t(mk2) * 2 * 32 +
          size_t(kPKS) * kPR * 2 + size_t(kPR) * rl.bw) * sizeof(double) +
         size_t(vk1 + vk2 + mk1 + mk2) * 4 * sizeof(uint32_t);
}

static bool make_vplan(int64_t Ns, int p, int M, VPlan& pl) {
  std::memset(&pl, 0, sizeof(pl));
  if (!modal_on(p, M) || p > kMaxF || M > 12) return false;
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
  const int NFV = M <= 4 ? 1 : M <= 8 ? 2 : 3;
  if (pl.NR > 8 * NFV || p - pl.pN > kMaxF - 1 || pl.pN > 2 || (pl.pN == 2 && M > 4)) return false;
  pl.vks = int(ceil_div(pl.KR, 4));
  pl.NM = M;
  pl.KM = int(ipow(M, p - 1));
  pl.mks = int(ceil_div(pl.KM, 4));
  const int NFM = M <= 8 ? 1 : 2;
  const RowLayout rl = row_layout(p, M);
  if (rl.bw > 256) return false;  // byte-packed offsets
  pl.smem = (size_t(pl.vks) * NFV * 32 + size_t(pl.mks) * NFM * 32 + size_t(kPKS) * kPR * 2 +
             size_t(kPR) * rl.bw) * sizeof(double) +
            size_t(pl.vks + pl.mks) * 4 * sizeof(uint32_t);
  if (pl.smem > 225 * 1024) return false;
  if (kPR * p > kPredNT) return false;
  pl.nblocks = ceil_div(tmax<int64_t>(Ns, 0), kPR);
  pl.grid = int(tmax<int64_t>(1, tmin<int64_t>(num_sms(), pl.nblocks)));
  pl.hc = herm_coef_host();
  return true;
}

template <int FK, int FE, int NFV, int NFM>
static int launch_pred(const double* Xs, int64_t Ns, const fagp_basis* b, const VPlan& pl, const double* op,
                       double sigma2, double c, double* mean, double* var, uint32_t* flags, cudaStream_t s) {
  auto kern = fused_predict_kernel<FK, FE, FK + FE - 1, NFV, NFM>;
  FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem)));
  kern<<<pl.grid, kPredNT, pl.smem, s>>>(Xs, Ns, view(b), pl, op, sigma2, c, mean, var, flags);
  return FAGP_OK;
}

template <int FK>
static int launch_pred_fk(const double* Xs, int64_t Ns, const fagp_basis* b, const VPlan& pl, const double* op,
                          double sigma2, double c, double* mean, double* var, uint32_t* flags, cudaStream_t s) {
  if (pl.pN == 2) {
    if constexpr (FK + 1 <= kMaxF - 1) return launch_pred<FK, 2, 1, 1>(Xs, Ns, b, pl, op, sigma2, c, mean, var, flags, s);
    return FAGP_EUNSUPPORTED;
  }
  if (pl.M <= 4) return launch_pred<FK, 1, 1, 1>(Xs, Ns, b, pl, op, sigma2, c, mean, var, flags, s);
  if (pl.M <= 8) return launch_pred<FK, 1, 2, 1>(Xs, Ns, b, pl, op, sigma2, c, mean, var, flags, s);
  return launch_pred<FK, 1, 3, 2>(Xs, Ns, b, pl, op, sigma2, c, mean, var, flags, s);
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
  const char* se = getenv("FAGP_PREDICT_SPLIT");
  if (b->p == 3 && pl.pN == 1 && b->M >= 9 && b->M <= 12 && !(se && se[0] == '0')) {
    const size_t smem = split_predict_smem(b->M);
    auto go = [&](auto kern) -> int {
      FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      kern<<<pl.grid, kPredNT, smem, s>>>(Xs, Ns, view(b), pl, op, sigma2, c, mean, var, flags);
      FAGP_LAUNCH_CHECK();
      return FAGP_OK;
    };
    const char* sg = getenv("FAGP_PREDICT_GROUPS");
    const bool g2 = !(sg && sg[0] == '1');
    switch (row_layout(3, b->M).bw) {  // compile-time row strides (M 9, 10: 100; 11: 116; 12: 132)
      // M as a template argument: compile-time section bounds (0.82 -> 0.76 ms at C3)
      case 100:
        if (b->M == 10)
          return g2 ? go(fused_predict_split_kernel<100, 10, 2>) : go(fused_predict_split_kernel<100, 10, 1>);
        return g2 ? go(fused_predict_split_kernel<100, 9, 2>) : go(fused_predict_split_kernel<100, 9, 1>);
      case 116: return g2 ? go(fused_predict_split_kernel<116, 11, 2>) : go(fused_predict_split_kernel<116, 11, 1>);
      case 132: return g2 ? go(fused_predict_split_kernel<132, 12, 2>) : go(fused_predict_split_kernel<132, 12, 1>);
      default: return FAGP_EUNSUPPORTED;
    }
  }
  int rc;
  switch (b->p - pl.pN) {
    case 1: rc = launch_pred_fk<1>(Xs, Ns, b, pl, op, sigma2, c, mean, var, flags, s); break;
    case 2: rc = launch_pred_fk<2>(Xs, Ns, b, pl, op, sigma2, c, mean, var, flags, s); break;
    case 3: rc = launch_pred_fk<3>(Xs, Ns, b, pl, op, sigma2, c, mean, var, flags, s); break;
    default: rc = FAGP_EUNSUPPORTED;
  }
  if (rc) return rc;
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // namespace fused
}  // namespace fagp

namespace fagp {
namespace tiled {  // gram_tiled.cu: the output-tiled fused Gram (shapes beyond fused_gram's registers)
bool eligible(int64_t N, int p, int M);
size_t workspace(int64_t N, int p, int M);
int gram(const double* X, const double* y, double c, int64_t N, const fagp_basis* b, double* out, void* ws,
         size_t ws_bytes, uint32_t* flags, cudaStream_t s);
}  // namespace tiled
namespace ptiled {  // predict_tiled.cu: the output-tiled fused predict
bool eligible(int p, int M);
size_t workspace(int64_t Ns, int p, int M);
int predict(const double* Xs, int64_t Ns, const fagp_basis* b, const double* op, double sigma2, double c,
            double* mean, double* var, void* ws, size_t ws_bytes, uint32_t* flags, cudaStream_t s);
}  // namespace ptiled
}  // namespace fagp

// =======================================================================================
// C ABI: the point-input entry points (tables only where no fused layout applies)
using namespace fagp;

extern "C" {

size_t fagp_gram_x_workspace_size(int64_t N, const fagp_basis* basis) {
  if (check_basis(basis) || N < 0) return 0;
  if (fused::gram_eligible(N, basis->p, basis->M)) return fused::gram_workspace(N, basis->p, basis->M);
  if (tiled::eligible(N, basis->p, basis->M)) return tiled::workspace(N, basis->p, basis->M);
  const size_t table = size_t(N) * table_width(basis->p, basis->M) * sizeof(double);
  return round_up(table, 256) + fagp_gram_workspace_size(N, basis);
}

int32_t fagp_gram_x_chunks(int64_t N, const fagp_basis* basis) {
  if (check_basis(basis) || N < 0) return 1;
  return fused::gram_chunks(N, basis->p, basis->M);
}

int fagp_gram_x_upload_chunk(const double* X_host, const double* y_host, int64_t N, const fagp_basis* basis,
                              int32_t k, double* X, double* y, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || (N > 0 && (X_host == nullptr || X == nullptr))) return FAGP_EINVAL;
  return fused::upload_chunk(X_host, y_host, N, basis->p, basis->M, k, X, y, static_cast<cudaStream_t>(stream));
}

int fagp_gram_x_stage_chunk(const double* X_src, const double* y_src, int64_t N, const fagp_basis* basis, int32_t k,
                            double* X_pinned, double* y_pinned, int32_t threads) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || (N > 0 && (X_src == nullptr || X_pinned == nullptr))) return FAGP_EINVAL;
  if (N == 0) return FAGP_OK;
  return fused::stage_chunk(X_src, y_src, N, basis->p, basis->M, k, X_pinned, y_pinned, threads);
}

int fagp_gram_x_chunk(const double* X, int64_t N, const fagp_basis* basis, const double* y, double mean_const,
                      int32_t k, double* gram, void* workspace, size_t workspace_bytes, uint32_t* flags,
                      void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (N < 0 || gram == nullptr || (N > 0 && X == nullptr)) return FAGP_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (fused::gram_eligible(N, basis->p, basis->M))
    return fused::gram(X, y, mean_const, N, basis, k, k + 1, gram, workspace, workspace_bytes, flags, s, nullptr);
  if (k != 0) return FAGP_EINVAL;
  if (tiled::eligible(N, basis->p, basis->M))
    return tiled::gram(X, y, mean_const, N, basis, gram, workspace, workspace_bytes, flags, s);
  const size_t table = round_up(size_t(N) * table_width(basis->p, basis->M) * sizeof(double), 256);
  if (workspace == nullptr || workspace_bytes < table + fagp_gram_workspace_size(N, basis)) return FAGP_EWORKSPACE;
  double* T = static_cast<double*>(workspace);
  if (N > 0) {
    st = fagp_basis_eval(X, N, basis, y, mean_const, T, flags, stream);
    if (st) return st;
  }
  return fagp_gram(T, N, basis, gram, static_cast<char*>(workspace) + table, workspace_bytes - table, flags, stream);
}

int fagp_gram_x(const double* X, int64_t N, const fagp_basis* basis, const double* y, double mean_const,
                double* gram, void* workspace, size_t workspace_bytes, uint32_t* flags, void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (fused::gram_eligible(N, basis->p, basis->M)) {
    if (N < 0 || gram == nullptr || (N > 0 && X == nullptr)) return FAGP_EINVAL;
    return fused::gram(X, y, mean_const, N, basis, 0, fused::gram_chunks(N, basis->p, basis->M), gram, workspace,
                       workspace_bytes, flags, static_cast<cudaStream_t>(stream), nullptr);
  }
  return fagp_gram_x_chunk(X, N, basis, y, mean_const, 0, gram, workspace, workspace_bytes, flags, stream);
}

int fagp_gram_x_pipelined(const double* X, int64_t N, const fagp_basis* basis, const double* y, double mean_const,
                          uint32_t* ready, double* gram, void* workspace, size_t workspace_bytes, uint32_t* flags,
                          void* stream) {
  int st = check_basis(basis);
  if (st) return st;
  if (!fused::gram_eligible(N, basis->p, basis->M)) return FAGP_EUNSUPPORTED;
  if (N < 0 || gram == nullptr || ready == nullptr || (N > 0 && X == nullptr)) return FAGP_EINVAL;
  return fused::gram(X, y, mean_const, N, basis, 0, fused::gram_chunks(N, basis->p, basis->M), gram, workspace,
                     workspace_bytes, flags, static_cast<cudaStream_t>(stream), ready);
}

int fagp_gram_x_signal(uint32_t* ready, int32_t k, void* stream) {
  // a stream-ordered 4-byte H2D copy: executed by a copy engine behind the chunk's rows (a
  // memset would be a kernel, which could not start beside the Gram that waits for it)
  static uint32_t* one = nullptr;
  if (one == nullptr) {
    void* h = nullptr;
    FAGP_CUDA_TRY(cudaHostAlloc(&h, sizeof(uint32_t), cudaHostAllocPortable));
    *static_cast<uint32_t*>(h) = 1u;
    one = static_cast<uint32_t*>(h);
  }
  if (ready == nullptr || k < 0) return FAGP_EINVAL;
  FAGP_CUDA_TRY(cudaMemcpyAsync(ready + k, one, sizeof(uint32_t), cudaMemcpyHostToDevice,
                                static_cast<cudaStream_t>(stream)));
  return FAGP_OK;
}

int fagp_route_info(int64_t N, int64_t Ns, const fagp_basis* basis, int32_t* out) {
  int st = check_basis(basis);
  if (st) return st;
  if (out == nullptr || N < 0 || Ns < 0) return FAGP_EINVAL;
  out[0] = fused::gram_eligible(N, basis->p, basis->M) ? 1 : tiled::eligible(N, basis->p, basis->M) ? 2 : 0;
  out[1] = fused::predict_eligible(basis->p, basis->M) ? 1 : ptiled::eligible(basis->p, basis->M) ? 2 : 0;
  out[2] = (modal_on(basis->p, basis->M) && basis->m <= 2048) ? 1 : 0;  // factor.cu kFactorInvMaxM
  return FAGP_OK;
}

int64_t fagp_predict_x_wave_rows(const fagp_basis* basis) {
  if (check_basis(basis) || !fused::predict_eligible(basis->p, basis->M)) return 0;
  return int64_t(num_sms()) * fused::kPR;
}

size_t fagp_predict_x_workspace_size(int64_t Ns, const fagp_basis* basis) {
  if (check_basis(basis) || Ns < 0) return 0;
  if (fused::predict_eligible(basis->p, basis->M)) return 0;
  if (ptiled::eligible(basis->p, basis->M)) return ptiled::workspace(Ns, basis->p, basis->M);
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
  if (ptiled::eligible(basis->p, basis->M))
    return ptiled::predict(Xs, Ns, basis, predict_op, sigma2, mean_const, mean, var, workspace, workspace_bytes,
                           flags, s);
  const size_t table = size_t(Ns) * table_width(basis->p, basis->M) * sizeof(double);
  if (workspace == nullptr || workspace_bytes < table) return FAGP_EWORKSPACE;
  double* Ts = static_cast<double*>(workspace);
  st = fagp_basis_eval(Xs, Ns, basis, nullptr, 0.0, Ts, flags, stream);
  if (st) return st;
  return fagp_predict(Ts, Ns, basis, predict_op, sigma2, mean_const, mean, var, flags, stream);
}

}  // extern "C"
