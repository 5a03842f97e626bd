// Output-tiled fused modal Gram: [K | t] for the shapes whose modal output does not fit one
// CTA's registers (BASELINE C4: p 4, M 8, L^p = 50,625 entries; C5: p 5, M 6, 161,051), with
// the eigenfunctions evaluated on chip exactly as in fused.cu -- no basis table in HBM.
//
//   K[kappa] = sum_r prod_d g_{d,kappa_d}(x_rd)                  (modal moments -> G = Phi^T Phi,
//                                                                 mercer.py:284-292, posterior.py:168)
//   t[a]     = sum_r (y_r - c) prod_d phi_{d,a_d}(x_rd)           (posterior.py:229-233)
//
// The dimensions are split in two halves, A = dims [0, q) and B = dims [q, p) (q = p / 2), so
// K is the GEMM over rows of the Khatri-Rao products  A_r = g_0 (x) ... (x) g_{q-1}  (L^q
// columns) and  B_r = g_q (x) ... (x) g_{p-1}  (L^(p-q) columns): both sides are wide (225 x 225
// at C4, 121 x 1331 at C5), so every generated operand fragment feeds 4 DMMAs.  t is the same
// GEMM with phi in place of g and r phi_{p-1} as the last B factor; its fragment pairs are dealt
// round-robin to the K tiles (JT per warp: C4 64 pairs over 4 tiles, C5 135 over 11 -- one per
// warp), so every CTA carries the same mix of work and no CTA runs a thin t-only tile.
//
// B200 mapping:
//  * Output tiles of 16 x 16 m8n8 fragments (128 x 128 entries); one CTA (16 warps, 4 x 4
//    fragments each, 32 accumulator doubles per thread) owns one tile for a contiguous row
//    range.  The CTAs are dealt to the tiles in proportion to each tile's per-k-step cost
//    (greedy, on the per-SM-sub-partition DMMA count), so edge tiles get more rows per CTA and
//    the makespan is ~N x total work / #SMs.  Fragments outside the output are skipped (a
//    warp-uniform branch), not padded; warps are laid out on the sub-partitions as a Latin
//    square (SMSP w % 4 holds one warp of every A row and B column of the tile), so a partial
//    edge tile still spreads its DMMAs over the four tensor pipes.
//  * Per block of BR rows: a production phase (all threads; two (row, dimension) evaluations
//    per thread in lockstep, eigfun.cuh, one exponential shared by phi and g) into a
//    shared-memory row slab, then BR / 4 DMMA k-steps whose A / B fragments are formed in
//    registers (q - 1 resp. p - q - 1 DMULs from conflict-free LDS.64, row stride == 4 mod 16).
//  * One partial per CTA (its K tile, then its t pairs; fragment-major, coalesced), summed per
//    output entry over the tile's CTAs in CTA order by reduce_kernel: deterministic, no atomics; the result is the
//    [K | t] buffer of fagp_gram (the multi-GPU all-reduce payload).
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "eigfun.cuh"
#include "modal.cuh"

namespace fagp {
namespace tiled {

#ifndef FAGP_TILED_UNROLL
#define FAGP_TILED_UNROLL 4
#endif
constexpr int kTiledUnroll = FAGP_TILED_UNROLL;  // k-loop unroll of the full-fragment path

constexpr int kW = 16, kNT = kW * 32;  // 16 warps
constexpr int kTF = 16;                // fragments per tile side
constexpr int kWF = 4;                 // fragments per warp side
constexpr int kMaxTiles = 48;
constexpr int kMaxF = 4;               // factors per side (p <= 8)
constexpr int kJT = 2;                 // t fragment pairs per warp (at most)
constexpr int kPartial = (kTF * kTF + kW * kJT) * 64;  // doubles per CTA partial: K tile | t pairs

struct Tile {
  int a0, na;  // A fragments [a0, a0 + na)
  int b0, nb;  // B fragments [b0, b0 + nb)
};

struct TPlan {
  int p, M, L, q;
  int64_t LA, LB, MA, MB;  // column counts: K sides L^q, L^(p-q); t sides M^q, M^(p-q)
  int goff, poff, rpoff, one, zero, bw;  // row slab layout (doubles), bw % 16 == 4
  int BR;                                // rows per block
  int masked;                            // 0: a warp with any valid fragment runs all 16 DMMAs (invalid
                                         // fragments are zero -- measured faster than predicated DMMAs); 1: skip
  long long* prof;                       // diagnostics build (-DFAGP_TILED_PROF): per CTA [tile, total, produce, k-loop, barrier] cycles of warp 0
  int ntiles;                            // K tiles
  int fr[2], nt[2];                      // per side: K fragments, tiles (fragments split evenly)
  int tfa, tfb, tpairs, jt;              // t: fragments per side, fragment pairs, pairs per warp
  int grid;
  int64_t Klen, len;                     // L^p, L^p + m
  int64_t N;
  Tile tiles[kMaxTiles];
  int first[kMaxTiles], cnt[kMaxTiles];  // CTAs [first, first + cnt) work on tile t
  int sbase[kMaxTiles];                  // tile t's partials: slots [sbase, sbase + cnt)
  // span = 1: the CTAs cut the tiles' total work (cost x rows, tile-major) evenly, so a CTA may
  // finish one tile and start the next (two partial slots); span = 0: whole CTAs per tile, rows
  // split evenly over a tile's CTAs
  int span;
  int wcost[kMaxTiles];                  // per-row cost of tile t (tile_cost)
  int64_t wstart[kMaxTiles + 1];         // work before tile t (wcost x N, prefix sums)
  int nslots;
  HermCoef hc;
};

// (tile, first row) at work position w of a spanning plan, rows rounded down to whole k-steps;
// the same integer arithmetic on the host (slot layout) and in the kernel (row ranges)
__host__ __device__ __forceinline__ void span_pos(const TPlan& pl, int64_t w, int& t, int64_t& row) {
  if (w >= pl.wstart[pl.ntiles]) {
    t = pl.ntiles - 1;
    row = pl.N;
    return;
  }
  t = 0;
  while (t + 1 < pl.ntiles && pl.wstart[t + 1] <= w) ++t;
  row = ((w - pl.wstart[t]) / pl.wcost[t]) & ~int64_t(3);
}
__host__ __device__ __forceinline__ int64_t span_bound(const TPlan& pl, int i) {
  return pl.wstart[pl.ntiles] / pl.grid * i + pl.wstart[pl.ntiles] % pl.grid * i / pl.grid;
}

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// Warp w runs on SM sub-partition w % 4 and owns A fragments 4 wa .. and B fragments 4 wb ..
// with wb = w / 4 and wa = (w - f(wb)) mod 4, f = (0, 2, 1, 3): a Latin square (every SMSP
// holds one warp of each A row and each B column of the tile) whose top-left 2 x 2 block also
// lands on four different SMSPs, so half tiles keep all four tensor pipes busy.
__host__ __device__ __forceinline__ void warp_tile(int w, int& wa, int& wb) {
  wb = w >> 2;
  const int f = (0x3120 >> (4 * wb)) & 0xf;  // f(0..3) = 0, 2, 1, 3
  wa = ((w & 3) - f + 4) & 3;
}

// Cycles per k-step of a tile with na x nb valid fragments (empirical, profiled per CTA with
// FAGP_TILED_PROF at C4 / C5): the busiest SM sub-partition's DMMA pipe time (16 cycles per
// DMMA) at the ~69% the k-loop sustains, or -- when a sub-partition holds fewer than four busy
// warps -- one warp's serial k-step (~700 cycles of LDS -> DMUL -> DMMA latency plus its DMMAs),
// which no other warp hides.
static int tile_cost(int na, int nb) {
  int pipe[4] = {0, 0, 0, 0}, serial[4] = {0, 0, 0, 0};
  for (int w = 0; w < kW; ++w) {
    int wa, wb;
    warp_tile(w, wa, wb);
    const int va = tmax(0, tmin(kWF, na - kWF * wa)), vb = tmax(0, tmin(kWF, nb - kWF * wb));
    const int d = va * vb > 0 ? kWF * kWF : 0;  // a warp with any valid fragment runs all 16 DMMAs
    pipe[w % 4] += 16 * d;
    if (d > 0) serial[w % 4] = tmax(serial[w % 4], 700 + 16 * d);
  }
  int c = 0;
  for (int s = 0; s < 4; ++s) c = tmax(c, tmax(pipe[s] * 100 / 69, serial[s]));
  return c;
}

static bool make_tplan(int64_t N, int p, int M, TPlan& pl) {
  std::memset(&pl, 0, sizeof(pl));
  if (!modal_on(p, M) || M > kHermMax / 2) return false;
  pl.p = p;
  pl.M = M;
  pl.L = modal_L(M);
  pl.q = p / 2;
  if (pl.q > kMaxF || p - pl.q > kMaxF) return false;
  pl.LA = ipow(pl.L, pl.q);
  pl.LB = ipow(pl.L, p - pl.q);
  pl.MA = ipow(M, pl.q);
  pl.MB = ipow(M, p - pl.q);
  pl.Klen = pl.LA * pl.LB;
  pl.len = pl.Klen + pl.MA * pl.MB;
  pl.N = N;
  pl.goff = 0;
  pl.poff = p * pl.L;
  pl.rpoff = pl.poff + p * M;
  pl.one = pl.rpoff + M;
  pl.zero = pl.one + 1;
  int w = pl.zero + 1;
  while (w % 16 != 4) ++w;
  pl.bw = w;
  // two (row, dimension) evaluations per thread per block; one spare row for idle items
  pl.BR = (2 * kNT / p) / 4 * 4;
  while (pl.BR > 4 && (size_t(pl.BR + 1) * pl.bw + size_t(pl.BR) * (p + 1)) * sizeof(double) > 220 * 1024) pl.BR -= 4;
  if (pl.BR < 4) return false;
  // tiles
  // the fragments of a side are split evenly over its tiles (tile i: [i f / n, (i + 1) f / n)),
  // so no tile is a thin remainder
  auto add = [&](int64_t ca, int64_t cb) -> bool {
    const int fa = int(ceil_div(ca, 8)), fb = int(ceil_div(cb, 8));
    const int nta = int(ceil_div(fa, kTF)), ntb = int(ceil_div(fb, kTF));
    pl.fr[0] = fa;
    pl.fr[1] = fb;
    pl.nt[0] = nta;
    pl.nt[1] = ntb;
    for (int ta = 0; ta < nta; ++ta)
      for (int tb = 0; tb < ntb; ++tb) {
        if (pl.ntiles >= kMaxTiles) return false;
        Tile& t = pl.tiles[pl.ntiles++];
        t.a0 = ta * fa / nta;
        t.na = (ta + 1) * fa / nta - t.a0;
        t.b0 = tb * fb / ntb;
        t.nb = (tb + 1) * fb / ntb - t.b0;
      }
    return true;
  };
  if (!add(pl.LA, pl.LB)) return false;
  pl.tfa = int(ceil_div(pl.MA, 8));
  pl.tfb = int(ceil_div(pl.MB, 8));
  pl.tpairs = pl.tfa * pl.tfb;
  pl.jt = int(ceil_div(pl.tpairs, int64_t(pl.ntiles) * kW));
  if (pl.jt > kJT) return false;
  // CTAs dealt to tiles by cost: greedy on cost / count (the makespan of a tile ~ rows / cnt x cost)
  const int G = tmax(num_sms(), pl.ntiles);
  for (int t = 0; t < pl.ntiles; ++t) pl.cnt[t] = 1;
  int64_t rows_cap = ceil_div(tmax<int64_t>(N, 1), 4);  // no more CTAs on a tile than 4-row groups
  for (int g = pl.ntiles; g < G; ++g) {
    int best = -1;
    double bv = -1.0;
    for (int t = 0; t < pl.ntiles; ++t) {
      if (pl.cnt[t] >= rows_cap) continue;
      const double v = double(tile_cost(pl.tiles[t].na, pl.tiles[t].nb)) / pl.cnt[t];
      if (v > bv) {
        bv = v;
        best = t;
      }
    }
    if (best < 0) break;
    ++pl.cnt[best];
  }
  int f = 0;
  for (int t = 0; t < pl.ntiles; ++t) {
    pl.first[t] = f;
    pl.sbase[t] = f;
    f += pl.cnt[t];
  }
  pl.grid = f;
  pl.nslots = f;
  // whole CTAs per tile leave the makespan at cost x rows / min count (C5: 11 equal tiles on 148
  // SMs -> 13 or 14 CTAs per tile, the 13-CTA tiles 7% longer); large N spans the tiles instead
  // (measured: C5 121.0 -> 119.8 ms; C4, whose deal is within 0.3% of even, 20.27 -> 20.43 ms, so
  // only a deal more than 2% off even spans)
  double mk = 0.0, tot = 0.0;
  for (int t = 0; t < pl.ntiles; ++t) {
    const double ct = tile_cost(pl.tiles[t].na, pl.tiles[t].nb);
    mk = ct / pl.cnt[t] > mk ? ct / pl.cnt[t] : mk;
    tot += ct;
  }
  const char* se = getenv("FAGP_TILED_SPAN");
  pl.span = pl.ntiles < G && N >= 4096 && mk * G > 1.02 * tot;
  if (se) pl.span = pl.ntiles < G && N >= 4096 && se[0] != '0';  // A/B knob: force either deal
  if (pl.span) {
    const TPlan whole = pl;  // the whole-CTA deal, kept if the spanning one is not well formed
    pl.grid = G;
    pl.wstart[0] = 0;
    for (int t = 0; t < pl.ntiles; ++t) {
      pl.wcost[t] = tile_cost(pl.tiles[t].na, pl.tiles[t].nb);
      pl.wstart[t + 1] = pl.wstart[t] + int64_t(pl.wcost[t]) * N;
      pl.first[t] = -1;
      pl.cnt[t] = 0;
    }
    int slots = 0;
    for (int i = 0; i < G; ++i) {
      int ts, te;
      int64_t rs, re;
      span_pos(pl, span_bound(pl, i), ts, rs);
      span_pos(pl, span_bound(pl, i + 1), te, re);
      for (int t = ts; t <= te; ++t) {
        const int64_t r0 = t == ts ? rs : 0, r1 = t == te ? re : N;
        if (r0 >= r1) continue;
        if (pl.first[t] < 0) {
          pl.first[t] = i;
          pl.sbase[t] = slots;
        }
        if (pl.first[t] + pl.cnt[t] != i) pl.span = 0;  // contributors must be consecutive CTAs
        ++pl.cnt[t];
        ++slots;
      }
    }
    for (int t = 0; t < pl.ntiles; ++t)
      if (pl.cnt[t] == 0) pl.span = 0;
    pl.nslots = slots;
    if (!pl.span) {
      pl = whole;
      pl.span = 0;
    }
  }
  pl.hc = herm_coef_host();
  if (const char* e = getenv("FAGP_TILED_MASKED")) pl.masked = atoi(e);  // A/B knob
  return true;
}

// 8-byte cp.async with zero fill (src-size 0) for elements outside the range
__device__ __forceinline__ void cp_async_8z(void* smem, const void* gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0));
}

// slab offsets of the F factors of column c of a side (dims [d0, d0 + F), radix R, first dim
// slowest); the last factor may come from another section (r phi_{p-1}); invalid -> (0, 1, ..)
template <int F>
__device__ __forceinline__ void col_offs(int64_t c, int64_t ncols, int d0, int R, int sec, int last_sec,
                                         const TPlan& pl, int (&off)[F]) {
  if (c >= ncols) {
    off[0] = pl.zero;
#pragma unroll
    for (int e = 1; e < F; ++e) off[e] = pl.one;
    return;
  }
#pragma unroll
  for (int e = F - 1; e >= 0; --e) {
    const int dig = int(c % R);
    c /= R;
    off[e] = (e == F - 1 && last_sec >= 0) ? last_sec + dig : sec + (d0 + e) * R + dig;
  }
}

template <int F>
__device__ __forceinline__ double prod(const double* row, const int (&off)[F]) {
  double v = row[off[0]];
#pragma unroll
  for (int f = 1; f < F; ++f) v = __dmul_rn(v, row[off[f]]);
  return v;
}

// One CTA: K tile T over rows [r0, r1), plus t pairs T + ntiles (warp + 16 j), j < JT.  FA = q,
// FB = p - q factors per side.
template <int FA, int FB, int JT, int BW>
__device__ __forceinline__ void tile_body(const double* __restrict__ X, const double* __restrict__ y, double c,
                                          const BasisView& b, const TPlan& pl, int T, int64_t r0, int64_t r1,
                                          double* __restrict__ part, double* slab, bool& bad_x) {
  const Tile tl = pl.tiles[T];
  const int bw = BW ? BW : pl.bw;  // compile-time row stride where known (C4: 116, C5: 100): the
                                   // k-loop's operand addresses become register + immediate
  const int p = pl.p, M = pl.M, L = pl.L;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int wa, wb;
  warp_tile(warp, wa, wb);
  const int nva = tmax(0, tmin(kWF, tl.na - kWF * wa)), nvb = tmax(0, tmin(kWF, tl.nb - kWF * wb));
  int offA[kWF][FA], offB[kWF][FB];
#pragma unroll
  for (int j = 0; j < kWF; ++j) {
    const int64_t ca = int64_t(tl.a0 + kWF * wa + j) * 8 + (lane >> 2);
    const int64_t cb = int64_t(tl.b0 + kWF * wb + j) * 8 + (lane >> 2);
    col_offs<FA>(j < nva ? ca : pl.LA, pl.LA, 0, L, pl.goff, -1, pl, offA[j]);
    col_offs<FB>(j < nvb ? cb : pl.LB, pl.LB, pl.q, L, pl.goff, -1, pl, offB[j]);
  }
  double acc[kWF][kWF][2];
#pragma unroll
  for (int j = 0; j < kWF; ++j)
#pragma unroll
    for (int k = 0; k < kWF; ++k) acc[j][k][0] = acc[j][k][1] = 0.0;
  // t pairs of this warp: pi = T + ntiles (warp + 16 j) -> fragments (pi / tfb, pi % tfb)
  // (offsets byte-packed: A factors in bytes [0, FA), B factors in [FA, FA + FB) of tpk[j][.])
  unsigned tpk[JT][2];
  bool tval[JT];
  double accT[JT][2];
#pragma unroll
  for (int j = 0; j < JT; ++j) {
    const int pi = T + pl.ntiles * (warp + kW * j);
    tval[j] = pi < pl.tpairs;
    const int fa = tval[j] ? pi / pl.tfb : 0, fb = tval[j] ? pi % pl.tfb : 0;
    const int64_t ca = int64_t(fa) * 8 + (lane >> 2), cb = int64_t(fb) * 8 + (lane >> 2);
    int oa[FA], ob[FB];
    col_offs<FA>(tval[j] ? ca : pl.MA, pl.MA, 0, M, pl.poff, -1, pl, oa);
    col_offs<FB>(tval[j] ? cb : pl.MB, pl.MB, pl.q, M, pl.poff, pl.rpoff, pl, ob);
    tpk[j][0] = tpk[j][1] = 0u;
#pragma unroll
    for (int f = 0; f < FA + FB; ++f) tpk[j][f >> 2] |= unsigned(f < FA ? oa[f] : ob[f - FA]) << (8 * (f & 3));
    accT[j][0] = accT[j][1] = 0.0;
  }
  auto tfac = [&](const double* row, int j, int f) { return row[(tpk[j][f >> 2] >> (8 * (f & 3))) & 0xffu]; };

  // production: items it = tid + u kNT (u < 2), row it / p, dimension it % p; idle items write
  // the spare row BR
  const int BR = pl.BR;
  int prow[2], pdim[2];
  bool pon[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int it = tid + u * kNT;
    pon[u] = it < BR * p;
    prow[u] = pon[u] ? it / p : BR;
    pdim[u] = pon[u] ? it - (it / p) * p : 0;
  }
  // the next block's x (BR p doubles) and y (BR) are staged by cp.async while this block is
  // contracted (no registers held across the k-loop)
  double* xs = slab + (BR + 1) * bw;  // [BR p]
  double* ys = xs + BR * p;              // [BR]
  auto load = [&](int64_t base) {
    const int64_t nr = tmin<int64_t>(BR, r1 - base);
    for (int e = tid; e < BR * p; e += kNT) {
      const bool ok = e < nr * p;
      cp_async_8z(xs + e, ok ? X + base * p + e : X, ok);
    }
    for (int e = tid; e < BR; e += kNT) {
      const bool ok = y != nullptr && e < nr;
      cp_async_8z(ys + e, ok ? y + base + e : X, ok);
    }
    cp_async_commit();
  };
  auto produce = [&](int64_t base) {
    cp_async_wait<0>();
    __syncthreads();
    // the two items one after the other (advancing them in lockstep needs more registers than the
    // 32 accumulators leave)
#pragma unroll 1
    for (int u = 0; u < 2; ++u) {
      if (!pon[u]) continue;
      const double px = xs[prow[u] * p + pdim[u]];
      const double py = (y != nullptr && pdim[u] == p - 1) ? ys[prow[u]] : c;
      double* row = slab + prow[u] * bw;
      const bool valid = base + prow[u] < r1;
      // the B side reads the last dimension only as r*phi: that task stores r*phi alone, the
      // others phi (scale 1)
      const bool last = pdim[u] == p - 1;
      double* oph = last ? row + pl.rpoff : row + pl.poff + pdim[u] * M;
      double* og = row + pl.goff + pdim[u] * L;
      if (pdim[u] == 0) {
        row[pl.one] = 1.0;
        row[pl.zero] = 0.0;
      }
      if (valid) {
        bad_x |= not_finite(px);
        // r = y - c (posterior.py:229)
        eval_phi_g_dim_u<true>(px, last ? __dsub_rn(py, c) : 1.0, b, pdim[u], pl.hc, oph, og, nullptr);
      } else {  // rows past the range contribute zero
        for (int k = 0; k < M; ++k) oph[k] = 0.0;
        for (int k = 0; k < L; ++k) og[k] = 0.0;
      }
    }
  };
  struct Ops {
    double a[kWF], b[kWF];
  };
  auto ops = [&](int i, Ops& o) {
    const double* row = slab + (i * 4 + (lane & 3)) * bw;
#pragma unroll
    for (int j = 0; j < kWF; ++j) o.a[j] = prod<FA>(row, offA[j]);
#pragma unroll
    for (int k = 0; k < kWF; ++k) o.b[k] = prod<FB>(row, offB[k]);
  };
  auto tstep = [&](int i) {
    const double* row = slab + (i * 4 + (lane & 3)) * bw;
#pragma unroll
    for (int j = 0; j < JT; ++j)
      if (tval[j]) {
        double a = tfac(row, j, 0), bv = tfac(row, j, FA);
#pragma unroll
        for (int f = 1; f < FA; ++f) a = __dmul_rn(a, tfac(row, j, f));
#pragma unroll
        for (int f = 1; f < FB; ++f) bv = __dmul_rn(bv, tfac(row, j, FA + f));
        dmma_8x8x4(accT[j][0], accT[j][1], a, bv);
      }
  };
  const bool full = !pl.masked || (nva == kWF && nvb == kWF);
  auto mma_full = [&](const Ops& o) {
#pragma unroll
    for (int j = 0; j < kWF; ++j)
#pragma unroll
      for (int k = 0; k < kWF; ++k) dmma_8x8x4(acc[j][k][0], acc[j][k][1], o.a[j], o.b[k]);
  };
  auto mma_part = [&](const Ops& o) {
#pragma unroll
    for (int j = 0; j < kWF; ++j)
#pragma unroll
      for (int k = 0; k < kWF; ++k)
        if (j < nva && k < nvb) dmma_8x8x4(acc[j][k][0], acc[j][k][1], o.a[j], o.b[k]);
  };

  const int64_t nrows = tmax<int64_t>(0, r1 - r0);
  const int64_t nblk = ceil_div(nrows, BR);
#ifdef FAGP_TILED_PROF
  long long tpr[3] = {0, 0, 0}, t0 = clock64();
#define TPROF(stmt) stmt
#else
#define TPROF(stmt)
#endif
  if (nblk > 0) load(r0);
  for (int64_t n = 0; n < nblk; ++n) {
    const int64_t base = r0 + n * BR;
    TPROF(long long ta = clock64());
    produce(base);
    __syncthreads();  // slab complete, staging buffer free
    if (n + 1 < nblk) load(base + BR);
    TPROF(long long tb = clock64(); tpr[0] += tb - ta);
    const int nks = int((tmin<int64_t>(BR, r1 - base) + 3) / 4);
    if (nva > 0 && nvb > 0) {
      if (full) {
#pragma unroll kTiledUnroll
        for (int i = 0; i < nks; ++i) {
          Ops o;
          ops(i, o);
          mma_full(o);
          tstep(i);
        }
      } else {
        for (int i = 0; i < nks; ++i) {
          Ops o;
          ops(i, o);
          mma_part(o);
          tstep(i);
        }
      }
    } else {
      for (int i = 0; i < nks; ++i) tstep(i);
    }
    TPROF(ta = clock64(); tpr[1] += ta - tb);
    __syncthreads();
    TPROF(tpr[2] += clock64() - ta);
  }
#ifdef FAGP_TILED_PROF
  if (pl.prof && tid == 0) {
    long long* q = pl.prof + 5 * blockIdx.x;
    q[1] = clock64() - t0;
    q[2] = tpr[0];
    q[3] = tpr[1];
    q[4] = tpr[2];
  }
#endif
#undef TPROF
  // partial tile: fragment (4 wa + j, 4 wb + k) at ((4 wa + j) * 16 + 4 wb + k) * 64, C-fragment order
#pragma unroll
  for (int j = 0; j < kWF; ++j)
#pragma unroll
    for (int k = 0; k < kWF; ++k) {
      const int f = (kWF * wa + j) * kTF + kWF * wb + k;
      *reinterpret_cast<double2*>(part + int64_t(f) * 64 + 2 * lane) = make_double2(acc[j][k][0], acc[j][k][1]);
    }
  // t pair slot warp + 16 j after the K tile
#pragma unroll
  for (int j = 0; j < JT; ++j)
    *reinterpret_cast<double2*>(part + int64_t(kTF * kTF + warp + kW * j) * 64 + 2 * lane) =
        make_double2(accT[j][0], accT[j][1]);
}

template <int FA, int FB, int JT, int BW>
__global__ void __launch_bounds__(kNT, 1)
tiled_gram_kernel(const double* __restrict__ X, const double* __restrict__ y, double c, BasisView b,
                  const __grid_constant__ TPlan pl, double* __restrict__ ws, uint32_t* flags) {
  extern __shared__ double slab[];  // [(BR + 1) * bw] row slab | [BR p] x | [BR] y staging
  const int cta = int(blockIdx.x);
  bool bad_x = false;
  if (pl.span) {  // this CTA's share of the tile-major work: one or two (tile, row range) segments
    int ts, te;
    int64_t rs, re;
    span_pos(pl, span_bound(pl, cta), ts, rs);
    span_pos(pl, span_bound(pl, cta + 1), te, re);
    bool any = false;
    for (int T = ts; T <= te; ++T) {
      const int64_t r0 = T == ts ? rs : 0, r1 = T == te ? re : pl.N;
      if (r0 >= r1) continue;
      if (any) __syncthreads();  // the previous segment's slab reads are done
      tile_body<FA, FB, JT, BW>(X, y, c, b, pl, T, r0, r1,
                                ws + int64_t(pl.sbase[T] + cta - pl.first[T]) * kPartial, slab, bad_x);
      if (pl.prof && threadIdx.x == 0 && !any) pl.prof[5 * cta] = T;
      any = true;
    }
  } else {
    int T = 0;
    while (T + 1 < pl.ntiles && cta >= pl.first[T + 1]) ++T;
    const int j = cta - pl.first[T], cnt = pl.cnt[T];
    const int64_t per = round_up(ceil_div(tmax<int64_t>(pl.N, 1), cnt), 4);
    const int64_t r0 = tmin<int64_t>(pl.N, int64_t(j) * per), r1 = tmin<int64_t>(pl.N, r0 + per);
    tile_body<FA, FB, JT, BW>(X, y, c, b, pl, T, r0, r1, ws + int64_t(cta) * kPartial, slab, bad_x);
    if (pl.prof && threadIdx.x == 0) pl.prof[5 * cta] = T;
  }
  if (bad_x) raise_flag(flags, FAGP_FLAG_X_NONFINITE);
}

// out[e] = sum over the CTAs of e's tile (in CTA order: deterministic) of the partial entry
__global__ void __launch_bounds__(256) reduce_kernel(const double* __restrict__ ws, const __grid_constant__ TPlan pl,
                                                     double* __restrict__ out, uint32_t* flags) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= pl.len) return;
  int64_t ca, cb, idx;
  int T;
  if (e < pl.Klen) {
    ca = e / pl.LB;
    cb = e - ca * pl.LB;
    // tile of fragment f on a side of F fragments in n even tiles: [i F / n, (i + 1) F / n)
    auto locate = [&](int f, int side, int& i, int& loc) {
      const int F = pl.fr[side], n = pl.nt[side];
      i = int(int64_t(f) * n / F);
      while (i + 1 < n && int64_t(i + 1) * F / n <= f) ++i;
      while (i > 0 && int64_t(i) * F / n > f) --i;
      loc = f - int(int64_t(i) * F / n);
    };
    int ta, tb, fa, fb;
    locate(int(ca / 8), 0, ta, fa);
    locate(int(cb / 8), 1, tb, fb);
    T = ta * pl.nt[1] + tb;
    idx = int64_t(fa * kTF + fb) * 64;
  } else {
    const int64_t q = e - pl.Klen;
    ca = q / pl.MB;
    cb = q - ca * pl.MB;
    const int pi = int(ca / 8) * pl.tfb + int(cb / 8);  // t pair -> tile pi % ntiles, slot pi / ntiles
    T = pi % pl.ntiles;
    idx = int64_t(kTF * kTF + pi / pl.ntiles) * 64;
  }
  idx += (ca % 8) * 8 + (cb % 8);
  const double* src = ws + int64_t(pl.sbase[T]) * kPartial + idx;
  const int n = pl.cnt[T];
  double s = 0.0;
  int i = 0;
  for (; i + 8 <= n; i += 8) {  // loads batched (an L2 round trip each otherwise), summed in order
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = src[int64_t(i + u) * kPartial];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; i < n; ++i) s += src[int64_t(i) * kPartial];
  out[e] = s;
  if (not_finite(s)) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
}

bool eligible(int64_t N, int p, int M) {
  if (const char* e = getenv("FAGP_GRAM_TILED"))
    if (e[0] == '0') return false;  // tuning / A-B knob: the table path instead
  TPlan pl;
  return make_tplan(N, p, M, pl);
}

size_t workspace(int64_t N, int p, int M) {
  TPlan pl;
  if (!make_tplan(N, p, M, pl)) return 0;
  return size_t(pl.nslots) * kPartial * sizeof(double);
}

template <int FA, int FB, int JT, int BW>
static int launch_bw(const double* X, const double* y, double c, const fagp_basis* b, const TPlan& pl, double* ws,
                  uint32_t* flags, cudaStream_t s) {
  const size_t smem = (size_t(pl.BR + 1) * pl.bw + size_t(pl.BR) * (pl.p + 1)) * sizeof(double);
  FAGP_CUDA_TRY(cudaFuncSetAttribute(tiled_gram_kernel<FA, FB, JT, BW>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  tiled_gram_kernel<FA, FB, JT, BW><<<pl.grid, kNT, smem, s>>>(X, y, c, view(b), pl, ws, flags);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

// BASELINE C4 (p 4, M 8: stride 116) and C5 (p 5, M 6: stride 100) get compile-time strides
template <int FA, int FB, int JT>
static int launch_jt(const double* X, const double* y, double c, const fagp_basis* b, const TPlan& pl, double* ws,
                     uint32_t* flags, cudaStream_t s) {
  if constexpr (FA == 2 && FB == 2 && JT == 1)
    if (pl.bw == 116) return launch_bw<FA, FB, JT, 116>(X, y, c, b, pl, ws, flags, s);
  if constexpr (FA == 2 && FB == 3 && JT == 1)
    if (pl.bw == 100) return launch_bw<FA, FB, JT, 100>(X, y, c, b, pl, ws, flags, s);
  return launch_bw<FA, FB, JT, 0>(X, y, c, b, pl, ws, flags, s);
}

template <int FA, int FB>
static int launch(const double* X, const double* y, double c, const fagp_basis* b, const TPlan& pl, double* ws,
                  uint32_t* flags, cudaStream_t s) {
  return pl.jt <= 1 ? launch_jt<FA, FB, 1>(X, y, c, b, pl, ws, flags, s) : launch_jt<FA, FB, kJT>(X, y, c, b, pl, ws, flags, s);
}

int gram(const double* X, const double* y, double c, int64_t N, const fagp_basis* b, double* out, void* ws,
         size_t ws_bytes, uint32_t* flags, cudaStream_t s) {
  TPlan pl;
  if (!make_tplan(N, b->p, b->M, pl)) return FAGP_EUNSUPPORTED;
#ifdef FAGP_TILED_PROF  // diagnostics build: per-CTA phase cycles printed to stderr
  FAGP_CUDA_TRY(cudaMalloc(&pl.prof, size_t(5) * pl.grid * sizeof(long long)));
#endif
  if (ws == nullptr || ws_bytes < size_t(pl.nslots) * kPartial * sizeof(double)) return FAGP_EWORKSPACE;
  double* w = static_cast<double*>(ws);
  int rc;
  const int key = pl.q * 10 + (pl.p - pl.q);
  switch (key) {
    case 11: rc = launch<1, 1>(X, y, c, b, pl, w, flags, s); break;
    case 12: rc = launch<1, 2>(X, y, c, b, pl, w, flags, s); break;
    case 22: rc = launch<2, 2>(X, y, c, b, pl, w, flags, s); break;
    case 23: rc = launch<2, 3>(X, y, c, b, pl, w, flags, s); break;
    case 33: rc = launch<3, 3>(X, y, c, b, pl, w, flags, s); break;
    case 34: rc = launch<3, 4>(X, y, c, b, pl, w, flags, s); break;
    case 44: rc = launch<4, 4>(X, y, c, b, pl, w, flags, s); break;
    default: rc = FAGP_EUNSUPPORTED;
  }
  if (rc) return rc;
  if (pl.prof) {
    std::vector<long long> h(size_t(5) * pl.grid);
    FAGP_CUDA_TRY(cudaStreamSynchronize(s));
    FAGP_CUDA_TRY(cudaMemcpy(h.data(), pl.prof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    for (int c = 0; c < pl.grid; ++c)
      fprintf(stderr, "tiled cta %3d tile %2d (0, %2d x %2d) total %lld produce %lld kloop %lld barrier %lld\n", c,
              int(h[5 * c]), pl.tiles[h[5 * c]].na, pl.tiles[h[5 * c]].nb, h[5 * c + 1],
              h[5 * c + 2], h[5 * c + 3], h[5 * c + 4]);
    cudaFree(pl.prof);
  }
  reduce_kernel<<<unsigned(ceil_div(pl.len, 256)), 256, 0, s>>>(w, pl, out, flags);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // namespace tiled
}  // namespace fagp
