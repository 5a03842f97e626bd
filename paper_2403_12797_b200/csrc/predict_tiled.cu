// Output-tiled fused modal predict: mean and variance for the shapes the one-CTA fused predict
// (fused.cu) cannot hold (BASELINE C4: p 4, M 8, L^p = 50,625 variance modes; C5: p 5, M 6,
// 161,051), with the eigenfunctions evaluated on chip -- no basis table in HBM.
//
//   var_i  = sigma2 sum_kappa C''[kappa] prod_d g_{d,kappa_d}(x*_i)   (posterior.py:249-263, diagonal)
//   mean_i = c + sum_a w[a] prod_d phi_{d,a_d}(x*_i)                   (posterior.py:247)
//
// Both are bilinear forms per test row in the Khatri-Rao halves of the dimensions, A = dims
// [0, q), B = dims [q, p):  var_i = gA_i^T C'' gB_i,  mean_i - c = phiA_i^T W phiB_i.  Per tile
// (a range of B columns, and a chunk of the A side) a CTA runs the GEMM  Y = gA(rows) x C''(A, B)
// on the FP64 tensor cores -- rows on the m8n8k4 M side, the A modes as K, the tile's B columns
// as N -- and folds Y with gB(rows) in the epilogue into one partial per row; the partials of the
// tiles are summed per row in fixed tile order by reduce_kernel (deterministic).
//
// B200 mapping:
//  * 16 warps = 4 row groups (16 rows = 2 m-fragments) x 4 column groups (4 n-fragments); 64-row
//    blocks; the tile's operand slice C''(A chunk, 128 B columns) stays in shared memory in
//    fragment-major order for the whole launch (one conflict-free LDS.64 per B fragment).
//  * A operands generated in registers from the row slab (q - 1 DMULs per fragment), their slab
//    offsets per k-step from a small packed table; production of the row slab as in the Gram
//    (eigfun.cuh, one exponential shared by phi and g).
//  * Tiles are dealt to the CTAs by a per-row cost (k-steps + production / epilogue), rows split
//    evenly over a tile's CTAs.
#include <type_traits>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "eigfun.cuh"
#include "modal.cuh"

namespace fagp {
namespace ptiled {

constexpr int kW = 16, kNT = kW * 32;
constexpr int kRF = 2;     // m-fragments (8 rows) per warp
constexpr int kCF = 4;     // n-fragments (8 columns) per warp
constexpr int kBR = 4 * kRF * 8;   // rows per block (4 row groups): 64
constexpr int kTN = 4 * kCF;       // n-fragments per tile (4 column groups): 16
constexpr int kMaxKS = 40;         // k-steps per tile (A chunk <= 160 modes)
constexpr int kMaxTiles = 64;
constexpr int kMaxF = 4;

struct Tile {
  int kind;        // 0: variance (g, C''), 1: mean (phi, w)
  int ka0, nka;    // A-side modes [ka0, ka0 + nka)
  int b0, nb;      // B-side n-fragments [b0, b0 + nb)
};

struct PPlan {
  int p, M, L, q;
  int64_t LA, LB, MA, MB;
  int goff, poff, one, zero, bw;
  int ntiles, nvar;
  Tile tiles[kMaxTiles];
  int first[kMaxTiles], cnt[kMaxTiles];
  int grid;
  int64_t Ns;
  // predict operand layout (modal::build_predict_op): C''[kappa] at op[kK * NP + kN], kN = dims
  // [0, pN), kK = dims [pN, p); w at op + KP * NP (dim 0 slowest)
  int pN;
  int64_t NRL, NP, KP;  // L^(p - pN) (the kK radix span), padded strides
  HermCoef hc;
  long long* prof;  // diagnostics build (-DFAGP_PTILED_PROF): per CTA [tile, cycles]
};

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

static bool make_pplan(int64_t Ns, int p, int M, PPlan& pl) {
  std::memset(&pl, 0, sizeof(pl));
  if (!modal_on(p, M) || M > kHermMax / 2 || p < 2) return false;
  pl.p = p;
  pl.M = M;
  pl.L = modal_L(M);
  pl.q = p / 2;
  if (pl.q > kMaxF || p - pl.q > kMaxF) return false;
  pl.LA = ipow(pl.L, pl.q);
  pl.LB = ipow(pl.L, p - pl.q);
  pl.MA = ipow(M, pl.q);
  pl.MB = ipow(M, p - pl.q);
  pl.Ns = Ns;
  pl.goff = 0;
  pl.poff = p * pl.L;
  pl.one = pl.poff + p * M;
  pl.zero = pl.one + 1;
  int w = pl.zero + 1;
  while (w % 16 != 4) ++w;
  pl.bw = w;
  if (pl.bw > 255) return false;  // byte-packed offsets
  const modal::Plan mp = modal::make_plan(0, p, M);
  pl.pN = mp.pN;
  pl.NRL = ipow(pl.L, p - mp.pN);
  pl.NP = mp.NP;
  pl.KP = mp.KP;
  // tiles: A side in chunks of <= 4 kMaxKS modes, B side in 16-fragment tiles (both split evenly)
  auto add = [&](int kind, int64_t ca, int64_t cb) -> bool {
    const int nka = int(ceil_div(ca, 4 * kMaxKS));
    const int fb = int(ceil_div(cb, 8)), ntb = int(ceil_div(fb, kTN));
    for (int a = 0; a < nka; ++a)
      for (int t = 0; t < ntb; ++t) {
        if (pl.ntiles >= kMaxTiles) return false;
        Tile& tl = pl.tiles[pl.ntiles++];
        tl.kind = kind;
        tl.ka0 = int(a * ca / nka);
        tl.nka = int((a + 1) * ca / nka) - tl.ka0;
        tl.b0 = t * fb / ntb;
        tl.nb = (t + 1) * fb / ntb - tl.b0;
      }
    return true;
  };
  if (!add(0, pl.LA, pl.LB)) return false;
  pl.nvar = pl.ntiles;
  if (!add(1, pl.MA, pl.MB)) return false;
  // per-row cost of a tile: its k-steps on the busiest sub-partition + production / epilogue
  // calibrated with -DFAGP_PTILED_PROF (per-CTA cycles) at C4 and C5: a k-step costs in proportion
  // to the busiest column group's n-fragments and to the share of column groups with any work (the
  // others' warps idle), plus a per-row production / epilogue term worth ~9 full k-steps (the old
  // model's 120 under-weighted it: C5's two mean tiles got 5 CTAs each and ran 9% past the
  // variance tiles)
  auto cost = [&](const Tile& t) {
    const int ks = int(ceil_div(t.nka, 4));
    const int cols = tmin(kCF, t.nb);                       // n-fragments of the busiest column group
    const int groups = tmin(4, int(ceil_div(t.nb, kCF)));   // column groups with work
    return double(ks) * (8.0 * cols + 6.0) * groups / 4.0 + 355.0;
  };
  const int G = tmax(num_sms(), pl.ntiles);
  for (int t = 0; t < pl.ntiles; ++t) pl.cnt[t] = 1;
  const int64_t cap = tmax<int64_t>(1, ceil_div(tmax<int64_t>(Ns, 1), kBR));
  for (int g = pl.ntiles; g < G; ++g) {
    int best = -1;
    double bv = -1.0;
    for (int t = 0; t < pl.ntiles; ++t) {
      if (pl.cnt[t] >= cap) continue;
      const double v = cost(pl.tiles[t]) / pl.cnt[t];
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
    f += pl.cnt[t];
  }
  pl.grid = f;
  pl.hc = herm_coef_host();
  return true;
}

static size_t smem_bytes(const PPlan& pl) {
  return (size_t(kMaxKS) * kTN * 32 + size_t(kBR + 2) * pl.bw + size_t(kBR) * pl.p + 2 * 4 * kBR) * sizeof(double) +
         size_t(kMaxKS) * 4 * sizeof(uint32_t);
}

__device__ __forceinline__ void cp_async_8z(void* smem, const void* gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0));
}

// column c of a side (F digits in radix R, first slowest) -> packed slab offsets (byte f = factor
// f); invalid -> (0, 1, ...)
template <int F>
__device__ __forceinline__ uint32_t pack_offs(int64_t c, int64_t ncols, int d0, int R, int sec, const PPlan& pl) {
  uint32_t pk = 0;
  if (c >= ncols) {
    pk = uint32_t(pl.zero);
#pragma unroll
    for (int f = 1; f < F; ++f) pk |= uint32_t(pl.one) << (8 * f);
    return pk;
  }
#pragma unroll
  for (int e = F - 1; e >= 0; --e) {
    const int dig = int(c % R);
    c /= R;
    pk |= uint32_t(sec + (d0 + e) * R + dig) << (8 * e);
  }
  return pk;
}

template <int F>
__device__ __forceinline__ double prod_pk(const double* row, uint32_t pk) {
  double v = row[pk & 0xffu];
#pragma unroll
  for (int f = 1; f < F; ++f) v = __dmul_rn(v, row[(pk >> (8 * f)) & 0xffu]);
  return v;
}

// G independent warp groups: G = 2 runs two 8-warp halves (2 row groups x 4 column groups each) on
// alternating 32-row blocks of the CTA's rows, each with its own slab, staging and reduction
// buffers and named barrier, so one group's production and epilogue overlap the other's DMMAs.
template <int FA, int FB, int BW, int G = 1>
__global__ void __launch_bounds__(kNT, 1)
tiled_predict_kernel(const double* __restrict__ Xs, BasisView b, const __grid_constant__ PPlan pl,
                     const double* __restrict__ op, double* __restrict__ part, uint32_t* flags) {
  extern __shared__ double sm[];
  const int bw = BW ? BW : pl.bw;
  constexpr int GT = kNT / G, RB = kBR / G, NRG = 4 / G;  // threads, rows, row groups per group
  double* Bt = sm;                              // [kMaxKS][kTN][32] fragment-major operand slice
  double* slab0 = Bt + kMaxKS * kTN * 32;       // [G][(RB + 1) * bw]
  double* xs0 = slab0 + (kBR + 2) * bw;         // [G][RB p] staged x of the group's next block
  double* red0 = xs0 + kBR * pl.p;              // [G][2][4][RB] column-group partials, double buffered
  uint32_t* offA = reinterpret_cast<uint32_t*>(red0 + 2 * 4 * kBR);  // [kMaxKS * 4]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = warp / (kW / G), gw = warp % (kW / G), gt = tid % GT;
  double* const slab = slab0 + gid * (RB + 1) * bw;
  double* const xs = xs0 + gid * RB * pl.p;
  double* const red = red0 + gid * 2 * 4 * RB;
  auto gsync = [&]() {
    if constexpr (G == 1)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(1 + gid), "r"(GT) : "memory");
  };
  const int p = pl.p, M = pl.M, L = pl.L;
  const int cta = int(blockIdx.x);
#ifdef FAGP_PTILED_PROF
  const long long t_start = clock64();
#endif
  int T = 0;
  while (T + 1 < pl.ntiles && cta >= pl.first[T + 1]) ++T;
  const Tile tl = pl.tiles[T];
  const bool var = tl.kind == 0;
  const int64_t per = round_up(ceil_div(tmax<int64_t>(pl.Ns, 1), pl.cnt[T]), 4);
  const int64_t r0 = tmin<int64_t>(pl.Ns, int64_t(cta - pl.first[T]) * per), r1 = tmin<int64_t>(pl.Ns, r0 + per);
  const int nks = int(ceil_div(tl.nka, 4));
  const int64_t nB = var ? pl.LB : pl.MB, nA = var ? pl.LA : pl.MA;
  const int R = var ? L : M, sec = var ? pl.goff : pl.poff;

  // the tile's operand slice: Bt[ks][nf][lane] = Op[kA = ka0 + 4 ks + (lane & 3)][kB = (b0 + nf) 8 + (lane >> 2)]
  for (int i = tid; i < nks * kTN * 32; i += kNT) {
    const int ln = i & 31, q = i >> 5, nf = q % kTN, ks = q / kTN;
    const int64_t kA = tl.ka0 + 4 * ks + (ln & 3), kB = int64_t(tl.b0 + nf) * 8 + (ln >> 2);
    double v = 0.0;
    if (4 * ks + (ln & 3) < tl.nka && nf < tl.nb && kB < nB) {
      if (var) {
        const int64_t kap = kA * pl.LB + kB;  // dim 0 slowest
        const int64_t kN = kap / pl.NRL, kK = kap - kN * pl.NRL;
        v = op[kK * pl.NP + kN];
      } else {
        v = op[pl.KP * pl.NP + kA * pl.MB + kB];
      }
    }
    Bt[i] = v;
  }
  // A-side slab offsets per (k-step, lane & 3)
  for (int i = tid; i < nks * 4; i += kNT) {
    const int64_t kA = tl.ka0 + i;
    offA[i] = pack_offs<FA>(i < tl.nka ? kA : nA, nA, 0, R, sec, pl);
  }
  // B-side offsets of this thread's epilogue columns: n-fragment cg * 4 + j, column 2 (lane & 3) + e
  // G = 1: SMSP = warp % 4 = row group, one warp of each column group per SMSP; G = 2: each SMSP
  // holds two warps of each group
  const int rg = gw % NRG, cg = gw / NRG;
  uint32_t offB[kCF][2];
#pragma unroll
  for (int j = 0; j < kCF; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int nf = cg * kCF + j;
      const int64_t kB = int64_t(tl.b0 + nf) * 8 + 2 * (lane & 3) + e;
      offB[j][e] = pack_offs<FB>((nf < tl.nb) ? kB : nB, nB, pl.q, R, sec, pl);
    }
  const bool active = cg * kCF < tl.nb;  // warps beyond the tile's columns skip the GEMM

  // production (two (row, dimension) items per thread, one after the other): phi and g
  int prow[2], pdim[2];
  bool pon[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int it = gt + u * GT;
    pon[u] = it < RB * p;
    prow[u] = pon[u] ? it / p : RB;
    pdim[u] = pon[u] ? it - (it / p) * p : 0;
  }
  bool bad_x = false;
  auto load = [&](int64_t base) {
    const int64_t nr = tmin<int64_t>(RB, r1 - base);
    for (int e = gt; e < RB * p; e += GT) {
      const bool ok = e < nr * p;
      cp_async_8z(xs + e, ok ? Xs + base * p + e : Xs, ok);
    }
    cp_async_commit();
  };
  auto produce = [&](int64_t base) {
    cp_async_wait<0>();
    gsync();
#pragma unroll 1
    for (int u = 0; u < 2; ++u) {
      if (!pon[u]) continue;
      double* row = slab + prow[u] * bw;
      const bool valid = base + prow[u] < r1;
      const double x = valid ? xs[prow[u] * p + pdim[u]] : 0.0;
      if (valid) bad_x |= not_finite(x);
      eval_phi_g_dim_u(x, 0.0, b, pdim[u], pl.hc, row + pl.poff + pdim[u] * M, row + pl.goff + pdim[u] * L, nullptr);
      if (pdim[u] == 0) {
        row[pl.one] = 1.0;
        row[pl.zero] = 0.0;
      }
    }
  };

  const int64_t nblk = ceil_div(tmax<int64_t>(0, r1 - r0), RB);
  if (gid < nblk) load(r0 + gid * RB);
  // stagger (G = 2): group 1 starts once group 0 has produced its first block
  bool staggered = G == 1 || gid == 1;
  if constexpr (G == 2)
    if (gid == 1) asm volatile("bar.sync 3, %0;" ::"r"(kNT) : "memory");
  int it = 0;
  for (int64_t n = gid; n < nblk; n += G, ++it) {
    const int64_t base = r0 + n * RB;
    produce(base);
    gsync();  // slab complete, staging free
    if constexpr (G == 2)
      if (!staggered) {
        asm volatile("bar.arrive 3, %0;" ::"r"(kNT) : "memory");
        staggered = true;
      }
    if (n + G < nblk) load(base + G * RB);
    double s[kRF] = {0.0, 0.0};
    if (active) {
      double acc[kRF][kCF][2];
#pragma unroll
      for (int f = 0; f < kRF; ++f)
#pragma unroll
        for (int j = 0; j < kCF; ++j) acc[f][j][0] = acc[f][j][1] = 0.0;
      const double* rowA = slab + (rg * 16 + (lane >> 2)) * bw;  // m-fragment f: + 8 f rows
      const double* Bw = Bt + (cg * kCF) * 32 + lane;
      auto kstep = [&](int ks) {
        const uint32_t pk = offA[4 * ks + (lane & 3)];
        double a[kRF], bb[kCF];
#pragma unroll
        for (int f = 0; f < kRF; ++f) a[f] = prod_pk<FA>(rowA + 8 * f * bw, pk);
#pragma unroll
        for (int j = 0; j < kCF; ++j) bb[j] = Bw[(ks * kTN + j) * 32];
#pragma unroll
        for (int f = 0; f < kRF; ++f)
#pragma unroll
          for (int j = 0; j < kCF; ++j) dmma_8x8x4(acc[f][j][0], acc[f][j][1], a[f], bb[j]);
      };
#pragma unroll 4
      for (int ks = 0; ks < nks; ++ks) kstep(ks);
      // epilogue: Y[row][col] * prod_{d >= q} (g | phi)_d[row][col digits], summed over the columns
#pragma unroll
      for (int f = 0; f < kRF; ++f) {
        const double* row = slab + (rg * 16 + 8 * f + (lane >> 2)) * bw;
#pragma unroll
        for (int j = 0; j < kCF; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) s[f] = fma(acc[f][j][e], prod_pk<FB>(row, offB[j][e]), s[f]);
      }
    }
#pragma unroll
    for (int f = 0; f < kRF; ++f) {
      s[f] += __shfl_xor_sync(0xffffffffu, s[f], 1);
      s[f] += __shfl_xor_sync(0xffffffffu, s[f], 2);
    }
    double* rb = red + (it & 1) * 4 * RB;
    if ((lane & 3) == 0)
#pragma unroll
      for (int f = 0; f < kRF; ++f) rb[cg * RB + rg * 16 + 8 * f + (lane >> 2)] = s[f];
    gsync();
    if (gt < RB && base + gt < r1) {
      const double v = ((rb[gt] + rb[RB + gt]) + rb[2 * RB + gt]) + rb[3 * RB + gt];
      part[int64_t(T) * pl.Ns + base + gt] = v;
    }
  }
  if constexpr (G == 2)
    if (!staggered) asm volatile("bar.arrive 3, %0;" ::"r"(kNT) : "memory");  // group 0 had no block
#ifdef FAGP_PTILED_PROF
  if (pl.prof && tid == 0) {
    pl.prof[2 * cta] = T;
    pl.prof[2 * cta + 1] = clock64() - t_start;
  }
#endif
  if (bad_x) raise_flag(flags, FAGP_FLAG_X_NONFINITE);
}

// mean_i = c + sum of the mean tiles' partials, var_i = sigma2 * sum of the variance tiles'
// partials (tile order: deterministic)
__global__ void reduce_kernel(const double* __restrict__ part, const __grid_constant__ PPlan pl, double sigma2,
                              double c, double* __restrict__ mean, double* __restrict__ var, uint32_t* flags) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= pl.Ns) return;
  double v = 0.0, m = 0.0;
  for (int t = 0; t < pl.nvar; ++t) v += part[int64_t(t) * pl.Ns + i];
  for (int t = pl.nvar; t < pl.ntiles; ++t) m += part[int64_t(t) * pl.Ns + i];
  const double mm = c + m;  // posterior.py:247
  mean[i] = mm;
  bool bad = not_finite(mm);
  if (var) {
    const double vv = sigma2 * v;
    var[i] = vv;
    bad |= not_finite(vv);
  }
  if (bad) raise_flag(flags, FAGP_FLAG_PHI_NONFINITE);
}

bool eligible(int p, int M) {
  if (const char* e = getenv("FAGP_PREDICT_TILED"))
    if (e[0] == '0') return false;  // A/B knob: the table path instead
  PPlan pl;
  return make_pplan(1, p, M, pl) && smem_bytes(pl) <= 227 * 1024;
}

size_t workspace(int64_t Ns, int p, int M) {
  PPlan pl;
  if (!make_pplan(Ns, p, M, pl)) return 0;
  return size_t(pl.ntiles) * size_t(tmax<int64_t>(Ns, 1)) * sizeof(double);
}

template <int FA, int FB, int BW>
static int launch_bw(const double* Xs, const fagp_basis* b, const PPlan& pl, const double* op, double* part,
                     uint32_t* flags, cudaStream_t s) {
  const size_t smem = smem_bytes(pl);
  const char* sg = getenv("FAGP_PREDICT_GROUPS");
  // two groups where the epilogue is light (FB <= 2: C4 5.26 -> 5.10 ms); at FB = 3 (C5) the
  // 32-row blocks' heavier epilogue and production cost more than the overlap buys (32.6 -> 34.3 ms)
  const bool g2 = FB <= 2 && !(sg && sg[0] == '1');
  auto kern = g2 ? tiled_predict_kernel<FA, FB, BW, 2> : tiled_predict_kernel<FA, FB, BW, 1>;
  FAGP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
#ifdef FAGP_PTILED_PROF
  PPlan pp = pl;
  FAGP_CUDA_TRY(cudaMalloc(&pp.prof, size_t(2) * pl.grid * sizeof(long long)));
  kern<<<pl.grid, kNT, smem, s>>>(Xs, view(b), pp, op, part, flags);
  {
    std::vector<long long> h(size_t(2) * pl.grid);
    FAGP_CUDA_TRY(cudaStreamSynchronize(s));
    FAGP_CUDA_TRY(cudaMemcpy(h.data(), pp.prof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    for (int c = 0; c < pl.grid; ++c)
      fprintf(stderr, "ptiled cta %3d tile %2lld kind %d nka %3d nb %2d cnt %3d cycles %lld\n", c, h[2 * c],
              pl.tiles[h[2 * c]].kind, pl.tiles[h[2 * c]].nka, pl.tiles[h[2 * c]].nb, pl.cnt[h[2 * c]], h[2 * c + 1]);
    cudaFree(pp.prof);
  }
#else
  kern<<<pl.grid, kNT, smem, s>>>(Xs, view(b), pl, op, part, flags);
#endif
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

template <int FA, int FB>
static int launch(const double* Xs, const fagp_basis* b, const PPlan& pl, const double* op, double* part,
                  uint32_t* flags, cudaStream_t s) {
  if (pl.bw == 100) return launch_bw<FA, FB, 100>(Xs, b, pl, op, part, flags, s);  // C4, C5
  return launch_bw<FA, FB, 0>(Xs, b, pl, op, part, flags, s);
}

int predict(const double* Xs, int64_t Ns, const fagp_basis* b, const double* op, double sigma2, double c,
            double* mean, double* var, void* ws, size_t ws_bytes, uint32_t* flags, cudaStream_t s) {
  PPlan pl;
  if (!make_pplan(Ns, b->p, b->M, pl)) return FAGP_EUNSUPPORTED;
  if (Ns == 0) return FAGP_OK;
  if (ws == nullptr || ws_bytes < workspace(Ns, b->p, b->M)) return FAGP_EWORKSPACE;
  double* part = static_cast<double*>(ws);
  int rc;
  switch (pl.q * 10 + (pl.p - pl.q)) {
    case 11: rc = launch<1, 1>(Xs, b, pl, op, part, flags, s); break;
    case 12: rc = launch<1, 2>(Xs, b, pl, op, part, flags, s); break;
    case 22: rc = launch<2, 2>(Xs, b, pl, op, part, flags, s); break;
    case 23: rc = launch<2, 3>(Xs, b, pl, op, part, flags, s); break;
    case 33: rc = launch<3, 3>(Xs, b, pl, op, part, flags, s); break;
    case 34: rc = launch<3, 4>(Xs, b, pl, op, part, flags, s); break;
    case 44: rc = launch<4, 4>(Xs, b, pl, op, part, flags, s); break;
    default: rc = FAGP_EUNSUPPORTED;
  }
  if (rc) return rc;
  reduce_kernel<<<unsigned(ceil_div(Ns, 256)), 256, 0, s>>>(part, pl, sigma2, c, mean, var, flags);
  FAGP_LAUNCH_CHECK();
  return FAGP_OK;
}

}  // namespace ptiled
}  // namespace fagp
