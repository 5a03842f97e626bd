// Per-point 1-D eigenfunction evaluation shared by the table kernel (basis.cu) and the
// fused kernels that never write a table (fused.cu).  One call = one (point, dimension).
//
//   phi_{d,i}(x) = (sqrt_beta_d * exp((-delta2_d * x) * x)) * h_i((rho_d beta_d) * x)   mercer.py:276-281
//   h_0 = 1, h_1 = z sqrt2, h_{k+1} = (z * c1[k]) * h_k - c2[k] * h_{k-1}            mercer.py:122-143
//   g_{d,k}(x)   = (beta_d * exp(((2 * -delta2_d) * x) * x)) * h_k(sqrt2 * rho_d beta_d x)   (modal.cu)
//
// Every multiply/subtract is an explicit round-to-nearest op so nvcc cannot contract it into
// an FMA: phi matches numpy's evaluation order bit for bit except for exp().
#pragma once

#include <cmath>

#include "common.cuh"

namespace fagp {

// c1[k] = sqrt(2/(k+1)), c2[k] = sqrt(k/(k+1)) exactly as the reference computes them with
// Python floats (mercer.py:137-142); IEEE division and sqrt are correctly rounded.
__device__ __forceinline__ double herm_c1(int k) { return __dsqrt_rn(__ddiv_rn(2.0, double(k + 1))); }
__device__ __forceinline__ double herm_c2(int k) { return __dsqrt_rn(__ddiv_rn(double(k), double(k + 1))); }

constexpr double kSqrt2 = 1.4142135623730951;  // math.sqrt(2.0)

// out[i * stride] = phi_{d,i}(x), i < M
__device__ __forceinline__ void eval_phi_dim(double x, const BasisView& b, int d, const double* c1, const double* c2,
                                             double* out, int stride = 1) {
  const int M = b.M;
  const double zr = __dmul_rn(b.rho_beta()[d], x);
  const double env = __dmul_rn(b.sqrt_beta()[d], exp(__dmul_rn(__dmul_rn(b.neg_delta2()[d], x), x)));
  double hm1 = 1.0;
  out[0] = __dmul_rn(env, 1.0);
  if (M > 1) {
    double h = __dmul_rn(zr, kSqrt2);
    out[stride] = __dmul_rn(env, h);
    for (int k = 1; k < M - 1; ++k) {
      const double hn = __dsub_rn(__dmul_rn(__dmul_rn(zr, c1[k]), h), __dmul_rn(c2[k], hm1));
      out[(k + 1) * stride] = __dmul_rn(env, hn);
      hm1 = h;
      h = hn;
    }
  }
}

// out[k * stride] = g_{d,k}(x), k < L = 2M - 1 (the modal functions spanning phi_a phi_b).
// g is not a reference quantity (only its span is), so it is evaluated for speed at full
// accuracy: the Gaussian as the square of phi's own exponential, exp(-2 delta2 x^2) =
// exp((-delta2 x) x)^2, and the recurrence with one FMA on the dependency chain
// (h_{k+1} = fma(y c1_k, h_k, -(c2_k h_{k-1})), the c2 product is off the chain).
__device__ __forceinline__ double g_amp(const BasisView& b, int d, double e1) {
  const double sb = b.sqrt_beta()[d];
  return __dmul_rn(__dmul_rn(sb, sb), __dmul_rn(e1, e1));
}

__device__ __forceinline__ double phi_exp(const BasisView& b, int d, double x) {
  return exp(__dmul_rn(__dmul_rn(b.neg_delta2()[d], x), x));
}

__device__ __forceinline__ void eval_g_dim(double x, const BasisView& b, int d, const double* c1, const double* c2,
                                           double* out, int stride = 1) {
  const int L = modal_L(b.M);
  const double amp = g_amp(b, d, phi_exp(b, d, x));
  const double yz = __dmul_rn(__dmul_rn(b.rho_beta()[d], x), kSqrt2);
  double gm1 = 1.0;
  out[0] = amp;
  if (L > 1) {
    double h = __dmul_rn(yz, kSqrt2);
    out[stride] = __dmul_rn(amp, h);
    for (int k = 1; k < L - 1; ++k) {
      const double hn = fma(__dmul_rn(yz, c1[k]), h, -__dmul_rn(c2[k], gm1));
      out[(k + 1) * stride] = __dmul_rn(amp, hn);
      gm1 = h;
      h = hn;
    }
  }
}

// Recurrence coefficients c1[k] = sqrt(2/(k+1)), c2[k] = sqrt(k/(k+1)) computed on the host (IEEE
// division and sqrt are correctly rounded: the same bits as herm_c1/herm_c2) and passed in the
// kernel parameters, so a fully unrolled recurrence reads them as constant-bank operands: no
// shared-memory load on the dependency chain.
constexpr int kHermMax = 24;  // L = 2M - 1 <= 23 (M <= 12) on the fused path
struct HermCoef {
  double c1[kHermMax], c2[kHermMax];
};

inline HermCoef herm_coef_host() {
  HermCoef h{};
  for (int k = 0; k < kHermMax; ++k) {
    h.c1[k] = std::sqrt(2.0 / double(k + 1));
    h.c2[k] = std::sqrt(double(k) / double(k + 1));
  }
  return h;
}

// eval_phi_g_dim with the recurrence unrolled to kHermMax steps (guarded by M, L) and the
// coefficients from `hc` (kernel parameters); identical operations and results.  kScaled: out_phi
// receives r * phi and out_rphi is ignored (a caller reading only r*phi of a dimension stores that
// alone, with r = 1 for the others -- one store stream per task, no divergence).
template <bool kScaled = false>
__device__ __forceinline__ void eval_phi_g_dim_u(double x, double r, const BasisView& b, int d, const HermCoef& hc,
                                                 double* out_phi, double* out_g, double* out_rphi) {
  const int M = b.M, L = modal_L(M);
  const double zr = __dmul_rn(b.rho_beta()[d], x);
  const double e1 = phi_exp(b, d, x);
  const double env = __dmul_rn(b.sqrt_beta()[d], e1);
  const double amp = g_amp(b, d, e1);
  const double yz = __dmul_rn(zr, kSqrt2);
  double hp = __dmul_rn(zr, kSqrt2), hpm = 1.0;
  double hg = __dmul_rn(yz, kSqrt2), hgm = 1.0;
  auto put_phi = [&](int k, double h) {
    const double v = __dmul_rn(env, h);
    if constexpr (kScaled) {
      out_phi[k] = __dmul_rn(r, v);
    } else {
      out_phi[k] = v;
      if (out_rphi) out_rphi[k] = __dmul_rn(r, v);
    }
  };
  put_phi(0, 1.0);
  out_g[0] = amp;
  if (M > 1) put_phi(1, hp);
  if (L > 1) out_g[1] = __dmul_rn(amp, hg);
#pragma unroll
  for (int k = 1; k < kHermMax - 1; ++k) {
    if (k < L - 1) {
      const double hgn = fma(__dmul_rn(yz, hc.c1[k]), hg, -__dmul_rn(hc.c2[k], hgm));
      out_g[k + 1] = __dmul_rn(amp, hgn);
      hgm = hg;
      hg = hgn;
      if (k < M - 1) {
        const double hpn = __dsub_rn(__dmul_rn(__dmul_rn(zr, hc.c1[k]), hp), __dmul_rn(hc.c2[k], hpm));
        put_phi(k + 1, hpn);
        hpm = hp;
        hp = hpn;
      }
    }
  }
}

// eval_phi_g_dim_u for T independent (point, dimension) tasks advanced in lockstep (T chains
// per thread hide each other's FP64 latency); identical operations and results per task.
// out_phi[t] receives s[t] * phi (s = 1 leaves phi bit-identical; s = r gives the r*phi slot of
// the last dimension): one store stream per task, so the warp's tasks never diverge.
template <int T>
__device__ __forceinline__ void eval_phi_g_dim_uT(const double (&x)[T], const double (&s)[T], const BasisView& b,
                                                  const int (&d)[T], const HermCoef& hc, double* const (&out_phi)[T],
                                                  double* const (&out_g)[T]) {
  const int M = b.M, L = modal_L(M);
  double zr[T], env[T], amp[T], yz[T], hp[T], hpm[T], hg[T], hgm[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    zr[t] = __dmul_rn(b.rho_beta()[d[t]], x[t]);
    const double e1 = phi_exp(b, d[t], x[t]);
    env[t] = __dmul_rn(b.sqrt_beta()[d[t]], e1);
    amp[t] = g_amp(b, d[t], e1);
    yz[t] = __dmul_rn(zr[t], kSqrt2);
    hp[t] = __dmul_rn(zr[t], kSqrt2);
    hpm[t] = 1.0;
    hg[t] = __dmul_rn(yz[t], kSqrt2);
    hgm[t] = 1.0;
  }
  auto put_phi = [&](int t, int k, double h) {
    out_phi[t][k] = __dmul_rn(s[t], __dmul_rn(env[t], h));
  };
#pragma unroll
  for (int t = 0; t < T; ++t) {
    put_phi(t, 0, 1.0);
    out_g[t][0] = amp[t];
    if (M > 1) put_phi(t, 1, hp[t]);
    if (L > 1) out_g[t][1] = __dmul_rn(amp[t], hg[t]);
  }
#pragma unroll
  for (int k = 1; k < kHermMax - 1; ++k) {
    if (k < L - 1) {
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const double hgn = fma(__dmul_rn(yz[t], hc.c1[k]), hg[t], -__dmul_rn(hc.c2[k], hgm[t]));
        out_g[t][k + 1] = __dmul_rn(amp[t], hgn);
        hgm[t] = hg[t];
        hg[t] = hgn;
      }
      if (k < M - 1) {
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const double hpn = __dsub_rn(__dmul_rn(__dmul_rn(zr[t], hc.c1[k]), hp[t]), __dmul_rn(hc.c2[k], hpm[t]));
          put_phi(t, k + 1, hpn);
          hpm[t] = hp[t];
          hp[t] = hpn;
        }
      }
    }
  }
}

// phi (reference order, bit-faithful) and g of one (point, dimension) sharing the exponential,
// the two recurrences advanced in one loop (independent chains); rphi (nullable) <- r * phi.
__device__ __forceinline__ void eval_phi_g_dim(double x, double r, const BasisView& b, int d, const double* c1,
                                               const double* c2, double* out_phi, double* out_g, double* out_rphi) {
  const int M = b.M, L = modal_L(M);
  const double zr = __dmul_rn(b.rho_beta()[d], x);
  const double e1 = phi_exp(b, d, x);
  const double env = __dmul_rn(b.sqrt_beta()[d], e1);
  const double amp = g_amp(b, d, e1);
  const double yz = __dmul_rn(zr, kSqrt2);
  double hp = __dmul_rn(zr, kSqrt2), hpm = 1.0;  // phi chain: h_1, h_0
  double hg = __dmul_rn(yz, kSqrt2), hgm = 1.0;  // g chain
  auto put_phi = [&](int k, double h) {
    const double v = __dmul_rn(env, h);
    out_phi[k] = v;
    if (out_rphi) out_rphi[k] = __dmul_rn(r, v);
  };
  put_phi(0, 1.0);
  out_g[0] = amp;
  if (M > 1) put_phi(1, hp);
  if (L > 1) out_g[1] = __dmul_rn(amp, hg);
  for (int k = 1; k < L - 1; ++k) {
    const double a1 = c1[k], a2 = c2[k];
    const double hgn = fma(__dmul_rn(yz, a1), hg, -__dmul_rn(a2, hgm));
    out_g[k + 1] = __dmul_rn(amp, hgn);
    hgm = hg;
    hg = hgn;
    if (k < M - 1) {
      const double hpn = __dsub_rn(__dmul_rn(__dmul_rn(zr, a1), hp), __dmul_rn(a2, hpm));
      put_phi(k + 1, hpn);
      hpm = hp;
      hp = hpn;
    }
  }
}

}  // namespace fagp

namespace fagp {

// T independent (point, dimension) evaluations advanced in lockstep: the same operations in
// the same order as eval_phi_dim / eval_g_dim for each point (bit-identical results), but T
// independent recurrence chains per thread, so the FP64 latency of one chain hides behind
// the others.  out_phi[t] / out_g[t] may be null (skip that section for point t).
template <int T>
__device__ __forceinline__ void eval_multi(const double (&x)[T], const int (&d)[T], const BasisView& b,
                                           const double* c1, const double* c2, double* const (&out_phi)[T],
                                           double* const (&out_g)[T], bool want_phi, bool want_g) {
  const int M = b.M, L = modal_L(M);
  double zr[T];
#pragma unroll
  for (int t = 0; t < T; ++t) zr[t] = __dmul_rn(b.rho_beta()[d[t]], x[t]);
  double e1[T];
  if (want_phi) {
    double env[T], h[T], hm1[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      e1[t] = phi_exp(b, d[t], x[t]);
      env[t] = __dmul_rn(b.sqrt_beta()[d[t]], e1[t]);
      hm1[t] = 1.0;
      h[t] = __dmul_rn(zr[t], kSqrt2);
      if (out_phi[t]) {
        out_phi[t][0] = __dmul_rn(env[t], 1.0);
        if (M > 1) out_phi[t][1] = __dmul_rn(env[t], h[t]);
      }
    }
    for (int k = 1; k < M - 1; ++k) {
      const double a1 = c1[k], a2 = c2[k];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const double hn = __dsub_rn(__dmul_rn(__dmul_rn(zr[t], a1), h[t]), __dmul_rn(a2, hm1[t]));
        if (out_phi[t]) out_phi[t][k + 1] = __dmul_rn(env[t], hn);
        hm1[t] = h[t];
        h[t] = hn;
      }
    }
  }
  if (want_g) {
    double amp[T], yz[T], h[T], gm1[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      amp[t] = g_amp(b, d[t], want_phi ? e1[t] : phi_exp(b, d[t], x[t]));
      yz[t] = __dmul_rn(zr[t], kSqrt2);
      gm1[t] = 1.0;
      h[t] = __dmul_rn(yz[t], kSqrt2);
      if (out_g[t]) {
        out_g[t][0] = amp[t];
        if (L > 1) out_g[t][1] = __dmul_rn(amp[t], h[t]);
      }
    }
    for (int k = 1; k < L - 1; ++k) {
      const double a1 = c1[k], a2 = c2[k];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const double hn = fma(__dmul_rn(yz[t], a1), h[t], -__dmul_rn(a2, gm1[t]));
        if (out_g[t]) out_g[t][k + 1] = __dmul_rn(amp[t], hn);
        gm1[t] = h[t];
        h[t] = hn;
      }
    }
  }
}

}  // namespace fagp
