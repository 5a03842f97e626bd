// Latency of one production task (phi + g of one (point, dimension), fused.cu's eval_phi_g_dim_u)
// in isolation: cycles per call for 384 busy threads of a 512-thread CTA, as in the Gram kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2403_12797_b200/csrc -I include -o tools/prod_probe tools/prod_probe.cu
#include <cstdio>
#include "eigfun.cuh"
using namespace fagp;

template <int MODE>
__global__ void __launch_bounds__(512) prod(const double* tab, HermCoef hc, double* out, long long* cyc) {
  __shared__ double slab[60 * 100];
  BasisView b{3, 10, 1000, tab};
  const int tid = threadIdx.x;
  const int prow = (tid / 3) % 60, pdim = tid % 3;
  double x = -0.9 + 1.8 * (tid + 0.5) / 512.0;
  long long t0 = clock64();
  for (int rep = 0; rep < 8; ++rep) {
    if (tid < 384) {
      double* row = slab + prow * 100;
      if (MODE == 0) eval_phi_g_dim_u(x, 0.5, b, pdim, hc, row + 57 + pdim * 10, row + pdim * 19, pdim == 2 ? row + 87 : nullptr);
      if (MODE == 1) row[pdim] = phi_exp(b, pdim, x);
      if (MODE == 2) {  // recurrences only (no exp)
        double h = x, hm = 1.0, acc = 0.0;
#pragma unroll
        for (int k = 1; k < 22; ++k) {
          const double hn = fma(__dmul_rn(x, hc.c1[k]), h, -__dmul_rn(hc.c2[k], hm));
          hm = h; h = hn; acc += hn;
        }
        row[pdim] = acc;
      }
    }
    x += 1e-3;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / 8;
  if (tid == 0) out[blockIdx.x] = slab[5];
}

int main() {
  double htab[3 * 3 + 30 + 55 * 19] = {0};
  for (int d = 0; d < 3; ++d) { htab[d] = 1.4953; htab[3 + d] = -0.618; htab[6 + d] = 1.2228; }
  double* tab; cudaMalloc(&tab, sizeof(htab)); cudaMemcpy(tab, htab, sizeof(htab), cudaMemcpyHostToDevice);
  double* out; cudaMalloc(&out, 1024 * 8);
  long long* cyc; cudaMalloc(&cyc, 1024 * 8);
  HermCoef hc = herm_coef_host();
  long long h[4];
  const char* names[] = {"phi+g (full task)", "exp only", "recurrence only (21 steps)"};
  for (int mode = 0; mode < 3; ++mode) {
    if (mode == 0) prod<0><<<4, 512>>>(tab, hc, out, cyc);
    if (mode == 1) prod<1><<<4, 512>>>(tab, hc, out, cyc);
    if (mode == 2) prod<2><<<4, 512>>>(tab, hc, out, cyc);
    cudaMemcpy(h, cyc, 4 * 8, cudaMemcpyDeviceToHost);
    printf("%-30s %lld cycles per call (CTA-wide, incl. __syncthreads)\n", names[mode], h[1]);
  }
  return 0;
}
