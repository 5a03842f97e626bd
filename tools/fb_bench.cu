// Latency of factor_block (chol.cu) on one CTA: nvcc ... -I include tools/fb_bench.cu -o tools/fb_bench
#include <cstdio>
#include "../paper_2403_12797_b200/csrc/chol.cu"
using namespace fagp::la;
__global__ void fb_kernel(double* A, double* diag, double* LiG, long long* cyc) {
  __shared__ double S[CB][CSP], Y[CB][CSP], rsv[CB + 8];
  const int tid = threadIdx.x;
  long long t0 = 0;
  for (int rep = 0; rep < 11; ++rep) {
    for (int e = tid; e < CB * CB; e += CNT) {
      const int i = e >> 5, k = e & 31;
      S[i][k] = (i == k ? 40.0 : 0.0) + 1.0 / (1.0 + i + k);
    }
    __syncthreads();
    if (rep == 1) t0 = clock64();
    factor_block(S, Y, rsv, 32, 0, A, 32, diag, LiG, tid);
    __syncthreads();
  }
  if (tid == 0) cyc[0] = (clock64() - t0) / 10;
}
__global__ void lat_kernel(double* out, long long* cyc, double x) {
  __shared__ double sm[256];
  const int tid = threadIdx.x;
  sm[tid] = x + tid;
  __syncthreads();
  long long t0 = clock64();
  double v = x;
  for (int i = 0; i < 1000; ++i) v = fma(v, 1.0000001, 0.5);
  long long t1 = clock64();
  for (int i = 0; i < 1000; ++i) __syncthreads();
  long long t2 = clock64();
  int idx = tid;
  for (int i = 0; i < 1000; ++i) idx = int(sm[idx & 127]) & 127;
  long long t3 = clock64();
  double r = x;
  for (int i = 0; i < 1000; ++i) r = rsqrt(r + 1.0);
  long long t4 = clock64();
  if (tid == 0) { cyc[0] = (t1 - t0); cyc[1] = (t2 - t1); cyc[2] = (t3 - t2); cyc[3] = t4 - t3; }
  out[tid] = v + idx + r;
}
int main() {
  {
    double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 32);
    lat_kernel<<<1, 128>>>(o, c, 1.0);
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("per-op cycles: dfma %.1f  syncthreads %.1f  lds-chain %.1f  rsqrt(+add) %.1f\n", h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0);
  }
  double *A, *d, *L; long long* c;
  cudaMalloc(&A, 32 * 32 * 8); cudaMalloc(&d, 32 * 8); cudaMalloc(&L, 32 * 32 * 8); cudaMalloc(&c, 8);
  fb_kernel<<<1, CNT>>>(A, d, L, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("factor_block: %lld cycles per call (%s)\n", h, cudaGetErrorString(cudaGetLastError()));
}
