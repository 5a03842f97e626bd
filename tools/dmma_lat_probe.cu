// Dependent-chain latency of DMMA.8x8x4 on B200: one warp, C independent accumulator chains
// interleaved, N steps each; prints cycles per step of one chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_lat_probe tools/dmma_lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int C>
__global__ void chain(double* out, long long* cyc, int n, double seed) {
  double d0[C], d1[C];
#pragma unroll
  for (int c = 0; c < C; ++c) { d0[c] = seed * c; d1[c] = seed; }
  const double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  __syncwarp();
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) dmma(d0[c], d1[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += d0[c] + d1[c];
  const long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
void run() {
  double* out; long long* cyc;
  cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 8);
  const int n = 4096;
  chain<C><<<1, 32>>>(out, cyc, n, 1e-3);
  chain<C><<<1, 32>>>(out, cyc, n, 1e-3);
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("chains %2d: %6.1f cycles per DMMA step of one chain, %5.1f cycles per DMMA issued\n", C,
         double(h) / n, double(h) / n / C);
}

int main() {
  run<1>(); run<2>(); run<4>(); run<8>(); run<16>();
  return 0;
}
