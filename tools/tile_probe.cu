// Micro-benchmark of gram_tiled.cu's inner k-step in isolation: 16 warps, each a 4 x 4 block of
// m8n8k4 DMMAs per 4-row k-step whose A / B operands are products of FA / FB values gathered
// from a shared-memory row slab (stride 100 doubles).  No global memory, no barriers.  Prints
// executed DMMA TF/s per (FA, FB) and operand mode.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tile_probe.cu -o tools/tile_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

constexpr int BW = 100, ROWS = 32;

// MODE 0: operands gathered from smem per k-step (the kernel's way); MODE 1: operands held in
// registers (pure DMMA issue, the ceiling); MODE 2: gathered, software-pipelined one k-step ahead
template <int FA, int FB, int MODE>
__global__ void __launch_bounds__(512, 1) tile(double* out, int iters) {
  __shared__ double slab[ROWS * BW];
  for (int i = threadIdx.x; i < ROWS * BW; i += blockDim.x) slab[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int offA[4][FA], offB[4][FB];
  for (int j = 0; j < 4; ++j) {
    const int c = (warp * 4 + j) * 8 + (lane >> 2);
    for (int f = 0; f < FA; ++f) offA[j][f] = f * 15 + (c + 3 * f) % 15;
    for (int f = 0; f < FB; ++f) offB[j][f] = 45 + f * 15 + (c + 5 * f) % 15;
  }
  double acc[4][4][2];
  for (int j = 0; j < 4; ++j)
    for (int k = 0; k < 4; ++k) acc[j][k][0] = acc[j][k][1] = 0.0;
  auto form = [&](const double* row, double (&a)[4], double (&b)[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double v = row[offA[j][0]];
#pragma unroll
      for (int f = 1; f < FA; ++f) v = __dmul_rn(v, row[offA[j][f]]);
      a[j] = v;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double v = row[offB[j][0]];
#pragma unroll
      for (int f = 1; f < FB; ++f) v = __dmul_rn(v, row[offB[j][f]]);
      b[j] = v;
    }
  };
  double a[4], b[4];
  form(slab + (lane & 3) * BW, a, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll 2
    for (int kk = 0; kk < ROWS / 4; ++kk) {
      const double* row = slab + (kk * 4 + (lane & 3)) * BW;
      if (MODE == 0) form(row, a, b);
      double an[4], bn[4];
      if (MODE == 2) form(slab + (((kk + 1) & (ROWS / 4 - 1)) * 4 + (lane & 3)) * BW, an, bn);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) dmma(acc[j][k][0], acc[j][k][1], a[j], b[k]);
      if (MODE == 2)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          a[j] = an[j];
          b[j] = bn[j];
        }
    }
  }
  double s = 0;
  for (int j = 0; j < 4; ++j)
    for (int k = 0; k < 4; ++k) s += acc[j][k][0] + acc[j][k][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int FA, int FB, int MODE>
void run(const char* name) {
  double* d;
  cudaMalloc(&d, 4096 * 8);
  const int iters = 2000;
  tile<FA, FB, MODE><<<148, 512>>>(d, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tile<FA, FB, MODE><<<148, 512>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmmas = 148.0 * 16 * 16 * (ROWS / 4) * double(iters);
  printf("%-28s %7.2f TF/s executed DMMA (%s)\n", name, dmmas * 512 / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<1, 1, 1>("registers only");
  run<1, 1, 0>("gather 1x1 (no DMUL)");
  run<2, 2, 0>("gather 2x2 (C4)");
  run<2, 3, 0>("gather 2x3 (C5)");
  run<2, 2, 2>("gather 2x2 pipelined");
  run<2, 3, 2>("gather 2x3 pipelined");
  run<1, 2, 0>("gather 1x2 (C3-like)");
  return 0;
}
