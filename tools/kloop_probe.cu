// Micro-benchmark of the fused Gram's inner k-loop (fused.cu) in isolation: operands gathered
// from a shared-memory row slab (stride 100 doubles), A = product of 2 slab values (DMUL), B =
// one slab value, JK x NFK + JT x NFT DMMAs per 4-row k-step; no global memory, no barriers.
// Prints executed DMMA TF/s per variant.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/kloop_probe tools/kloop_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

constexpr int BW = 100, ROWS = 32;

// CHAIN > 0: every 4th warp (one per sub-partition) also runs a dependent DMUL/DSUB chain of
// CHAIN steps per 16 k-steps (the eigenfunction recurrence's shape)
template <int JK, int NFK, int JT, int NFT, bool PRODUCT, int CHAIN>
__global__ void __launch_bounds__(512) kloop(double* out, int iters) {
  __shared__ double slab[ROWS * BW];
  for (int i = threadIdx.x; i < ROWS * BW; i += blockDim.x) slab[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int offA[JK + JT][2], offB[NFK + NFT];
  for (int j = 0; j < JK + JT; ++j) {
    offA[j][0] = (warp * 3 + j) % 19;
    offA[j][1] = 19 + (lane >> 2) + 8 * (j & 1);
  }
  for (int n = 0; n < NFK + NFT; ++n) offB[n] = 38 + 8 * n + (lane >> 2);
  double acc[JK * NFK + JT * NFT][2];
  for (int q = 0; q < JK * NFK + JT * NFT; ++q) acc[q][0] = acc[q][1] = 0.0;
  double h = 1.0 + 1e-9 * lane, hm = 1.0, z = 0.7 + 1e-9 * warp;
  for (int it = 0; it < iters; ++it) {
    if (CHAIN > 0 && (warp >> 2) == (it & 3)) {
      for (int q = 0; q < CHAIN; ++q) {
        const double hn = __dsub_rn(__dmul_rn(__dmul_rn(z, slab[q & 31]), h), __dmul_rn(slab[(q + 7) & 31], hm));
        hm = h;
        h = hn;
      }
    }
#pragma unroll 2
    for (int kk = 0; kk < ROWS / 4; ++kk) {
      const double* row = slab + (kk * 4 + (lane & 3)) * BW;
      double b[NFK + NFT];
#pragma unroll
      for (int n = 0; n < NFK + NFT; ++n) b[n] = row[offB[n]];
#pragma unroll
      for (int j = 0; j < JK + JT; ++j) {
        const double a = PRODUCT ? __dmul_rn(row[offA[j][0]], row[offA[j][1]]) : row[offA[j][1]];
        const int nf = j < JK ? NFK : NFT, base = j < JK ? j * NFK : JK * NFK + (j - JK) * NFT;
#pragma unroll
        for (int n = 0; n < (j < JK ? NFK : NFT); ++n) dmma(acc[base + n][0], acc[base + n][1], a, b[j < JK ? n : NFK + n]);
      }
    }
  }
  double s = h;
  for (int q = 0; q < JK * NFK + JT * NFT; ++q) s += acc[q][0] + acc[q][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int JK, int NFK, int JT, int NFT, bool PRODUCT, int CHAIN = 0>
void run(const char* name, int warps, int ctas_per_sm, int sms) {
  double* out;
  cudaMalloc(&out, 8192 * sizeof(double));
  const int iters = 2000, grid = sms * ctas_per_sm, threads = warps * 32;
  auto k = kloop<JK, NFK, JT, NFT, PRODUCT, CHAIN>;
  k<<<grid, threads>>>(out, 2);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    k<<<grid, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double dmmas = double(grid) * warps * iters * (ROWS / 4) * (JK * NFK + JT * NFT);
  printf("%-40s warps/SM %2d : %6.2f TF/s executed\n", name, warps * ctas_per_sm, dmmas * 512 / (best * 1e-3) / 1e12);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("  error %s\n", cudaGetErrorString(e));
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<3, 3, 1, 2, true>("gram C3 (3x3 + 1x2, DMUL A)", 16, 1, sms);
  run<3, 3, 1, 2, true, 30>("+ 30-step dependent chain / 8 k-steps", 16, 1, sms);
  run<3, 3, 1, 2, true, 60>("+ 60-step dependent chain / 8 k-steps", 16, 1, sms);
  run<3, 3, 1, 2, true, 120>("+ 120-step dependent chain / 8 k-steps", 16, 1, sms);
  return 0;
}
