// Does FP64 CUDA-core work (DMUL) steal FP64 tensor (DMMA) throughput on B200?
// Each warp issues, per iteration, 12 independent DMMA.8x8x4 and ND independent DMULs
// (4 warps per SM sub-partition).  Prints DMMA TF/s for ND = 0, 2, 4, 8, 12.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_mix_probe tools/dmma_mix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int ND>
__global__ void mix(double* out, int iters, double seed) {
  double acc0[12], acc1[12], m[ND > 0 ? ND : 1];
#pragma unroll
  for (int i = 0; i < 12; ++i) { acc0[i] = seed * i; acc1[i] = seed; }
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) m[i] = seed + i;
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9, f = 1.0000000001;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      dmma(acc0[i], acc1[i], a, b);
      if (i < ND) m[i] = __dmul_rn(m[i], f);
    }
#pragma unroll
    for (int i = 12; i < ND; ++i) m[i] = __dmul_rn(m[i], f);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 12; ++i) s += acc0[i] + acc1[i];
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) s += m[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int ND>
double run(int sms) {
  double* out;
  cudaMalloc(&out, 4096 * sizeof(double));
  const int iters = 4000, threads = 512;
  mix<ND><<<sms, threads>>>(out, 10, 1.0000001);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    mix<ND><<<sms, threads>>>(out, iters, 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFree(out);
  const double flops = double(sms) * threads / 32 * iters * 12 * 512.0;
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"dmma_tflops_vs_dmul_per_12_dmma\": {\"0\": %.3f, \"2\": %.3f, \"4\": %.3f, \"8\": %.3f, \"12\": %.3f, \"24\": %.3f}}\n",
         run<0>(sms), run<2>(sms), run<4>(sms), run<8>(sms), run<12>(sms), run<24>(sms));
  return 0;
}
