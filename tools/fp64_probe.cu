// FP64 peak probe for B200 (sm_100a): verifies the mma.m8n8k4.f64 fragment layout
// and measures register-only DMMA and DFMA throughput. Used to fix the roofline
// denominator (MEASURED_PEAKS.json has no FP64 entry). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void layout_kernel(const double* A, const double* B, double* C) {
  int lane = threadIdx.x;
  double a = A[(lane >> 2) * 4 + (lane & 3)];   // A 8x4 row-major
  double b = B[(lane & 3) * 8 + (lane >> 2)];   // B 4x8 row-major
  double d0 = 0, d1 = 0;
  dmma(d0, d1, a, b);
  C[(lane >> 2) * 8 + (lane & 3) * 2 + 0] = d0;
  C[(lane >> 2) * 8 + (lane & 3) * 2 + 1] = d1;
}

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double acc0[NACC], acc1[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc0[i] = seed * i; acc1[i] = seed; }
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc0[i], acc1[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc0[i] + acc1[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = seed * i;
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename K>
double time_kernel(K kern, int blocks, int threads, int iters, double flops_per_iter_thread_or_warp, bool per_warp) {
  double* out; CK(cudaMalloc(&out, 1024 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters, 1.0000001); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters, 1.0000001);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double units = per_warp ? (double)blocks * threads / 32 : (double)blocks * threads;
  double tf = units * iters * flops_per_iter_thread_or_warp / (best * 1e-3) / 1e12;
  cudaFree(out);
  return tf;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d,\n", prop.name, prop.multiProcessorCount, clk);
  // layout check
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = (i * 7 % 13) - 6.0; hB[i] = (i * 5 % 11) - 5.0; }
  for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) { double s = 0; for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c]; ref[r * 8 + c] = s; }
  double *dA, *dB, *dC; CK(cudaMalloc(&dA, 256)); CK(cudaMalloc(&dB, 256)); CK(cudaMalloc(&dC, 512));
  CK(cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice));
  layout_kernel<<<1, 32>>>(dA, dB, dC); CK(cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost));
  int bad = 0; for (int i = 0; i < 64; ++i) bad += hC[i] != ref[i];
  printf(" \"dmma_layout_ok\": %s,\n", bad ? "false" : "true");
  int sms = prop.multiProcessorCount;
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      double tf = time_kernel(dmma_loop<8>, sms * bps, wpb * 32, iters, 8 * 512.0, true);
      printf(" \"dmma_tflops_w%d_b%d\": %.3f,\n", wpb, bps, tf);
    }
  }
  double tf16 = time_kernel(dmma_loop<16>, sms * 2, 256, iters, 16 * 512.0, true);
  printf(" \"dmma_tflops_acc16\": %.3f,\n", tf16);
  for (int wpb : {8, 16, 32}) {
    double tf = time_kernel(dfma_loop<8>, sms * 2, wpb * 32, iters, 8 * 2.0, false);
    printf(" \"dfma_tflops_w%d\": %.3f,\n", wpb, tf);
  }
  printf(" \"done\": true}\n");
  return 0;
}
