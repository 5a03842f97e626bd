// Throughput of the FP64 mma.sync shapes on sm_100a: m8n8k4 (1 DMMA) against the sm_90+ shapes
// m16n8k4 / m16n8k8 / m16n8k16 -- register-only loops, 8 independent accumulators per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dmma_shape_probe.cu -o tools/dmma_shape_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int SH>
__device__ __forceinline__ void mma(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  if constexpr (SH == 0) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b[0]));
  } else if constexpr (SH == 1) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  } else if constexpr (SH == 2) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]),
          "d"(b[1]));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
        "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
          "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
}

template <int SH>
__global__ void loop(double* out, int iters, double seed) {
  double c[8][4], a[8], b[4];
  for (int i = 0; i < 8; ++i) {
    a[i] = seed + i * 1e-9 + threadIdx.x * 1e-12;
    for (int j = 0; j < 4; ++j) c[i][j] = seed * j;
  }
  for (int j = 0; j < 4; ++j) b[j] = seed - j * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) mma<SH>(c[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int SH>
double run(int sms, int warps, int iters) {
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  loop<SH><<<sms, warps * 32>>>(out, iters, 1.0000001);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    loop<SH><<<sms, warps * 32>>>(out, iters, 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fma_per = SH == 0 ? 256 : SH == 1 ? 512 : SH == 2 ? 1024 : 2048;
  cudaFree(out);
  return double(sms) * warps * iters * 8 * fma_per * 2 / (best * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  for (int w : {4, 8, 16}) {
    printf("warps/SM %2d:", w);
    printf(" %s %.2f", names[0], run<0>(sms, w, 4000));
    printf(" %s %.2f", names[1], run<1>(sms, w, 2000));
    printf(" %s %.2f", names[2], run<2>(sms, w, 1000));
    printf(" %s %.2f TF\n", names[3], run<3>(sms, w, 500));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
