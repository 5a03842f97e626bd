// Dependent-chain latencies on this GPU (one warp, clock64): DFMA, DMUL, MUFU.RCP64H + Newton
// (rcp_nr), rsqrt(double), SHFL of a double, STS -> __syncwarp -> LDS round trip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/lat_probe.cu -o tools/lat_probe
#include <cstdio>

__device__ __forceinline__ double rcp_nr(double p) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
  double e = fma(-p, r, 1.0);
  r = fma(r, e, r);
  e = fma(-p, r, 1.0);
  return fma(r, e, r);
}

__device__ double* g_sink;
__device__ __forceinline__ long long clk(double dep) {
  if (dep == -1.2345) *g_sink = dep;  // forces dep before the clock read (branch)
  __syncwarp();
  return clock64();
}
__global__ void lat(double seed, long long* out, double* sink) {
  __shared__ double buf[64];
  const int lane = threadIdx.x;
  double x = seed + lane * 1e-3;
  constexpr int N = 256;
  long long t0, t1;
  // DFMA chain
  t0 = clk(x);
#pragma unroll 16
  for (int i = 0; i < N; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(0.999), "d"(1e-3));
  t1 = clk(x);
  out[0] = (t1 - t0) / N;
  // DMUL chain
  t0 = clk(x);
#pragma unroll 16
  for (int i = 0; i < N; ++i) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(1.0000001));
  t1 = clk(x);
  out[1] = (t1 - t0) / N;
  // rcp approx alone
  t0 = clk(x);
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    x = r;
  }
  t1 = clk(x);
  out[2] = (t1 - t0) / N;
  // rcp_nr chain
  t0 = clk(x);
#pragma unroll 16
  for (int i = 0; i < N; ++i) { x = rcp_nr(x); asm volatile("" : "+d"(x)); }
  t1 = clk(x);
  out[3] = (t1 - t0) / N;
  // rsqrt chain
  x = 2.0 + lane;
  t0 = clk(x);
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = rsqrt(x) + 1.5;
  t1 = clk(x);
  out[4] = (t1 - t0) / N;
  // shfl of a double chain
  t0 = clk(x);
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31);
  t1 = clk(x);
  out[5] = (t1 - t0) / N;
  // STS -> syncwarp -> LDS chain
  t0 = clk(x);
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    buf[lane] = x;
    __syncwarp();
    x = buf[(lane + 1) & 31];
    __syncwarp();
  }
  t1 = clk(x);
  out[6] = (t1 - t0) / N;
  // DSETP + FSEL-dependent (pivot test) chain: x = x > 0 ? x * c : x
  t0 = clk(x);
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x > 0.0 ? fma(x, 0.5, 1.0) : x;
  t1 = clk(x);
  out[7] = (t1 - t0) / N;
  // loop overhead reference: integer chain
  int v = lane;
  t0 = clk(x);
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = v * 3 + 1;
  t1 = clk(x);
  out[8] = (t1 - t0) / N;
  sink[lane] = x + v;
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 16 * 8);
  cudaMalloc(&s, 64 * 8);
  for (int rep = 0; rep < 2; ++rep) lat<<<1, 32>>>(1.5, d, s);
  long long h[16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"DFMA", "DMUL", "MUFU.RCP64H", "rcp_nr", "rsqrt+add", "SHFL f64", "STS-sync-LDS", "DSETP+sel+DFMA", "IMAD (loop ref)"};
  for (int i = 0; i < 9; ++i) printf("%-16s %lld cycles per step\n", names[i], h[i]);
  return 0;
}
