// Latency of the 32 x 32 pivot factor + inverse of the persistent Cholesky inverse (chol.cu):
// factor_block (warp column chain + forward elimination) against factor_inv_block (LDL^T chain
// with the Y elimination on a second warp), one CTA, clock64 around each call; checks L^{-1}
// against a host Cholesky inverse.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/pivot_probe.cu -o tools/pivot_probe
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define FAGP_PIVOT_PROF
#include "../paper_2403_12797_b200/csrc/chol.cu"

using namespace fagp::la;

template <int variant>
__global__ void __launch_bounds__(CNT) probe(const double* Sg, int nb, int reps, double* LiG,
                                             long long* cyc, int* badout) {
  __shared__ __align__(16) double S0[CB][CSP], S1[CB][CSP], S2[CB][CSP];
  __shared__ double rsv[CB + 8];
  __shared__ __align__(8) uint64_t colbar[CB];
  const int tid = threadIdx.x;
  if (tid == 0) factor_inv_init(colbar);
  __syncthreads();
  long long tot = 0;
  int bad = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = tid; e < CB * CB; e += CNT) S0[e >> 5][e & 31] = Sg[e];
    __syncthreads();
    const long long t0 = clock64();
    if (tid == 0) g_piv[0][CB + 1] = t0;
    if (variant == 0)
      bad = factor_block(S0, S1, rsv, nb, 0, nullptr, 0, nullptr, LiG, tid, S2);
    else if (variant == 1)
      bad = factor_inv_block<1>(S0, S1, nb, LiG, S2, colbar, r & 1, tid);
    else
      bad = factor_inv_block<0>(S0, S1, nb, LiG, S2, colbar, r & 1, tid);
    __syncthreads();
    const long long t1 = clock64();
    if (r > 0) tot += t1 - t0;
  }
  if (tid == 0) {
    *cyc = tot / (reps - 1);
    *badout = bad;
  }
}

int main() {
  const int n = CB;
  std::vector<double> B(n * n), S(n * n);
  srand(3);
  for (auto& v : B) v = double(rand()) / RAND_MAX - 0.5;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0;
      for (int k = 0; k < n; ++k) s += B[i * n + k] * B[j * n + k];
      S[i * n + j] = s + (i == j ? 0.05 : 0.0);
    }
  // host reference: L, L^{-1}
  std::vector<long double> L(n * n, 0), Li(n * n, 0);
  for (int j = 0; j < n; ++j) {
    long double d = S[j * n + j];
    for (int k = 0; k < j; ++k) d -= L[j * n + k] * L[j * n + k];
    L[j * n + j] = sqrtl(d);
    for (int i = j + 1; i < n; ++i) {
      long double v = S[i * n + j];
      for (int k = 0; k < j; ++k) v -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = v / L[j * n + j];
    }
  }
  for (int c = 0; c < n; ++c)
    for (int r = c; r < n; ++r) {
      long double v = r == c ? 1.0L : 0.0L;
      for (int k = c; k < r; ++k) v -= L[r * n + k] * Li[k * n + c];
      Li[r * n + c] = v / L[r * n + r];
    }
  double *dS, *dL;
  long long* dc;
  int* db;
  cudaMalloc(&dS, n * n * 8);
  cudaMalloc(&dL, n * n * 8);
  cudaMalloc(&dc, 8);
  cudaMalloc(&db, 4);
  cudaMemcpy(dS, S.data(), n * n * 8, cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 3; ++variant)
    for (int nb : {32, 8}) {
      if (variant == 2) probe<2><<<1, CNT>>>(dS, nb, 20, dL, dc, db); else if (variant) probe<1><<<1, CNT>>>(dS, nb, 20, dL, dc, db); else probe<0><<<1, CNT>>>(dS, nb, 20, dL, dc, db);
      long long cyc;
      int bad;
      std::vector<double> out(n * n);
      cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&bad, db, 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(out.data(), dL, n * n * 8, cudaMemcpyDeviceToHost);
      double err = 0, mx = 0;
      if (nb == 32) {
        for (int e = 0; e < n * n; ++e) {
          err = fmax(err, fabs(double(out[e] - Li[e])));
          mx = fmax(mx, fabs(double(Li[e])));
        }
      }
      printf("variant %d nb %2d: %lld cycles (%.2f us at 1.965 GHz) bad %d  max|Li - ref|/max|ref| %.2e  (%s)\n",
             variant, nb, cyc, cyc / 1965.0, bad, nb == 32 ? err / mx : 0.0, cudaGetErrorString(cudaGetLastError()));
    }
  {
    probe<1><<<1, CNT>>>(dS, 32, 3, dL, dc, db);
    long long pv[2][CB + 2];
    cudaMemcpyFromSymbol(pv, g_piv, sizeof(pv));
    const long long t0 = pv[0][CB + 1];
    printf("variant 1 timeline (cycles from the call): column: warp0 start | warp1 start\n");
    for (int j = 0; j < CB; ++j) printf("  %2d: %6lld | %6lld\n", j, pv[0][j] - t0, pv[1][j] - t0);
    printf("  after the barrier %lld\n", pv[1][CB] - t0);
  }
  // breakdown: make pivot 5 negative
  std::vector<double> Sb = S;
  Sb[5 * n + 5] = -1.0;
  cudaMemcpy(dS, Sb.data(), n * n * 8, cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 3; ++variant) {
    if (variant == 2) probe<2><<<1, CNT>>>(dS, 32, 3, dL, dc, db); else if (variant) probe<1><<<1, CNT>>>(dS, 32, 3, dL, dc, db); else probe<0><<<1, CNT>>>(dS, 32, 3, dL, dc, db);
    int bad;
    cudaMemcpy(&bad, db, 4, cudaMemcpyDeviceToHost);
    printf("variant %d breakdown column %d (expect 6)\n", variant, bad);
  }
  return 0;
}
