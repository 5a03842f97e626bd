// Phase timing of the persistent Cholesky inverse (chol.cu, cholinv_persistent_kernel) with
// %globaltimer marks.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFAGP_CHOL_PROFILE -I include \
//        tools/cholinv_prof.cu -o tools/cholinv_prof && tools/cholinv_prof 1000
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2403_12797_b200/csrc/chol.cu"

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 1000;
  std::vector<double> A(m * m), B(m * m);
  srand(1);
  for (auto& v : B) v = double(rand()) / RAND_MAX - 0.5;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < m; ++j) {
      double s = 0;
      for (int64_t k = 0; k < m; k += 7) s += B[i * m + k] * B[j * m + k];
      A[i * m + j] = s + (i == j ? double(m) : 0.0);
    }
  double *dA, *dW, *scr, *X, *D;
  int* info;
  cudaMalloc(&dA, m * m * 8); cudaMalloc(&dW, m * m * 8); cudaMalloc(&X, m * m * 8); cudaMalloc(&D, m * m * 8);
  cudaMalloc(&scr, fagp::la::cholinv_scratch_len(m) * 8); cudaMalloc(&info, 4);
  cudaMemcpy(dA, A.data(), m * m * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dW, dA, m * m * 8, cudaMemcpyDeviceToDevice);
    cudaMemset(info, 0, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    int rc = fagp::la::chol_inverse_persistent(dW, m, m, info, scr, X, D, m, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rc %d total %.1f us (%s)\n", rc, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  unsigned long long prof[64][4][6];
  cudaMemcpyFromSymbol(prof, fagp::la::g_chol_prof, sizeof(prof));
  const int steps = int((m + 31) / 32);
  printf("step: phaseA  sync1  phaseB  sync2   (us, CTA 0 | CTA 1 phaseB)\n");
  double tot[4] = {0, 0, 0, 0};
  for (int k = 0; k < steps && k < 63; ++k) {
    auto d = [&](int c, int a, int b) { return (prof[k][c][b] - prof[k][c][a]) * 1e-3; };
    for (int q = 0; q < 4; ++q) tot[q] += d(0, q, q + 1);
    if (k % 4 == 0) printf("%3d  %6.2f %6.2f %6.2f %6.2f | %6.2f\n", k, d(0, 0, 1), d(0, 1, 2), d(0, 2, 3), d(0, 3, 4), d(1, 2, 3));
  }
  double fb = 0;
  for (int k = 0; k + 1 < steps && k < 62; ++k) fb += (prof[k][0][3] - prof[k][0][5]) * 1e-3;
  printf("CTA 0 factor_block total %.1f us (%.2f per step)\n", fb, fb / (steps - 1));
  printf("sum: phaseA %.1f sync1 %.1f phaseB %.1f sync2 %.1f us; phase C %.1f us\n", tot[0], tot[1], tot[2], tot[3],
         (prof[63][0][5] - prof[steps - 1][0][4]) * 1e-3);
  unsigned long long bmax[64];
  int bcta[64];
  cudaMemcpyFromSymbol(bmax, fagp::la::g_chol_bmax, sizeof(bmax));
  cudaMemcpyFromSymbol(bcta, fagp::la::g_chol_bmax_cta, sizeof(bcta));
  printf("step: CTA0 B-end | latest B-end (cta) | step length   (us from CTA 0's step start)\n");
  for (int k = 0; k < steps && k < 63; k += 2)
    printf("%3d  %6.2f | %6.2f (%3d) | %6.2f\n", k, (prof[k][0][3] - prof[k][0][0]) * 1e-3,
           (long long)(bmax[k] - prof[k][0][0]) * 1e-3, bcta[k], (prof[k][0][4] - prof[k][0][0]) * 1e-3);
  unsigned long long b8[2][256];
  cudaMemcpyFromSymbol(b8, fagp::la::g_chol_b8, sizeof(b8));
  printf("step 8 phase B per CTA (us): start rel. CTA0 step start / duration\n");
  for (int c = 0; c < 148; ++c)
    printf("%3d:%5.2f/%5.2f%s", c, (long long)(b8[0][c] - prof[8][0][0]) * 1e-3, (long long)(b8[1][c] - b8[0][c]) * 1e-3,
           c % 6 == 5 ? "\n" : "  ");
  printf("\n");
  unsigned long long jb[16];
  cudaMemcpyFromSymbol(jb, fagp::la::g_chol_job, sizeof(jb));
  printf("step 8, CTA 5 phase B (us from its phase-B start): issued %.2f", (long long)(jb[0] - b8[0][5]) * 1e-3);
  for (int q = 0; q < 6; ++q)
    if (jb[1 + 2 * q]) printf(" | job %d ready %.2f done %.2f", q, (long long)(jb[1 + 2 * q] - b8[0][5]) * 1e-3,
                              (long long)(jb[2 + 2 * q] - b8[0][5]) * 1e-3);
  printf(" | end %.2f\n", (long long)(b8[1][5] - b8[0][5]) * 1e-3);
  return 0;
}
