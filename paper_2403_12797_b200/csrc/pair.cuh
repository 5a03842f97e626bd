// Pair-structured path (pair.cu): plan and host entry points used by the C ABI files.
#pragma once

#include "common.cuh"

namespace fagp {
namespace pairk {

struct PairPlan {
  int P;              // unordered pairs per dimension, M (M + 1) / 2
  int pL;             // Gram: dims [0, pL) on the A side, [pL, p) on the B side
  int pN;             // variance: dims [0, pN) on the N (epilogue) side, [pN, p) on the K side
  int64_t GA, GB;     // Gram sides P^pL, P^(p - pL)
  int gtA, gtB;       // Gram tiles (128 x 56)
  int S;              // Gram split-K row chunks
  int64_t chunk_rows; // rows per chunk (multiple of 16)
  int64_t KR, NR;     // variance K / N sides (real)
  int64_t KP, NP;     // ... padded to 16 / 56
  int64_t Hlen;       // P^p distinct Gram entries
  int64_t SA, SB;     // t = Phi^T r as "singleton" tiles: M^pL x M^(p - pL)
  int stA, stB;       // singleton tiles (128 x 56)
  int tile0, nrun;    // tiles launched: [tile0, tile0 + nrun) (t-only runs skip the pair tiles)
};

// The pair form pays off for p >= 2 (for p = 1 it is the SYRK itself).
bool enabled(int p, int M);
PairPlan make_plan(int64_t N, int p, int M, bool t_only = false);

int64_t gram_len(const fagp_basis* b);                       // Hlen + m: [H | t]
size_t gram_workspace(int64_t N, const fagp_basis* b);
int gram(const double* T, int64_t N, const fagp_basis* b, double* out, void* ws, size_t ws_bytes, uint32_t* flags,
         cudaStream_t s);
// A (m x m, nullable), G (m x m, nullable), t (m, nullable) from [H | t]
int system(const double* gram, const double* sqrt_lam, double sigma2, double jit, const fagp_basis* b, double* A,
           double* G, double* t, cudaStream_t s);
// t = Phi^T v alone (the singleton tiles), v already in the table's residual column
size_t tmatvec_workspace(int64_t N, const fagp_basis* b);
int tmatvec(const double* T, int64_t N, const fagp_basis* b, double* t, void* ws, size_t ws_bytes, cudaStream_t s);
// y = Phi x over the rows of a table (any p >= 1)
int matvec(const double* T, int64_t N, const fagp_basis* b, const double* x, double c, double* y, uint32_t* flags,
           cudaStream_t s);
int64_t predict_op_len(const fagp_basis* b);                 // KP * NP + m: [Ct | w]
// Ct from D = X^T X (caller computes D, m x m, ld m) and s; w appended.
// sqrt_lam may be NULL: then Ct folds D itself (the literal route's inner matrix)
int build_predict_op(const double* D, const double* sqrt_lam, const double* w, const fagp_basis* b, double* op,
                     cudaStream_t s);
int set_weights(double* op, const double* w, const fagp_basis* b, cudaStream_t s);
int predict(const double* Ts, int64_t Ns, const fagp_basis* b, const double* op, double sigma2, double mean_const,
            double* mean, double* var, uint32_t* flags, cudaStream_t s);

}  // namespace pairk
}  // namespace fagp
