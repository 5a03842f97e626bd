// Modal (Hermite-linearised) path (modal.cu): plan and host entry points used by the C ABI files.
#pragma once

#include "common.cuh"

namespace fagp {
namespace modal {

struct Plan {
  int P, L;            // unordered pairs per dimension M(M+1)/2; modal functions per dimension 2M-1
  int pA;              // Gram: dims [0, pA) on the 128-wide A side, [pA, p) on the 24-wide B side
  int64_t KA, KB;      // K sides L^pA, L^(p - pA)
  int ktA, ktB;        // K tiles
  int64_t SA, SB;      // t = Phi^T r sides M^pA, M^(p - pA)
  int stA, stB;        // t tiles
  int tile0, nrun;     // tiles launched: [tile0, tile0 + nrun), K tiles first (t-only runs skip them)
  int S;               // split-K row chunks
  int64_t chunk_rows;  // rows per chunk (multiple of 16)
  int pN;              // variance: dims [0, pN) on the N (epilogue) side, [pN, p) on the K side
  int64_t NR, KR;      // L^pN, L^(p - pN)
  int64_t NP, KP;      // ... padded to 24 / 16
  int64_t Klen, Hlen;  // L^p modal Gram entries, P^p pair entries
};

bool enabled(int p, int M);  // == modal_on(p, M)
Plan make_plan(int64_t N, int p, int M, bool t_only = false);

// fagp_gram output [K | t]: K = sum_r prod_d g_d (L^p), t = Phi^T r (m)
int64_t gram_len(const fagp_basis* b);
size_t gram_workspace(int64_t N, const fagp_basis* b);
int gram(const double* T, int64_t N, const fagp_basis* b, double* out, void* ws, size_t ws_bytes, uint32_t* flags,
         cudaStream_t s);
// t = Phi^T v alone (v already in the table's residual column)
size_t tmatvec_workspace(int64_t N, const fagp_basis* b);
int tmatvec(const double* T, int64_t N, const fagp_basis* b, double* t, void* ws, size_t ws_bytes, cudaStream_t s);

// doubles of scratch the pair-space transforms need (2 * P^p: two P^p buffers)
int64_t scratch_len(const fagp_basis* b);
// H (P^p pair-indexed Gram) from [K | t]; tmp: P^p doubles
int expand(const double* gram, const fagp_basis* b, double* H, double* tmp, cudaStream_t s);
// A (m x m, nullable), G (m x m, nullable) from H; t (m, nullable) copied from [K | t]
int system(const double* H, const double* gram, const double* sqrt_lam, double sigma2, double jit,
           const fagp_basis* b, double* A, double* G, double* t, cudaStream_t s);

// y = c + Phi x over the rows of a table (any 1 <= p <= 8)
int matvec(const double* T, int64_t N, const fagp_basis* b, const double* x, double c, double* y, uint32_t* flags,
           cudaStream_t s);

int64_t predict_op_len(const fagp_basis* b);  // KP * NP + m: [C'' | w]
// C'' from D (m x m) and s (nullable: fold D itself); w appended.  S0, S1: P^p doubles each.
int build_predict_op(const double* D, const double* sqrt_lam, const double* w, const fagp_basis* b, double* op,
                     double* S0, double* S1, cudaStream_t s);
int set_weights(double* op, const double* w, const fagp_basis* b, cudaStream_t s);
int predict(const double* Ts, int64_t Ns, const fagp_basis* b, const double* op, double sigma2, double mean_const,
            double* mean, double* var, uint32_t* flags, cudaStream_t s);

}  // namespace modal
}  // namespace fagp
