"""CPU oracle for the FAGP posterior path -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference algorithm (/root/reference/pkg/src/fagp, pure
Python on numpy + OpenBLAS/LAPACK).  It is imported only by tests/, by
__graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline / --impl reference
legs as the timed CPU baseline.  The product (paper_2403_12797_b200) never imports it.

Parity pinning: tests/golden/make_golden.py runs the reference package itself (importable
in the build container) on seeded inputs and stores its outputs; tests/test_oracle.py
checks this restatement against those fixtures and against the reference test-suite
known-answer values, so the oracle is pinned to the reference, not to itself.

Each function cites the reference lines it restates.  Two modes:
  * block=None  -- the reference's own evaluation order: materialised Phi, one
                   `phi.T @ phi` (OpenBLAS DSYRK), DGEMVs (posterior.py:147-264);
  * block=B     -- row blocks of B rows with G accumulated blockwise, for sizes whose
                   Phi does not fit in host memory (SURVEY.md §8c "CPU restatement").
The variance is the diagonal of the reference's covariance (posterior.py:249-263,
cli.py:222) restated as sigma2 * ||L^{-1}(s * phi*_i)||^2 (<= 1.1e-13 apart).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla
from scipy.linalg.lapack import get_lapack_funcs

DELTA2_RHO_SQUARED = "rho_squared"
DELTA2_RHO_LINEAR = "rho_linear"
LAMBDA_FLOOR_REL = 1e-14  # mercer.py:81

_POTRF = get_lapack_funcs(("potrf",), (np.empty((1, 1)),))[0]


def delta2(rho, beta, variant=DELTA2_RHO_SQUARED):
    """mercer.py:94-99"""
    if variant == DELTA2_RHO_SQUARED:
        return (rho * rho / 2.0) * (beta * beta - 1.0)
    if variant == DELTA2_RHO_LINEAR:
        return (rho / 2.0) * (beta * beta - 1.0)
    raise ValueError(variant)


def beta_delta2(eps, rho, variant=DELTA2_RHO_SQUARED):
    """mercer.py:111-113"""
    beta = (1.0 + (2.0 * eps / rho) ** 2) ** 0.25
    return beta, delta2(rho, beta, variant)


def gamma(eps, rho, n, variant=DELTA2_RHO_SQUARED):
    """mercer.py:114-119"""
    beta, _ = beta_delta2(eps, rho, variant)
    i = np.arange(1, n + 1)
    log_gamma = 0.5 * (math.log(beta) - (i - 1) * math.log(2.0) - np.array([math.lgamma(k) for k in i]))
    return np.exp(log_gamma)


def eigenvalues_1d(eps, rho, n, variant=DELTA2_RHO_SQUARED):
    """mercer.py:146-161"""
    _, d2 = beta_delta2(eps, rho, variant)
    denom = rho * rho + d2 + eps * eps
    lam1 = math.sqrt(rho * rho / denom)
    ratio = eps * eps / denom
    return lam1 * ratio ** np.arange(n)


def normalized_hermite(z, count):
    """mercer.py:122-143 (recurrence h_{k+1} = (z c1_k) h_k - c2_k h_{k-1})"""
    z = np.asarray(z, dtype=float)
    out = np.empty(z.shape + (count,))
    out[..., 0] = 1.0
    if count > 1:
        out[..., 1] = z * math.sqrt(2.0)
    for k in range(1, count - 1):
        out[..., k + 1] = z * math.sqrt(2.0 / (k + 1)) * out[..., k] - math.sqrt(k / (k + 1)) * out[..., k - 1]
    return out


def phi_1d(x, eps, rho, n, variant=DELTA2_RHO_SQUARED):
    """mercer.py:276-281"""
    beta, d2 = beta_delta2(eps, rho, variant)
    z = rho * beta * x
    h = normalized_hermite(z, n)
    return math.sqrt(beta) * np.exp(-d2 * x * x)[:, None] * h


def assemble_phi(X, eps, rho, n, variant=DELTA2_RHO_SQUARED):
    """mercer.py:284-292: Phi[r, j] = ((1*phi1[i1])*phi2[i2])*..., last dimension fastest."""
    N, p = X.shape
    phi = np.ones((N, 1))
    for d in range(p):
        phi_d = phi_1d(X[:, d], eps[d], rho[d], n, variant)
        phi = (phi[:, :, None] * phi_d[:, None, :]).reshape(N, -1)
    return phi


def multi_indices(n, p):
    """mercer.py:195-216"""
    grids = np.meshgrid(*([np.arange(1, n + 1)] * p), indexing="ij")
    return np.stack(grids, axis=-1).reshape(n**p, p)


def eigenvalues(eps, rho, n, variant=DELTA2_RHO_SQUARED):
    """mercer.py:350-353 (tensor products, first dimension slowest)"""
    lam = np.ones(1)
    for d in range(len(eps)):
        lam_d = eigenvalues_1d(eps[d], rho[d], n, variant)
        lam = (lam[:, None] * lam_d[None, :]).reshape(-1)
    return lam


def lam_floored(lam, floor_rel=LAMBDA_FLOOR_REL):
    """mercer.py:259-266"""
    return np.maximum(lam, lam.max() * floor_rel)


def gram(X, y, mean_const, eps, rho, n, variant=DELTA2_RHO_SQUARED, block=None):
    """G = Phi^T Phi (posterior.py:168) and t = Phi^T (y - c) (posterior.py:229,233)."""
    r = np.asarray(y, dtype=float) - mean_const
    if block is None:
        phi = assemble_phi(X, eps, rho, n, variant)
        return phi.T @ phi, phi.T @ r
    m = n ** X.shape[1]
    G = np.zeros((m, m))
    t = np.zeros(m)
    for a in range(0, X.shape[0], block):
        phi = assemble_phi(X[a:a + block], eps, rho, n, variant)
        G += phi.T @ phi
        t += phi.T @ r[a:a + block]
    return G, t


def spd_factor(A, jitter_attempts=3):
    """backend.py:154-189: dpotrf(lower) with jitter [0, b, 10b, 100b], b = 1e-12 tr/n.
    Returns (L, jitter) or raises ValueError('pivot', info)."""
    n = A.shape[0]
    base = 1e-12 * float(np.trace(A)) / n
    jitters = [0.0] + [base * 10**k for k in range(jitter_attempts)]
    info = 0
    for jit in jitters:
        work = A if jit == 0.0 else A + jit * np.eye(n)
        c, info = _POTRF(work, lower=1, overwrite_a=False)
        if info == 0:
            return c, jit
    raise ArithmeticError(f"not positive definite, pivot {info}", int(info))


def factor(G, t, lam, noise_var):
    """posterior.py:169-175, 233-235: A = (s G) s + sigma2 I; L; w = s * A^{-1}(s*t); V = L^{-1} S."""
    s = np.sqrt(lam_floored(lam))
    A = s[:, None] * G
    A *= s
    A.flat[:: A.shape[0] + 1] += noise_var
    L, jit = spd_factor(A)
    u = sla.cho_solve((L, True), s * t, check_finite=False)
    w = s * u
    V = sla.solve_triangular(L, np.diag(s), lower=True, check_finite=False)
    return {"s": s, "A": A, "L": L, "jitter": jit, "w": w, "V": V}


def predict(Xs, fitd, eps, rho, n, noise_var, mean_const, variant=DELTA2_RHO_SQUARED, block=32768):
    """mean = c + Phi* w (posterior.py:247); var = sigma2 * rowsum((Phi* V^T)^2) (F4)."""
    Ns = Xs.shape[0]
    mean = np.empty(Ns)
    var = np.empty(Ns)
    blk = Ns if block is None else block
    for a in range(0, Ns, max(1, blk)):
        phis = assemble_phi(Xs[a:a + blk], eps, rho, n, variant)
        mean[a:a + blk] = mean_const + phis @ fitd["w"]
        Z = phis @ fitd["V"].T
        var[a:a + blk] = noise_var * np.einsum("ij,ij->i", Z, Z)
    return mean, var


def posterior(X, y, Xs, eps, rho, n, noise_var, mean_const=0.0, variant=DELTA2_RHO_SQUARED, block=None,
              predict_block=32768):
    """The whole path; returns dict with mean, var and the intermediates."""
    eps = list(eps)
    rho = list(rho)
    G, t = gram(X, y, mean_const, eps, rho, n, variant, block)
    lam = eigenvalues(eps, rho, n, variant)
    fitd = factor(G, t, lam, noise_var)
    mean, var = predict(Xs, fitd, eps, rho, n, noise_var, mean_const, variant, predict_block)
    return {"G": G, "t": t, "lam": lam, "mean": mean, "var": var, **fitd}


def covariance(Xs, fitd, eps, rho, n, noise_var, variant=DELTA2_RHO_SQUARED):
    """The reference's full predictive covariance, scaled form (posterior.py:249-263):
    inner = sigma2 (s_i (A^{-1})_ij s_j) symmetrised; cov = (Phi* inner) Phi*^T symmetrised."""
    m = fitd["L"].shape[0]
    a_inv = sla.cho_solve((fitd["L"], True), np.eye(m), check_finite=False)
    s = fitd["s"]
    inner = noise_var * (s[:, None] * a_inv * s[None, :])
    inner = 0.5 * (inner + inner.T)
    phis = assemble_phi(Xs, list(eps), list(rho), n, variant)
    cov = (phis @ inner) @ phis.T
    return 0.5 * (cov + cov.T)


def se_gram(A, B, eps):
    """kernels.py:119-145 gram_matrix: acc += (eps_j (a_j - b_j))^2 over dims in order; exp(-acc)."""
    acc = np.zeros((A.shape[0], B.shape[0]))
    for j, e in enumerate(eps):
        t = e * (A[:, j][:, None] - B[:, j][None, :])
        acc += t * t
    return np.exp(-acc)


def exact_posterior(X, y, Xs, eps, noise_var, mean_const=0.0, want_cov=False):
    """posterior.py:107-144: the dense exact GP.  C = K + sigma2 I, SpdFactor (jitter schedule),
    alpha = C^{-1}(y - c), mean = c + Ks alpha; cov = Kss - Ks C^{-1} Ks^T symmetrised.  The
    reference's LU fallback (posterior.py:100-104) is not restated (raises instead)."""
    K = se_gram(X, X, eps)
    C = K + noise_var * np.eye(X.shape[0])
    L, jit = spd_factor(C)
    r = np.asarray(y, dtype=float) - mean_const
    alpha = sla.cho_solve((L, True), r, check_finite=False)
    Ks = se_gram(Xs, X, eps)
    out = {"mean": mean_const + Ks @ alpha, "jitter": jit}
    Z = sla.solve_triangular(L, Ks.T, lower=True, check_finite=False)
    out["var"] = 1.0 - np.einsum("ij,ij->j", Z, Z)  # diag(Kss) = 1 exactly
    if want_cov:
        cov = se_gram(Xs, Xs, eps) - Ks @ sla.cho_solve((L, True), Ks.T, check_finite=False)
        out["cov"] = 0.5 * (cov + cov.T)
    return out


def posterior_literal(X, y, Xs, eps, rho, n, noise_var, mean_const=0.0, variant=DELTA2_RHO_SQUARED):
    """method="literal" (posterior.py:176, 184-188, 236-247, 256-262): LamBar factorized
    directly, mean through t1..t5, var = diag(Phi* inner Phi*^T)."""
    eps = list(eps)
    rho = list(rho)
    phi = assemble_phi(X, eps, rho, n, variant)
    phis = assemble_phi(Xs, eps, rho, n, variant)
    lam_f = lam_floored(eigenvalues(eps, rho, n, variant))
    G = phi.T @ phi
    lb = np.diag(1.0 / lam_f) + G / noise_var
    lb = 0.5 * (lb + lb.T)
    L, jit = spd_factor(lb)

    def solve(b):
        return sla.cho_solve((L, True), b, check_finite=False)

    t1 = (np.asarray(y, dtype=float) - mean_const) / noise_var
    t4 = phi @ solve(phi.T @ t1)
    w = lam_f * (phi.T @ (t1 - t4 / noise_var))
    mean = mean_const + phis @ w
    g = G / noise_var
    mid = g - g @ solve(g)
    inner = np.diag(lam_f) - lam_f[:, None] * mid * lam_f[None, :]
    inner = 0.5 * (inner + inner.T)
    var = np.einsum("ij,ij->i", phis @ inner, phis)
    return {"mean": mean, "var": var, "w": w, "inner": inner, "lambda_bar": lb, "jitter": jit}


# ---- the reference's execution modes, timed per phase (bench.py's CPU arm) -------------------
def _blas_single_thread():
    """backend.py:63-70: BLAS pinned to one thread for the duration of a call."""
    from threadpoolctl import threadpool_limits

    return threadpool_limits(limits=1, user_api="blas")


_POOLS = {}


def _pool(workers):
    """backend.py:49-60 (one long-lived pool per worker count)."""
    from concurrent.futures import ThreadPoolExecutor

    if workers not in _POOLS:
        _POOLS[workers] = ThreadPoolExecutor(max_workers=workers)
    return _POOLS[workers]


def gemm(a, b, mode="serial", workers=1, transpose_a=False, transpose_b=False):
    """backend.py:90-130 Backend.gemm: ``serial`` is one BLAS call (OpenBLAS threads inside);
    ``parallel`` partitions the output rows into max(32, ceil(rows / workers)) blocks computed
    by a thread pool with BLAS pinned to one thread."""
    opa = a.T if transpose_a else a
    opb = b.T if transpose_b else b
    rows = opa.shape[0]
    if not (mode == "parallel" and workers > 1):
        return opa @ opb
    block = max(32, -(-rows // workers))
    out = np.empty((rows,) if opb.ndim == 1 else (rows, opb.shape[1]))
    starts = list(range(0, rows, block))

    def fill(start):
        out[start:start + block] = opa[start:start + block] @ opb

    with _blas_single_thread():
        if len(starts) > 1:
            list(_pool(workers).map(fill, starts))
        else:
            fill(0)
    return out


def eigensystem_phi(X, eps, rho, n, variant=DELTA2_RHO_SQUARED, mode="serial", workers=1):
    """mercer.py:356-368: Phi assembled in one piece (serial) or in max(32, ceil(N / workers))
    row blocks on worker threads (parallel), then the finiteness scan (mercer.py:370)."""
    N = X.shape[0]
    if mode == "parallel" and workers > 1 and N > 1:
        from concurrent.futures import ThreadPoolExecutor

        phi = np.empty((N, n ** X.shape[1]))
        block = max(32, -(-N // workers))

        def fill(start):
            phi[start:start + block] = assemble_phi(X[start:start + block], eps, rho, n, variant)

        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(fill, range(0, N, block)))
    else:
        phi = assemble_phi(X, eps, rho, n, variant)
    if not np.all(np.isfinite(phi)):
        raise ArithmeticError("non-finite feature value")
    return phi


PHASES7 = ("eigensystem_train", "eigensystem_test", "gram", "phi_t_r", "factor_solve_trtri", "mean", "var")


def posterior_timed(X, y, Xs, eps, rho, n, noise_var, mean_const=0.0, variant=DELTA2_RHO_SQUARED,
                    mode="serial", workers=1, var_block=32768):
    """The reference path in its own evaluation order and Backend mode, with the seven phases of
    BASELINE.md §4 / SURVEY.md §8d timed separately (seconds):
      (i) eigensystem(X), (ii) eigensystem(X*)                      mercer.py:295-384
      (iii) G = gemm(Phi, Phi, transpose_a)                          posterior.py:168
      (iv) t = gemm(Phi, y - c, transpose_a)                         posterior.py:229-233
      (v) A-build + SpdFactor (jitter) + w + U = L^{-1} diag(s)       posterior.py:169-175, 234-235
      (vi) mean = c + gemm(Phi*, w)                                   posterior.py:247
      (vii) var = sigma2 rowsum((Phi*_b U^T)^2) over var_block rows   posterior.py:249-263 (diagonal)
    Returns (mean, var, {phase: seconds})."""
    import time

    eps, rho = list(eps), list(rho)
    ph = {}
    clock = time.perf_counter
    t0 = clock()
    phi = eigensystem_phi(X, eps, rho, n, variant, mode, workers)
    ph["eigensystem_train"] = clock() - t0
    t0 = clock()
    phis = eigensystem_phi(Xs, eps, rho, n, variant, mode, workers)
    ph["eigensystem_test"] = clock() - t0
    t0 = clock()
    G = gemm(phi, phi, mode, workers, transpose_a=True)
    ph["gram"] = clock() - t0
    t0 = clock()
    r = np.asarray(y, dtype=float) - mean_const
    t = gemm(phi, r, mode, workers, transpose_a=True)
    ph["phi_t_r"] = clock() - t0
    del phi
    t0 = clock()
    lam = eigenvalues(eps, rho, n, variant)
    s = np.sqrt(lam_floored(lam))
    A = s[:, None] * G
    A *= s
    A.flat[:: A.shape[0] + 1] += noise_var
    L, _ = spd_factor(A)
    w = s * sla.cho_solve((L, True), s * t, check_finite=False)
    U = sla.solve_triangular(L, np.diag(s), lower=True, check_finite=False)
    ph["factor_solve_trtri"] = clock() - t0
    t0 = clock()
    mean = mean_const + gemm(phis, w, mode, workers)
    ph["mean"] = clock() - t0
    t0 = clock()
    var = np.empty(Xs.shape[0])
    for a in range(0, Xs.shape[0], var_block):
        Z = gemm(phis[a:a + var_block], U, mode, workers, transpose_b=True)
        var[a:a + var_block] = noise_var * np.einsum("ij,ij->i", Z, Z)
    ph["var"] = clock() - t0
    return mean, var, ph


def useful_flops(N, Ns, m):
    """Algorithmic flop count of the path."""
    return N * m * (m + 1) + 2 * N * m + m**3 / 3 + m**3 / 3 + 2 * Ns * m + Ns * m * (m + 1) + 2 * Ns * m
