"""The exact dense GP posterior on the device -- the reference's validation route
(exact_posterior, /root/reference/pkg/src/fagp/posterior.py:107-144), SURVEY.md §8f rank 3.

    K  = gram_matrix(X, X)        fagp_se_gram (kernels.py:119-145 order; exact unit diagonal)
    C  = K + sigma2 I             (the same launch, diag_add = sigma2)
    L  = chol(C)                  fagp_potrf, SpdFactor's jitter schedule [0, b, 10b, 100b] on the host
    alpha = C^{-1} (y - c)        fagp_potrs
    mean = c + Ks alpha           fagp_dgemm, Ks = gram_matrix(X*, X)
    cov  = Kss - Ks C^{-1} Ks^T   fagp_potrs + fagp_dgemm, symmetrised (want_cov)
    var  = diag(cov)              (always; from the same solve)
O(N^3) time and O(N^2) memory: calibration scale, as in the reference.  Deviation: no LU
fallback (posterior.py:100-104) -- a breakdown after the jitter schedule raises NumericalError.
"""

from __future__ import annotations

import numpy as np

from . import _device as dev
from . import _lib
from .errors import NumericalError
from .kernels import as_ard

__all__ = ["se_gram", "exact_posterior"]

JITTER_ATTEMPTS = 3  # backend.py:165


def se_gram(A, B, kernel, diag_add=0.0):
    """Device K[i, j] = exp(-sum_d (eps_d (A_id - B_jd))^2) (+ diag_add on i == j)."""
    kernel = as_ard(kernel)
    p = kernel.p
    Ad, Bd = dev.points(A, p, "A"), dev.points(B, p, "B")
    na, nb = int(Ad.shape[0]), int(Bd.shape[0])
    K = dev.empty((na, nb), device=Ad.device)
    eps = np.array([k.epsilon for k in kernel.per_dim], dtype=np.float64)
    _lib.check(_lib.lib().fagp_se_gram(_lib.ptr(Ad), na, _lib.ptr(Bd), nb, p, _lib.ptr(eps), float(diag_add),
                                       _lib.ptr(K), nb, _lib.stream_handle()), "se_gram")
    return K


def _spd_factor(C):
    """SpdFactor (backend.py:154-189) on the device: potrf attempts with escalating jitter."""
    from .linalg import potrf

    n = int(C.shape[0])
    base = 1e-12 * float(dev.to_host(C.diagonal().contiguous()).sum()) / n  # np.trace
    jitters = [0.0] + [base * 10**k for k in range(JITTER_ATTEMPTS)]
    info = 0
    for jit in jitters:
        work = C
        if jit != 0.0:  # m + jit * np.eye(n): one rounding on the diagonal
            work = C.clone()
            work.diagonal().add_(jit)
        L, info = potrf(work)
        if info == 0:
            return L, jit
    raise NumericalError(f"matrix of order {n} is not positive definite: leading minor {info} failed even with "
                         f"diagonal jitter up to {jitters[-1]:.3e}", pivot_index=int(info))


def exact_posterior(train, Xstar, model, want_cov=False, return_device=False):
    """Drop-in for fagp.posterior.exact_posterior (same arguments and validation), on the GPU.
    Returns PosteriorResult(mean, cov, var)."""
    from .linalg import dgemm, potrs
    from .posterior import PosteriorResult

    kernel = as_ard(model.kernel)
    p = kernel.p
    X = dev.points(train.X, p, "train.X")
    if X.shape[0] < 1:
        raise ValueError("training set must be nonempty")
    N = int(X.shape[0])
    yd = dev.to_device(np.asarray(train.y, dtype=float) if not dev.is_tensor(train.y) else train.y)
    if tuple(yd.shape) != (N,):
        raise ValueError(f"y has shape {tuple(yd.shape)}, expected ({N},)")
    Xs = dev.points(Xstar, p, "Xstar")
    C = se_gram(X, X, kernel, diag_add=model.noise_var)
    L, _ = _spd_factor(C)
    r = yd - model.mean_const if model.mean_const != 0.0 else yd.clone()
    alpha = potrs(L, r)
    Ks = se_gram(Xs, X, kernel)
    mean = dgemm(Ks, alpha)
    if model.mean_const != 0.0:
        mean = mean + model.mean_const
    W = potrs(L, Ks.T.contiguous())                      # C^{-1} Ks^T  (N x N*)
    Kss = se_gram(Xs, Xs, kernel)
    cov = dgemm(Ks, W, alpha=-1.0, beta=1.0, out=Kss)    # Kss - Ks C^{-1} Ks^T
    cov = 0.5 * (cov + cov.T)
    var = cov.diagonal().clone()
    if not want_cov:
        cov = None
    if return_device:
        return PosteriorResult(mean=mean, cov=cov, var=var)
    return PosteriorResult(mean=dev.to_host(mean), cov=None if cov is None else dev.to_host(cov),
                           var=dev.to_host(var))
