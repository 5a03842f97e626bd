"""Eigen-decomposition of the SE kernel: host constants + device evaluation.

Mirror of /root/reference/pkg/src/fagp/mercer.py (same names and semantics).  The split is:

* scalar shape constants (beta, delta^2, gamma), the per-dimension eigenvalues and the
  basis table are computed on the host with the reference's own formulas (they are
  O(p*M) scalars, bit-identical to mercer.py:102-161);
* everything per row -- the Hermite recurrence, the eigenfunction table, the tensor-
  product features -- runs in the CUDA kernels of libfagp_b200.so (csrc/basis.cu).

:class:`EigenSystem` is lazy: it keeps X and its 1-D eigenfunction table on the device
and only materialises ``phi`` (N x m) when that attribute is read.  The posterior path
never reads it: the Gram and predict kernels generate feature tiles on chip.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _device as dev
from . import _lib
from .errors import BudgetError, NumericalError
from .kernels import ArdKernelParams, KernelParams1D, as_ard

__all__ = [
    "DELTA2_RHO_SQUARED",
    "DELTA2_RHO_LINEAR",
    "DEFAULT_MEMORY_CAP",
    "LAMBDA_FLOOR_REL",
    "ShapeParams",
    "shape_params",
    "normalized_hermite",
    "eigenvalues_1d",
    "eigenfunction_1d",
    "multi_indices",
    "estimate_bytes",
    "basis_table",
    "Basis",
    "EigenSystem",
    "eigensystem",
    "reconstruct_kernel",
]

DELTA2_RHO_SQUARED = "rho_squared"
DELTA2_RHO_LINEAR = "rho_linear"
DEFAULT_MEMORY_CAP = 8 << 30  # mercer.py:78
LAMBDA_FLOOR_REL = 1e-14  # mercer.py:81


@dataclass(frozen=True)
class ShapeParams:
    beta: float
    delta2: float
    gamma: np.ndarray


def _delta2(rho, beta, variant):
    """mercer.py:94-99"""
    if variant == DELTA2_RHO_SQUARED:
        return (rho * rho / 2.0) * (beta * beta - 1.0)
    if variant == DELTA2_RHO_LINEAR:
        return (rho / 2.0) * (beta * beta - 1.0)
    raise ValueError(f"unknown delta2 variant {variant!r}")


def shape_params(params, n, delta2_variant=DELTA2_RHO_SQUARED):
    """beta, delta^2 and gamma_1..gamma_n of one dimension (mercer.py:102-119)."""
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    eps, rho = params.epsilon, params.rho
    beta = (1.0 + (2.0 * eps / rho) ** 2) ** 0.25
    delta2 = _delta2(rho, beta, delta2_variant)
    i = np.arange(1, n + 1)
    log_gamma = 0.5 * (math.log(beta) - (i - 1) * math.log(2.0) - np.array([math.lgamma(k) for k in i]))
    return ShapeParams(beta=beta, delta2=delta2, gamma=np.exp(log_gamma))


def eigenvalues_1d(params, n, delta2_variant=DELTA2_RHO_SQUARED):
    """lam_i = lam_1 r^(i-1), raw (mercer.py:146-161)."""
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    eps, rho = params.epsilon, params.rho
    sp = shape_params(params, 1, delta2_variant)
    denom = rho * rho + sp.delta2 + eps * eps
    lam1 = math.sqrt(rho * rho / denom)
    ratio = eps * eps / denom
    return lam1 * ratio ** np.arange(n)


def estimate_bytes(N, n, p):
    """The reference's budget estimate of a materialised eigensystem (mercer.py:219-224).

    Kept for API parity: eigensystem() refuses exactly when the reference would.  The GPU
    path never materialises Phi; its real footprint is :func:`device_bytes`.
    """
    m = n**p
    return 8 * (N * m + m * m + 2 * m)


def device_bytes(N, n, p):
    """Device bytes one eigensystem really holds here: X and its 1-D table."""
    return 8 * N * p * (1 + n)


def multi_indices(n, p, max_count=None):
    """All n^p multi-indices, first component slowest, 1-based int64 (mercer.py:195-216).

    Enumerated by the C ABI (fagp_multi_indices); bit-exact with the reference.
    """
    if n < 1 or p < 1:
        raise ValueError(f"n and p must be >= 1, got n={n}, p={p}")
    count = n**p
    if max_count is not None and count > max_count:
        raise BudgetError(
            f"n^p = {n}^{p} = {count} exceeds the configured limit of {max_count}", n_features=count
        )
    out = np.empty((count, p), dtype=np.int64)
    _lib.check(_lib.load().fagp_multi_indices(int(n), int(p), _lib.ptr(out)), "multi_indices")
    return out


def basis_table(params, n, delta2_variant=DELTA2_RHO_SQUARED):
    """Host table of the C ABI (include/fagp_b200.h: struct fagp_basis), bit-exact constants.

    [rho*beta]*p, [-delta2]*p, [sqrt(beta)]*p, then eigenvalues_1d per dimension.
    """
    params = as_ard(params)
    p = params.p
    rb, nd, sb, lam = [], [], [], []
    for k in params.per_dim:
        sp = shape_params(k, n, delta2_variant)
        rb.append(k.rho * sp.beta)  # mercer.py:279
        nd.append(-sp.delta2)  # mercer.py:281
        sb.append(math.sqrt(sp.beta))  # mercer.py:281
        lam.append(eigenvalues_1d(k, n, delta2_variant))
    modal = modal_coeffs(n)
    table = np.concatenate([np.array(rb), np.array(nd), np.array(sb), np.concatenate(lam), modal.reshape(-1)])
    assert table.shape == (int(_lib.load().fagp_basis_table_len(p, n)),)
    return table


def modal_coeffs(n):
    """V (P x L): h_a(z) h_b(z) = sum_k V[pair(a,b), k] h_k(sqrt2 z) (fagp_modal_coeffs, host)."""
    P, L = n * (n + 1) // 2, 2 * n - 1
    out = np.empty((P, L))
    _lib.check(_lib.load().fagp_modal_coeffs(int(n), out.ctypes.data_as(ctypes.c_void_p)), "modal_coeffs")
    return out


class Basis:
    """Device copy of the basis table plus the ctypes ``fagp_basis`` struct that points at it."""

    def __init__(self, params, n, delta2_variant=DELTA2_RHO_SQUARED, device=None):
        params = as_ard(params)
        if params.p > _lib.MAX_P:
            raise ValueError(f"p = {params.p} exceeds the supported maximum of {_lib.MAX_P}")
        if n < 1:
            raise ValueError(f"n must be >= 1, got {n}")
        self.params = params
        self.n = int(n)
        self.p = params.p
        self.m = self.n**self.p
        self.delta2_variant = delta2_variant
        self.width = int(_lib.load().fagp_table_width(self.p, self.n))  # table row width W
        self.host_table = basis_table(params, n, delta2_variant)
        self.table = dev.to_device(self.host_table, device)
        self.struct = _lib.FagpBasis(self.p, self.n, self.m, self.table.data_ptr())

    @property
    def ref(self):
        import ctypes

        return ctypes.byref(self.struct)


def normalized_hermite(z, count):
    """h_k(z) = H_k(z)/sqrt(2^k k!), k < count, on the device (mercer.py:122-143)."""
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    zh = np.asarray(z, dtype=float)
    zd = dev.to_device(zh.reshape(-1))
    out = dev.empty((zd.shape[0], count))
    L = _lib.lib()
    _lib.check(L.fagp_hermite(_lib.ptr(zd), zd.shape[0], int(count), _lib.ptr(out), _lib.stream_handle()), "hermite")
    return dev.to_host(out).reshape(zh.shape + (count,))


def eigenfunction_1d(i, x, params, delta2_variant=DELTA2_RHO_SQUARED):
    """phi_i(x) for one dimension, evaluated on the device (mercer.py:164-192)."""
    if i < 1:
        raise ValueError(f"eigenfunction index must be >= 1, got {i}")
    xh = np.asarray(x, dtype=float)
    if not np.all(np.isfinite(xh)):
        raise ValueError("eigenfunction_1d requires finite x")
    basis = Basis(ArdKernelParams((KernelParams1D(params.epsilon, params.rho),)), i, delta2_variant)
    xd = dev.to_device(xh.reshape(-1, 1))
    T = dev.empty((xd.shape[0], basis.width))
    L = _lib.lib()
    _lib.check(L.fagp_basis_eval(_lib.ptr(xd), xd.shape[0], basis.ref, None, 0.0, _lib.ptr(T), None,
                                 _lib.stream_handle()), "eigenfunction_1d")
    val = dev.to_host(T[:, i - 1]).reshape(xh.shape)
    return val if val.ndim else float(val)


@dataclass
class EigenSystem:
    """Device-resident truncated eigensystem (reference: mercer.py:227-273).

    ``lam``, ``indices`` are host arrays exactly as in the reference; ``phi`` is
    materialised from the device table on first access (N x m, float64, host numpy).
    """

    lam: np.ndarray
    params: ArdKernelParams
    n: int
    delta2_variant: str
    X: object  # device tensor (N, p)
    table: object  # device tensor (N, W): per-row 1-D eigenfunction values (+ r, 1, 0)
    basis: Basis
    floor_rel: float = field(default=LAMBDA_FLOOR_REL, repr=False)
    _phi: np.ndarray | None = field(default=None, repr=False)
    _indices: np.ndarray | None = field(default=None, repr=False)

    @property
    def size(self):
        return self.lam.shape[0]

    @property
    def N(self):
        return int(self.X.shape[0])

    @property
    def indices(self):
        if self._indices is None:
            self._indices = multi_indices(self.n, self.params.p)
        return self._indices

    @property
    def lam_floored(self):
        """mercer.py:259-266"""
        return np.maximum(self.lam, self.lam.max() * self.floor_rel)

    @property
    def phi(self):
        if self._phi is None:
            self._phi = dev.to_host(self.phi_device())
        return self._phi

    def phi_device(self):
        out = dev.empty((self.N, self.size))
        L = _lib.lib()
        _lib.check(L.fagp_features(_lib.ptr(self.table), self.N, self.basis.ref, _lib.ptr(out), None,
                                   _lib.stream_handle()), "features")
        return out

    def compatible_with(self, other):
        return (
            as_ard(self.params) == as_ard(other.params)
            and self.n == other.n
            and self.delta2_variant == other.delta2_variant
        )


def _budget(N, n, p, memory_cap):
    if memory_cap is None:
        return
    est = estimate_bytes(N, n, p)
    if est > memory_cap:
        raise BudgetError(
            f"eigensystem with n^p = {n}^{p} = {n**p} features over N={N} points "
            f"needs an estimated {est} bytes, above the cap of {memory_cap} bytes; "
            f"reduce n or p, or raise the cap",
            n_features=n**p,
            estimated_bytes=est,
            cap_bytes=memory_cap,
        )


def raise_nonfinite(table, X, basis, what="feature"):
    """Name the first non-finite feature like the reference does (mercer.py:371-376)."""
    L = _lib.lib()
    first = dev.empty((1,), dtype="int64")
    _lib.check(L.fagp_find_nonfinite(_lib.ptr(table), int(table.shape[0]), basis.ref, _lib.ptr(first),
                                     _lib.stream_handle()), "find_nonfinite")
    e = int(dev.to_host(first)[0])
    if e < 0:
        return
    i, j = divmod(e, basis.m)
    point = dev.to_host(X[i])
    idx = tuple(int(v) for v in multi_indices(basis.n, basis.p)[j])
    raise NumericalError(f"non-finite {what} value at row {i}, column {j} (point {point}, multi-index {idx})")


def eigensystem(X, params, n, backend=None, memory_cap=DEFAULT_MEMORY_CAP, delta2_variant=DELTA2_RHO_SQUARED):
    """Build the device eigensystem of the n^p tensor-product pairs on X (mercer.py:295-384).

    Same validation order and errors as the reference: ValueError (shape, non-finite X,
    n), BudgetError (reference estimate over ``memory_cap``; ``None`` disables), and
    NumericalError naming the first non-finite feature.
    """
    params = as_ard(params)
    Xd = dev.points(X, params.p, "X")
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    N, p = int(Xd.shape[0]), params.p
    _budget(N, n, p, memory_cap)
    basis = Basis(params, n, delta2_variant, device=Xd.device)
    L = _lib.lib()
    table = dev.empty((N, basis.width))
    flags = dev.zeros((1,), dtype="int32")
    s = _lib.stream_handle()
    if N > 0:
        _lib.check(L.fagp_basis_eval(_lib.ptr(Xd), N, basis.ref, None, 0.0, _lib.ptr(table), _lib.ptr(flags), s),
                   "basis_eval")
    lam = dev.empty((basis.m,))
    _lib.check(L.fagp_eigenvalues(basis.ref, LAMBDA_FLOOR_REL, _lib.ptr(lam), None, None, s), "eigenvalues")
    if int(dev.to_host(flags)[0]) & _lib.FLAG_X_NONFINITE:
        raise ValueError("X must be finite")
    raise_nonfinite(table, Xd, basis)
    return EigenSystem(lam=dev.to_host(lam), params=params, n=int(n), delta2_variant=delta2_variant, X=Xd,
                       table=table, basis=basis)


def reconstruct_kernel(es_a, es_b):
    """Low-rank kernel Phi_A Lam Phi_B^T (mercer.py:387-400); test/diagnostic helper."""
    if not es_a.compatible_with(es_b):
        raise ValueError("eigensystems were built with different params, n, or delta2 variant")
    import torch

    s = torch.as_tensor(np.sqrt(es_a.lam), device=es_a.X.device)
    return dev.to_host((es_a.phi_device() * s) @ (es_b.phi_device() * s).T)
