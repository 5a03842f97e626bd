"""FAGP posterior on the GPU: the drop-in surface of /root/reference/pkg/src/fagp/posterior.py.

Pipeline of :func:`fagp_posterior` (posterior.py:267-318 in the reference), every stage a
call into libfagp_b200.so on the current CUDA stream:

    fagp_eigenvalues                           lam, lam_floored, s           (mercer.py:350-353)
    fagp_gram_x(X, y)                          eigenfunctions on chip         (mercer.py:276-281)
                                               + Gram [K | t] on DMMA         (posterior.py:168,233)
    [torch.distributed all_reduce of the packed Gram when sharded]
    fagp_factor                                A, Cholesky+jitter, w, op      (posterior.py:171-175,234-235)
    fagp_predict_x(X*)                         eigenfunctions on chip         (posterior.py:247,249-263)
                                               + mean and variance on DMMA

``method="literal"`` (the reference's cross-check route, posterior.py:236-244, 256-260) runs
on the device too: see :mod:`literal`.

``PosteriorResult`` gains ``var`` (the per-point predictive variance, i.e. the diagonal of
the reference's covariance that `fagp predict` reports, cli.py:222).  The full N* x N*
covariance (``want_cov=True``) is formed from the same factor for modest N*.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, replace

import numpy as np

from . import _device as dev
from . import _lib
from .errors import NumericalError
from .kernels import as_ard
from .literal import lambda_bar_matrix, literal_posterior
from .mercer import (
    DEFAULT_MEMORY_CAP,
    DELTA2_RHO_SQUARED,
    LAMBDA_FLOOR_REL,
    Basis,
    _budget,
    raise_nonfinite,
)

__all__ = [
    "GpModel",
    "PosteriorResult",
    "Fit",
    "fit",
    "predict",
    "fagp_posterior",
    "fagp_posterior_from_eigensystems",
    "lambda_bar",
    "LambdaBarSolve",
    "set_fault_injection",
]

JITTER_ATTEMPTS = 3  # backend.py:165 (SpdFactor default)

_FAULT_FLIP_MEAN_SIGN = False


def set_fault_injection(enabled):
    """Test hook: flip the sign of w before the mean (posterior.py:54-62, 245-246)."""
    global _FAULT_FLIP_MEAN_SIGN
    _FAULT_FLIP_MEAN_SIGN = bool(enabled)


@dataclass(frozen=True)
class GpModel:
    """Same fields and validation as the reference (posterior.py:65-82)."""

    kernel: object
    noise_var: float
    mean_const: float = 0.0
    n_eigen: int | None = None

    def __post_init__(self):
        if not np.isfinite(self.noise_var) or self.noise_var <= 0:
            raise ValueError(f"noise_var must be finite and > 0, got {self.noise_var!r}")
        if self.n_eigen is not None and self.n_eigen < 1:
            raise ValueError(f"n_eigen must be >= 1, got {self.n_eigen}")


@dataclass
class PosteriorResult:
    """mean (N*,), optional cov (N*, N*) as in the reference, plus var (N*,)."""

    mean: object
    cov: object | None = None
    var: object | None = None


class _Flags:
    """Two device flag words: [train, test]."""

    def __init__(self, device=None):
        self.dev = dev.zeros((2,), dtype="int32", device=device)

    def ptr(self, k):
        return ctypes.c_void_p(self.dev.data_ptr() + 4 * k)

    def read(self):
        return [int(v) for v in dev.to_host(self.dev)]


@dataclass
class Fit:
    """Device fit state (immutable after fit; predict calls may run concurrently)."""

    basis: Basis
    noise_var: float
    mean_const: float
    N: int
    lam: object  # device (m,)
    lam_floored: object
    sqrt_lam: object
    packed: object  # packed extended Gram ((m+1)(m+2)/2,)
    L: object  # (m, m) lower Cholesky factor of A (None on the inverse route)
    t: object  # Phi^T (y - c)
    w: object  # s * A^{-1}(s * t)
    predict_op: object  # [V^T | w] operand of fagp_predict
    jitter: float
    G: object | None = None
    Ainv: object | None = None  # (m, m) A^{-1} (modal shapes, fagp_factor_inv)

    @property
    def m(self):
        return self.basis.m


def _check_y(y, N):
    if dev.is_tensor(y):
        yd = dev.to_device(y)
        shape = tuple(yd.shape)
    else:
        yh = np.asarray(y, dtype=float)
        shape = yh.shape
        yd = dev.to_device(yh) if shape == (N,) else None
    if shape != (N,):
        raise ValueError(f"y has shape {shape}, expected ({N},)")
    return yd


def _stage_tables(basis, Xd, flag_ptr, s, yd=None, mean_const=0.0):
    N = int(Xd.shape[0])
    T = dev.empty((N, basis.width), device=Xd.device)
    if N > 0:
        _lib.check(_lib.lib().fagp_basis_eval(_lib.ptr(Xd), N, basis.ref, _lib.ptr(yd), float(mean_const), _lib.ptr(T),
                                              flag_ptr, s), "basis_eval")
    return T


def gram_packed(basis, T, yd=None, mean_const=0.0, flag_ptr=None, stream=None):
    """fagp_gram on a table: packed upper triangle of [Phi|r]^T[Phi|r] (device).  The
    table's residual column is (re)written from ``yd`` first (zero when ``yd`` is None)."""
    L = _lib.lib()
    s = _lib.stream_handle(stream)
    N = int(T.shape[0])
    if N > 0:
        _lib.check(L.fagp_set_residual(_lib.ptr(T), N, basis.ref, _lib.ptr(yd), float(mean_const), s), "set_residual")
    packed = dev.empty((int(L.fagp_gram_len(basis.ref)),), device=T.device)
    wsz = int(L.fagp_gram_workspace_size(N, basis.ref))
    ws = dev.empty((max(1, wsz // 8),), device=T.device)
    _lib.check(L.fagp_gram(_lib.ptr(T), N, basis.ref, _lib.ptr(packed), _lib.ptr(ws), wsz, flag_ptr, s), "gram")
    return packed


def gram_x_packed(basis, Xd, yd=None, mean_const=0.0, flag_ptr=None, stream=None):
    """fagp_gram_x: the same `gram` buffer straight from the points (eigenfunctions on chip)."""
    L = _lib.lib()
    s = _lib.stream_handle(stream)
    N = int(Xd.shape[0])
    packed = dev.empty((int(L.fagp_gram_len(basis.ref)),), device=Xd.device)
    wsz = int(L.fagp_gram_x_workspace_size(N, basis.ref))
    ws = dev.empty((max(1, -(-wsz // 8)),), device=Xd.device)
    _lib.check(L.fagp_gram_x(_lib.ptr(Xd), N, basis.ref, _lib.ptr(yd), float(mean_const), _lib.ptr(packed),
                             _lib.ptr(ws), wsz, flag_ptr, s), "gram_x")
    return packed


def factor_packed(basis, packed, noise_var, mean_const, N, keep_gram=False, stream=None, need_L=False):
    """fagp_factor / fagp_factor_inv: jitter schedule, weights, predict operand.  Modal shapes
    take the fused inverse route (A^{-1}, no L) unless ``need_L``.  Returns (Fit, status, pivot)."""
    L = _lib.lib()
    s = _lib.stream_handle(stream)
    m = basis.m
    device = packed.device
    lam = dev.empty((m,), device=device)
    lam_f = dev.empty((m,), device=device)
    sq = dev.empty((m,), device=device)
    _lib.check(L.fagp_eigenvalues(basis.ref, LAMBDA_FLOOR_REL, _lib.ptr(lam), _lib.ptr(lam_f), _lib.ptr(sq), s),
               "eigenvalues")
    G = dev.empty((m, m), device=device) if keep_gram else None
    t = dev.empty((m,), device=device)
    w = dev.empty((m,), device=device)
    P = dev.empty((int(L.fagp_predict_operand_len(basis.ref)),), device=device)
    wsz = int(L.fagp_factor_workspace_size(m))
    ws = dev.empty((max(1, wsz // 8),), device=device)
    jit = ctypes.c_double(0.0)
    piv = ctypes.c_int32(0)
    Lf = Ainv = None
    st = _lib.FAGP_EUNSUPPORTED
    if not need_L:
        Ainv = dev.empty((m, m), device=device)
        st = L.fagp_factor_inv(_lib.ptr(packed), basis.ref, _lib.ptr(sq), float(noise_var), JITTER_ATTEMPTS,
                               _lib.ptr(Ainv), _lib.ptr(G), _lib.ptr(t), _lib.ptr(w), _lib.ptr(P), ctypes.byref(jit),
                               ctypes.byref(piv), _lib.ptr(ws), wsz, s)
        if st == _lib.FAGP_EUNSUPPORTED:
            Ainv = None
    if st == _lib.FAGP_EUNSUPPORTED:
        Lf = dev.empty((m, m), device=device)
        st = L.fagp_factor(_lib.ptr(packed), basis.ref, _lib.ptr(sq), float(noise_var), JITTER_ATTEMPTS, _lib.ptr(Lf),
                           _lib.ptr(G), _lib.ptr(t), _lib.ptr(w), _lib.ptr(P), ctypes.byref(jit), ctypes.byref(piv),
                           _lib.ptr(ws), wsz, s)
    f = Fit(basis=basis, noise_var=float(noise_var), mean_const=float(mean_const), N=N, lam=lam, lam_floored=lam_f,
            sqrt_lam=sq, packed=packed, L=Lf, t=t, w=w, predict_op=P, jitter=float(jit.value), G=G, Ainv=Ainv)
    return f, st, int(piv.value)


def gram_unpack(basis, packed):
    """Full symmetric G (m x m) and t (m) from a `gram` buffer (device tensors)."""
    L = _lib.lib()
    G = dev.empty((basis.m, basis.m), device=packed.device)
    t = dev.empty((basis.m,), device=packed.device)
    wsz = int(L.fagp_gram_unpack_workspace_size(basis.ref))
    ws = dev.empty((max(1, wsz // 8),), device=packed.device)
    _lib.check(L.fagp_gram_unpack(_lib.ptr(packed), basis.ref, _lib.ptr(G), _lib.ptr(t), _lib.ptr(ws), wsz,
                                  _lib.stream_handle()), "gram_unpack")
    return G, t


def _raise_factor(st, piv, m):
    if st == _lib.FAGP_ENOTPD:
        raise NumericalError(
            f"matrix of order {m} is not positive definite: leading minor {piv} "
            f"failed even with diagonal jitter", pivot_index=piv)
    _lib.check(st, "factor", pivot_index=piv)


def _apply_fault(f, stream=None):
    if _FAULT_FLIP_MEAN_SIGN:
        f.w.neg_()
        _lib.check(_lib.lib().fagp_set_mean_weights(_lib.ptr(f.predict_op), _lib.ptr(f.w), f.basis.ref,
                                                    _lib.stream_handle(stream)), "set_mean_weights")


def predict_device(f, Ts, want_var=True, flag_ptr=None, stream=None):
    """fagp_predict on a staged test table; returns device (mean, var|None)."""
    L = _lib.lib()
    s = _lib.stream_handle(stream)
    Ns = int(Ts.shape[0])
    mean = dev.empty((Ns,), device=Ts.device)
    var = dev.empty((Ns,), device=Ts.device) if want_var else None
    if Ns > 0:
        _lib.check(L.fagp_predict(_lib.ptr(Ts), Ns, f.basis.ref, _lib.ptr(f.predict_op), f.noise_var, f.mean_const,
                                  _lib.ptr(mean), _lib.ptr(var), flag_ptr, s), "predict")
    return mean, var


def predict_x_device(f, Xs, want_var=True, flag_ptr=None, stream=None):
    """fagp_predict_x straight from the test points; returns device (mean, var|None)."""
    L = _lib.lib()
    s = _lib.stream_handle(stream)
    Ns = int(Xs.shape[0])
    mean = dev.empty((Ns,), device=Xs.device)
    var = dev.empty((Ns,), device=Xs.device) if want_var else None
    if Ns > 0:
        wsz = int(L.fagp_predict_x_workspace_size(Ns, f.basis.ref))
        ws = dev.empty((max(1, -(-wsz // 8)),), device=Xs.device)
        _lib.check(L.fagp_predict_x(_lib.ptr(Xs), Ns, f.basis.ref, _lib.ptr(f.predict_op), f.noise_var, f.mean_const,
                                    _lib.ptr(mean), _lib.ptr(var), flag_ptr, _lib.ptr(ws), wsz, s), "predict_x")
    return mean, var


def _covariance(f, Ts):
    """Full predictive covariance (posterior.py:249-263): sigma2 * Z Z^T with Z = Phi* V^T on
    the Cholesky route, sigma2 * (Phi* S) A^{-1} (Phi* S)^T on the inverse route."""
    from .linalg import dgemm

    m = f.m
    Ns = int(Ts.shape[0])
    phis = dev.empty((Ns, m), device=Ts.device)
    _lib.check(_lib.lib().fagp_features(_lib.ptr(Ts), Ns, f.basis.ref, _lib.ptr(phis), None, _lib.stream_handle()),
               "features")
    if f.L is None:
        Zs = phis * f.sqrt_lam  # Phi* S
        Y = dgemm(Zs, f.Ainv)
        cov = dgemm(Y, Zs, trans_b=True, alpha=f.noise_var)
    else:
        V = trtri_scaled(f)
        Z = dgemm(phis, V, trans_b=True)  # Z = Phi* V^T
        cov = dgemm(Z, Z, trans_b=True, alpha=f.noise_var)
    cov = 0.5 * (cov + cov.T)
    return cov


def trtri_scaled(f):
    """V = L^{-1} diag(s) (m x m, device)."""
    L = _lib.lib()
    m = f.m
    V = dev.empty((m, m), device=f.L.device)
    wsz = int(L.fagp_trtri_workspace_size(m))
    ws = dev.empty((max(1, wsz // 8),), device=f.L.device)
    _lib.check(L.fagp_trtri(_lib.ptr(f.L), _lib.ptr(f.sqrt_lam), m, _lib.ptr(V), _lib.ptr(ws), wsz,
                            _lib.stream_handle()), "trtri")
    return V


def _as_train(train, p):
    X = dev.points(train.X, p, "train.X")
    N = int(X.shape[0])
    return X, _check_y(train.y, N)


def fit(train, model, backend=None, memory_cap=DEFAULT_MEMORY_CAP, delta2_variant=DELTA2_RHO_SQUARED,
        keep_gram=False, group=None):
    """Fit handle: the Gram contraction, its (optional) cross-rank reduction and the factor.

    ``group``: a torch.distributed process group over which ``train`` rows are sharded
    (each rank passes its own shard); the packed Gram is all-reduced (sum) before the
    factorisation, which every rank then runs redundantly.
    """
    if model.n_eigen is None:
        raise ValueError("model.n_eigen must be set for the fast posterior")
    kernel = as_ard(model.kernel)
    X, yd = _as_train(train, kernel.p)
    N = int(X.shape[0])
    _budget(N, model.n_eigen, kernel.p, memory_cap)
    basis = Basis(kernel, model.n_eigen, delta2_variant, device=X.device)
    flags = _Flags(X.device)
    s = _lib.stream_handle()
    packed = gram_x_packed(basis, X, yd, model.mean_const, flags.ptr(0))
    if group is not None:
        from .distributed import all_reduce_sum

        all_reduce_sum(packed, group)
    f, st, piv = factor_packed(basis, packed, model.noise_var, model.mean_const, N, keep_gram=keep_gram)
    fl = flags.read()
    if fl[0] & _lib.FLAG_X_NONFINITE:
        raise ValueError("X must be finite")
    if fl[0] & _lib.FLAG_PHI_NONFINITE:
        raise_nonfinite(_stage_tables(basis, X, None, s), X, basis)
    if st != _lib.FAGP_OK:
        _raise_factor(st, piv, basis.m)
    _apply_fault(f)
    return f


def predict(f, Xstar, want_var=True, want_cov=False, return_device=False):
    """Posterior mean (and variance / covariance) at X* for a fit handle."""
    Xs = dev.points(Xstar, f.basis.p, "Xstar")
    flags = _Flags(Xs.device)
    mean, var = predict_x_device(f, Xs, want_var=want_var, flag_ptr=flags.ptr(1))
    cov = _covariance(f, _stage_tables(f.basis, Xs, None, _lib.stream_handle())) if want_cov else None
    fl = flags.read()
    if fl[1] & _lib.FLAG_X_NONFINITE:
        raise ValueError("Xstar must be finite")
    if fl[1] & _lib.FLAG_PHI_NONFINITE:
        raise_nonfinite(_stage_tables(f.basis, Xs, None, _lib.stream_handle()), Xs, f.basis)
    if return_device:
        return PosteriorResult(mean=mean, cov=cov, var=var)
    return PosteriorResult(mean=dev.to_host(mean), cov=None if cov is None else dev.to_host(cov),
                           var=None if var is None else dev.to_host(var))


def fagp_posterior(train, Xstar, model, backend=None, want_cov=False, method="scaled",
                   memory_cap=DEFAULT_MEMORY_CAP, delta2_variant=DELTA2_RHO_SQUARED, want_var=True,
                   return_device=False, group=None):
    """Drop-in for fagp.posterior.fagp_posterior (posterior.py:267-318), on the GPU.

    Same arguments, validation order and exceptions.  ``backend`` is accepted for
    signature compatibility (any reference Backend); execution is always the CUDA path.
    Extra keywords: ``want_var`` (default True) fills ``result.var``; ``return_device``
    keeps the outputs as CUDA tensors; ``group`` shards the training rows over a
    torch.distributed group (each rank passes its own train/test shards; the packed Gram
    is all-reduced before the factorisation).
    """
    from .engine import PosteriorEngine

    if model.n_eigen is None:
        raise ValueError("model.n_eigen must be set for the fast posterior")
    if method not in ("scaled", "literal"):
        raise ValueError(f"form must be 'scaled' or 'literal', got {method!r}")
    kernel = as_ard(model.kernel)
    p = kernel.p
    if (method == "scaled" and not return_device
            and not any(dev.is_cuda(a) for a in (train.X, train.y, Xstar))):
        return _posterior_host(train, Xstar, model, kernel, want_cov, memory_cap, delta2_variant, want_var, group)
    X = dev.points(train.X, p, "train.X")
    dev.points_shape(Xstar, p, "Xstar")
    Xs, xs_ready = dev.upload_async(Xstar if dev.is_tensor(Xstar) else np.atleast_2d(np.asarray(Xstar, dtype=float)),
                                    X.device)
    Xs = Xs.reshape(-1, p)
    N, Ns = int(X.shape[0]), int(Xs.shape[0])
    yd = _check_y(train.y, N)
    _budget(N, model.n_eigen, p, memory_cap)
    _budget(Ns, model.n_eigen, p, memory_cap)
    if method == "literal":
        if group is not None:
            raise ValueError("method='literal' does not shard (group must be None)")
        dev.wait_upload(xs_ready)
        basis = Basis(kernel, model.n_eigen, delta2_variant, device=X.device)
        flags = _Flags(X.device)
        s = _lib.stream_handle()
        T = _stage_tables(basis, X, flags.ptr(0), s)
        Ts = _stage_tables(basis, Xs, flags.ptr(1), s)
        mean, var, cov = literal_posterior(basis, T, Ts, yd, model.noise_var, model.mean_const, want_var=want_var,
                                           want_cov=want_cov, fault_flip=_FAULT_FLIP_MEAN_SIGN, X=X, Xs=Xs,
                                           flags=flags)
        return _result(mean, var, cov, return_device)
    eng = PosteriorEngine(kernel, model.n_eigen, N, Ns, model.noise_var, model.mean_const, delta2_variant,
                          device=X.device, group=group, want_var=want_var)
    mean, var = eng.run(X, yd, Xs, fault_flip=_FAULT_FLIP_MEAN_SIGN, xs_ready=xs_ready)
    eng.check(X, Xs, yd)
    cov = None
    if want_cov:
        cov = _covariance(_engine_fit(eng, N), eng.table(Xs))
    return _result(mean, var, cov, return_device)


def _engine_fit(eng, N):
    """The Fit view of an engine's factorisation (for the full covariance)."""
    return Fit(basis=eng.basis, noise_var=eng.noise_var, mean_const=eng.mean_const, N=N, lam=eng.lam,
               lam_floored=eng.lam_floored, sqrt_lam=eng.sqrt_lam, packed=eng.packed, L=eng.L, t=eng.t, w=eng.w,
               predict_op=eng.predict_op, jitter=float(eng.jitter.value), Ainv=eng.Ainv)


_ENGINES = threading.local()


def _engine_for(key, make):
    """One cached PosteriorEngine per thread (buffers, streams and pinned staging reused across
    calls of the same shape; thread-local, so concurrent callers never share one)."""
    cached = getattr(_ENGINES, "entry", None)
    if cached is not None and cached[0] == key:
        return cached[1]
    _ENGINES.entry = None
    eng = make()
    _ENGINES.entry = (key, eng)
    return eng


def _posterior_host(train, Xstar, model, kernel, want_cov, memory_cap, delta2_variant, want_var, group):
    """fagp_posterior for host inputs: PosteriorEngine.run_host pipelines the H2D uploads with
    the Gram chunks and the D2H of the results with the predict chunks."""
    from .engine import PosteriorEngine

    p = kernel.p
    Xh = dev.host_points(train.X, p, "train.X")
    Xsh = dev.host_points(Xstar, p, "Xstar")
    N, Ns = int(Xh.shape[0]), int(Xsh.shape[0])
    yh = dev.host_vector(train.y, N)
    _budget(N, model.n_eigen, p, memory_cap)
    _budget(Ns, model.n_eigen, p, memory_cap)
    device = dev.device_of()
    key = (kernel, int(model.n_eigen), N, Ns, float(model.noise_var), float(model.mean_const), delta2_variant,
           str(device), bool(want_var), id(group))
    eng = _engine_for(key, lambda: PosteriorEngine(kernel, model.n_eigen, N, Ns, model.noise_var, model.mean_const,
                                                   delta2_variant, device=device, group=group, want_var=want_var))
    mean, var = eng.run_host(Xh, yh, Xsh, fault_flip=_FAULT_FLIP_MEAN_SIGN)
    eng.check(eng.X, eng.Xs, eng.y)
    cov = None
    if want_cov:
        cov = dev.to_host(_covariance(_engine_fit(eng, N), eng.table(eng.Xs)))
    return PosteriorResult(mean=mean, cov=cov, var=var)


def _result(mean, var, cov, return_device):
    if return_device:
        return PosteriorResult(mean=mean, cov=cov, var=var)
    return PosteriorResult(mean=dev.to_host(mean), cov=None if cov is None else dev.to_host(cov),
                           var=None if var is None else dev.to_host(var))


def fagp_posterior_from_eigensystems(es, es_star, y, model, backend=None, want_cov=False, method="scaled",
                                     want_var=True, return_device=False):
    """Split form (posterior.py:210-264) on device eigensystems from :func:`mercer.eigensystem`."""
    if not es.compatible_with(es_star):
        raise ValueError("train and test eigensystems are incompatible")
    if as_ard(es.params) != as_ard(model.kernel):
        raise ValueError("eigensystem params do not match model.kernel")
    yd = _check_y(y, es.N)
    if method not in ("scaled", "literal"):
        raise ValueError(f"form must be 'scaled' or 'literal', got {method!r}")
    if method == "literal":
        # the tables are the eigensystems' own; phi_tmatvec rewrites only the residual column
        mean, var, cov = literal_posterior(es.basis, es.table, es_star.table, yd, model.noise_var, model.mean_const,
                                           want_var=want_var, want_cov=want_cov, fault_flip=_FAULT_FLIP_MEAN_SIGN)
        return _result(mean, var, cov, return_device)
    packed = gram_x_packed(es.basis, es.X, yd, model.mean_const)
    f, st, piv = factor_packed(es.basis, packed, model.noise_var, model.mean_const, es.N)
    if st != _lib.FAGP_OK:
        _raise_factor(st, piv, es.basis.m)
    _apply_fault(f)
    mean, var = predict_x_device(f, es_star.X, want_var=want_var)
    cov = _covariance(f, es_star.table) if want_cov else None
    return _result(mean, var, cov, return_device)


class LambdaBarSolve:
    """Solve handle for LamBar = Lam^{-1} + Phi^T Phi / sigma2 (posterior.py:147-202), on device.

    ``form="scaled"`` factorises A = sigma2 I + S G S (fagp_factor); ``form="literal"``
    factorises LamBar itself (fagp_potrf with the same jitter schedule).
    """

    def __init__(self, es, noise_var, backend=None, form="scaled"):
        if noise_var <= 0:
            raise ValueError(f"noise_var must be > 0, got {noise_var!r}")
        if form not in ("scaled", "literal"):
            raise ValueError(f"form must be 'scaled' or 'literal', got {form!r}")
        self.form = form
        self.noise_var = float(noise_var)
        self._es = es
        packed = gram_x_packed(es.basis, es.X, None, 0.0)
        f, st, piv = factor_packed(es.basis, packed, noise_var, 0.0, es.N, keep_gram=True, need_L=True)
        self._fit = f
        self._gram = f.G
        self.lam_floored = dev.to_host(f.lam_floored)
        self.sqrt_lam = dev.to_host(f.sqrt_lam)
        if form == "scaled":
            if st != _lib.FAGP_OK:
                _raise_factor(st, piv, es.size)
            from .backend import SpdFactor

            self._factor = SpdFactor._from_device_factor(f.L, f.jitter)
        else:
            from .backend import SpdFactor

            self._factor = SpdFactor(self._matrix_device(), check_symmetric=False)

    @property
    def size(self):
        return self._es.size

    def _matrix_device(self):
        return lambda_bar_matrix(self._gram, self._fit.lam_floored, self.noise_var)

    @property
    def matrix(self):
        """Explicit symmetric LamBar (posterior.py:184-187)."""
        return dev.to_host(self._matrix_device())

    def solve_inner(self, b):
        """Solve against whichever matrix was factorised (A or LamBar)."""
        return self._factor.solve(b)

    def solve(self, b):
        """Solve LamBar x = b (posterior.py:193-202); device arithmetic, host in/out."""
        bd = dev.to_device(np.asarray(b, dtype=float))
        if self.form == "literal":
            return self._factor.solve(bd)
        s = self._fit.sqrt_lam
        scaled = s[:, None] * bd if bd.dim() == 2 else s * bd
        x = self._factor.solve(scaled, return_device=True)
        x = s[:, None] * x if x.dim() == 2 else s * x
        return dev.to_host(self.noise_var * x)


def lambda_bar(es, noise_var, backend=None, form="scaled"):
    return LambdaBarSolve(es, noise_var, backend=backend, form=form)


# keep dataclasses.replace importable for callers that tweak a model, as the reference's
# bench does (bench.py:254)
replace = replace
