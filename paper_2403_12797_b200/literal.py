"""method="literal" on the GPU: the reference's cross-check route (posterior.py:236-244, 256-260).

LamBar = diag(1/lam_f) + Phi^T Phi / sigma2 is factorized directly (SpdFactor, same jitter
schedule) and the mean goes through the reference's t1..t5 chain -- two Phi^T products
and one Phi product over the training rows, each generated on chip from the 1-D tables
(fagp_phi_tmatvec / fagp_phi_matvec), never materialising Phi.  The covariance inner matrix
``diag(lam_f) - lam_f * (g - g LamBar^{-1} g) * lam_f`` is folded into the same predict
operand the scaled route uses (pair form) or contracted against Phi* directly (p = 1).

Every elementwise step is one fagp_vec_op call that rounds like the numpy operator it
restates; torch only allocates.
"""

from __future__ import annotations

from . import _device as dev
from . import _lib
from .errors import NumericalError
from .mercer import LAMBDA_FLOOR_REL, raise_nonfinite

__all__ = ["phi_matvec", "phi_tmatvec", "vec_op", "lambda_bar_matrix", "literal_inner", "rowdot",
           "literal_posterior"]


def phi_matvec(basis, T, x, mean_const=0.0, flag_ptr=None):
    """mean_const + Phi x over the rows of table T (device)."""
    N = int(T.shape[0])
    out = dev.empty((N,), device=T.device)
    if N > 0:
        _lib.check(_lib.lib().fagp_phi_matvec(_lib.ptr(T), N, basis.ref, _lib.ptr(x), float(mean_const), _lib.ptr(out),
                                              flag_ptr, _lib.stream_handle()), "phi_matvec")
    return out


def phi_tmatvec(basis, T, v):
    """Phi^T v over the rows of table T (device; overwrites T's residual column)."""
    L = _lib.lib()
    N = int(T.shape[0])
    out = dev.empty((basis.m,), device=T.device)
    wsz = int(L.fagp_phi_tmatvec_workspace_size(N, basis.ref))
    ws = dev.empty((max(1, wsz // 8),), device=T.device)
    _lib.check(L.fagp_phi_tmatvec(_lib.ptr(T), N, basis.ref, _lib.ptr(v), _lib.ptr(out), _lib.ptr(ws), wsz,
                                  _lib.stream_handle()), "phi_tmatvec")
    return out


def vec_op(op, x, y=None, alpha=0.0):
    """One numpy elementwise operator on device vectors/matrices (fagp_vec_op)."""
    out = dev.empty(tuple(x.shape), device=x.device)
    _lib.check(_lib.lib().fagp_vec_op(int(op), int(x.numel()), _lib.ptr(x), _lib.ptr(y), float(alpha), _lib.ptr(out),
                                      _lib.stream_handle()), "vec_op")
    return out


def lambda_bar_matrix(G, lam_f, noise_var):
    """Explicit symmetric LamBar (LambdaBarSolve.matrix, posterior.py:184-188)."""
    m = int(G.shape[0])
    out = dev.empty((m, m), device=G.device)
    _lib.check(_lib.lib().fagp_lambda_bar(_lib.ptr(G), _lib.ptr(lam_f), m, float(noise_var), _lib.ptr(out),
                                          _lib.stream_handle()), "lambda_bar")
    return out


def literal_inner(mid, lam_f):
    """sym(diag(lam_f) - lam_f[:, None] * mid * lam_f[None, :]) (posterior.py:259-261)."""
    m = int(mid.shape[0])
    out = dev.empty((m, m), device=mid.device)
    _lib.check(_lib.lib().fagp_literal_inner(_lib.ptr(mid), _lib.ptr(lam_f), m, _lib.ptr(out),
                                             _lib.stream_handle()), "literal_inner")
    return out


def rowdot(A, B):
    n, k = int(A.shape[0]), int(A.shape[1])
    out = dev.empty((n,), device=A.device)
    _lib.check(_lib.lib().fagp_rowdot(_lib.ptr(A), _lib.ptr(B), n, k, _lib.ptr(out), _lib.stream_handle()), "rowdot")
    return out


def _features(basis, Ts):
    Ns = int(Ts.shape[0])
    phis = dev.empty((Ns, basis.m), device=Ts.device)
    if Ns > 0:
        _lib.check(_lib.lib().fagp_features(_lib.ptr(Ts), Ns, basis.ref, _lib.ptr(phis), None, _lib.stream_handle()),
                   "features")
    return phis


def literal_posterior(basis, T, Ts, yd, noise_var, mean_const, want_var=True, want_cov=False, fault_flip=False,
                      X=None, Xs=None, flags=None):
    """The literal route on staged tables T (train) / Ts (test).  Returns device
    (mean, var|None, cov|None).  ``flags``: the posterior's _Flags (checked, in the
    reference's validation order, before the factorisation)."""
    from .backend import SpdFactor
    from .linalg import dgemm
    from .posterior import gram_packed, gram_unpack

    L = _lib.lib()
    s = _lib.stream_handle()
    m = basis.m
    device = T.device
    sigma2 = float(noise_var)
    lam = dev.empty((m,), device=device)
    lam_f = dev.empty((m,), device=device)
    sq = dev.empty((m,), device=device)
    _lib.check(L.fagp_eigenvalues(basis.ref, LAMBDA_FLOOR_REL, _lib.ptr(lam), _lib.ptr(lam_f), _lib.ptr(sq), s),
               "eigenvalues")
    # LambdaBarSolve(form="literal") (posterior.py:168, 176): G = Phi^T Phi, factor LamBar
    packed = gram_packed(basis, T, None, 0.0, None if flags is None else flags.ptr(0))
    G, _ = gram_unpack(basis, packed)
    if flags is not None:
        fl = flags.read()
        if fl[0] & _lib.FLAG_X_NONFINITE:
            raise ValueError("X must be finite")
        if fl[0] & _lib.FLAG_PHI_NONFINITE:
            raise_nonfinite(T, X, basis)
        if fl[1] & _lib.FLAG_X_NONFINITE:
            raise ValueError("X must be finite")
        if int(Ts.shape[0]):
            raise_nonfinite(Ts, Xs, basis)
    fac = SpdFactor(lambda_bar_matrix(G, lam_f, sigma2), check_symmetric=False)
    # mean (posterior.py:237-247)
    r = vec_op(_lib.VEC_SUB_SCALAR, yd, alpha=mean_const)
    t1 = vec_op(_lib.VEC_DIV, r, alpha=sigma2)
    t2 = phi_tmatvec(basis, T, t1)
    t3 = fac.solve(t2, return_device=True)
    t4 = phi_matvec(basis, T, t3)
    t5 = vec_op(_lib.VEC_SUB_DIV, t1, t4, alpha=sigma2)
    u = phi_tmatvec(basis, T, t5)
    w = vec_op(_lib.VEC_MUL, lam_f, u)
    if fault_flip:
        w = w.neg()
    Ns = int(Ts.shape[0])
    var = cov = None
    if not (want_var or want_cov):
        return phi_matvec(basis, Ts, w, mean_const), None, None
    # inner (posterior.py:256-261): g = G / sigma2, mid = g - g @ solve(g)
    g = vec_op(_lib.VEC_DIV, G, alpha=sigma2)
    z = fac.solve(g, return_device=True)
    mid = vec_op(_lib.VEC_SUB, g, dgemm(g, z))
    inner = literal_inner(mid, lam_f)
    pair = _pair_form(basis)
    if pair:
        op = dev.empty((int(L.fagp_predict_operand_len(basis.ref)),), device=device)
        wsz = int(L.fagp_inner_operand_workspace_size(basis.ref))
        ws = dev.empty((max(1, wsz // 8),), device=device)
        _lib.check(L.fagp_inner_operand(_lib.ptr(inner), _lib.ptr(w), basis.ref, _lib.ptr(op), _lib.ptr(ws), wsz, s),
                   "inner_operand")
        mean = dev.empty((Ns,), device=device)
        var = dev.empty((Ns,), device=device) if want_var else None
        if Ns > 0:
            _lib.check(L.fagp_predict(_lib.ptr(Ts), Ns, basis.ref, _lib.ptr(op), 1.0, float(mean_const),
                                      _lib.ptr(mean), _lib.ptr(var), None, s), "predict")
    else:
        mean = phi_matvec(basis, Ts, w, mean_const)
    if want_cov or (want_var and not pair):
        phis = _features(basis, Ts)
        B = dgemm(phis, inner)
        if want_var and not pair:
            var = rowdot(phis, B)
        if want_cov:
            cov = dgemm(B, phis, trans_b=True)
            cov = 0.5 * (cov + cov.T)
    return mean, var, cov


def _pair_form(basis):
    """True when the library runs the modal kernels for this basis (2 <= p <= 8)."""
    st = _lib.lib().fagp_inner_operand(None, None, basis.ref, None, None, 0, None)
    if st == _lib.FAGP_EUNSUPPORTED:
        return False
    if st == _lib.FAGP_EINVAL:
        return True
    raise NumericalError(f"unexpected status {st} probing the operand form")
