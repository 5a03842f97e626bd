"""Thin device wrappers over the dense FP64 kernels of libfagp_b200.so (generic DGEMM,
Cholesky, cho_solve, triangular inverse).  Row-major CUDA float64 tensors in and out."""

from __future__ import annotations

from . import _device as dev
from . import _lib


def dgemm(a, b, trans_a=False, trans_b=False, alpha=1.0, beta=0.0, out=None):
    """alpha * op(a) @ op(b) + beta * out on the FP64 DMMA kernel (fagp_dgemm)."""
    a = dev.to_device(a)
    b = dev.to_device(b)
    b2 = b.reshape(-1, 1) if b.dim() == 1 else b
    M, K = (a.shape[1], a.shape[0]) if trans_a else (a.shape[0], a.shape[1])
    Kb, N = (b2.shape[1], b2.shape[0]) if trans_b else (b2.shape[0], b2.shape[1])
    if K != Kb:
        raise ValueError(f"inner dimensions do not conform: op(a) is {(M, K)}, op(b) is {(Kb, N)}")
    if out is None:
        out = dev.empty((M, N), device=a.device)
        beta = 0.0
    _lib.check(_lib.lib().fagp_dgemm(int(trans_a), int(trans_b), M, N, K, float(alpha), _lib.ptr(a), a.shape[1],
                                     _lib.ptr(b2), b2.shape[1], float(beta), _lib.ptr(out), N,
                                     _lib.stream_handle()), "dgemm")
    return out.reshape(-1) if b.dim() == 1 else out


def potrf(a):
    """Lower Cholesky factor (no jitter).  Returns (L, info) with LAPACK's 1-based info."""
    L = dev.to_device(a).clone()
    m = int(L.shape[0])
    info = dev.zeros((1,), dtype="int32", device=L.device)
    wsz = int(_lib.lib().fagp_potrf_workspace_size(m))
    ws = dev.empty((max(1, wsz // 8),), device=L.device)
    _lib.check(_lib.lib().fagp_potrf(_lib.ptr(L), m, _lib.ptr(info), _lib.ptr(ws), wsz, _lib.stream_handle()),
               "potrf")
    return L, int(dev.to_host(info)[0])


def spd_inverse(a):
    """A^{-1} of an SPD matrix (Cholesky + triangular inverse + X^T X in one persistent kernel).
    Returns (Ainv, info) with dpotrf's 1-based info on breakdown."""
    A = dev.to_device(a).clone()
    m = int(A.shape[0])
    Ainv = dev.empty((m, m), device=A.device)
    info = dev.zeros((1,), dtype="int32", device=A.device)
    wsz = int(_lib.lib().fagp_spd_inverse_workspace_size(m))
    ws = dev.empty((max(1, -(-wsz // 8)),), device=A.device)
    _lib.check(_lib.lib().fagp_spd_inverse(_lib.ptr(A), m, _lib.ptr(Ainv), _lib.ptr(info), _lib.ptr(ws), wsz,
                                           _lib.stream_handle()), "spd_inverse")
    return Ainv, int(dev.to_host(info)[0])


def potrs(L, b):
    """A^{-1} b given the lower factor (cho_solve, backend.py:191-193)."""
    m = int(L.shape[0])
    bt = dev.to_device(b)
    one = bt.dim() == 1
    B = bt.reshape(m, -1).clone().contiguous()
    _lib.check(_lib.lib().fagp_potrs(_lib.ptr(L), m, _lib.ptr(B), int(B.shape[1]), _lib.stream_handle()), "potrs")
    return B.reshape(-1) if one else B


def trtri(L, s=None):
    """L^{-1} diag(s) (lower triangular)."""
    m = int(L.shape[0])
    V = dev.empty((m, m), device=L.device)
    wsz = int(_lib.lib().fagp_trtri_workspace_size(m))
    ws = dev.empty((max(1, wsz // 8),), device=L.device)
    sd = None if s is None else dev.to_device(s)
    _lib.check(_lib.lib().fagp_trtri(_lib.ptr(L), _lib.ptr(sd), m, _lib.ptr(V), _lib.ptr(ws), wsz,
                                     _lib.stream_handle()), "trtri")
    return V
