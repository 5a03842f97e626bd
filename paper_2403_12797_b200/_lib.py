"""ctypes binding of libfagp_b200.so (the C ABI declared in include/fagp_b200.h).

This is the only module that touches the shared library.  Every compute entry point is
reached through :func:`lib`, which loads the in-tree .so and refuses to run without it:
there is no CPU fallback anywhere in the package.  Status codes are mapped onto the
reference's exception types (errors.py:6-21) by :func:`check`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import BudgetError, NumericalError

LIB_PATH = Path(__file__).resolve().parent / "libfagp_b200.so"

FAGP_OK = 0
FAGP_EINVAL = 1
FAGP_EBUDGET = 2
FAGP_ENOTPD = 3
FAGP_ENONFINITE = 4
FAGP_ECUDA = 5
FAGP_EWORKSPACE = 6
FAGP_EUNSUPPORTED = 7

FLAG_X_NONFINITE = 1
FLAG_PHI_NONFINITE = 2
FLAG_STALLED = 4  # a pipelined Gram never saw an input chunk's signal

MAX_P = 16
ABI_VERSION = 1


class FagpBasis(ctypes.Structure):
    """Mirror of ``struct fagp_basis``."""

    _fields_ = [
        ("p", ctypes.c_int32),
        ("M", ctypes.c_int32),
        ("m", ctypes.c_int64),
        ("table", ctypes.c_void_p),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double
_SZ = ctypes.c_size_t
_BASIS = ctypes.POINTER(FagpBasis)

# name -> (restype, argtypes); must list every symbol in include/fagp_b200.h
SIGNATURES = {
    "fagp_abi_version": (ctypes.c_int, []),
    "fagp_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "fagp_basis_table_len": (_I64, [_I32, _I32]),
    "fagp_modal_coeffs": (ctypes.c_int, [_I32, _P]),
    "fagp_multi_indices": (ctypes.c_int, [_I32, _I32, _P]),
    "fagp_read_flags": (ctypes.c_int, [_P, _P, _P]),
    "fagp_eigenvalues": (ctypes.c_int, [_BASIS, _D, _P, _P, _P, _P]),
    "fagp_hermite": (ctypes.c_int, [_P, _I64, _I32, _P, _P]),
    "fagp_table_width": (_I32, [_I32, _I32]),
    "fagp_basis_eval": (ctypes.c_int, [_P, _I64, _BASIS, _P, _D, _P, _P, _P]),
    "fagp_set_residual": (ctypes.c_int, [_P, _I64, _BASIS, _P, _D, _P]),
    "fagp_features": (ctypes.c_int, [_P, _I64, _BASIS, _P, _P, _P]),
    "fagp_find_nonfinite": (ctypes.c_int, [_P, _I64, _BASIS, _P, _P]),
    "fagp_gram_len": (_I64, [_BASIS]),
    "fagp_gram_unpack_workspace_size": (ctypes.c_size_t, [_BASIS]),
    "fagp_gram_unpack": (ctypes.c_int, [_P, _BASIS, _P, _P, _P, ctypes.c_size_t, _P]),
    "fagp_gram_workspace_size": (_SZ, [_I64, _BASIS]),
    "fagp_gram": (ctypes.c_int, [_P, _I64, _BASIS, _P, _P, _SZ, _P, _P]),
    "fagp_gram_x_workspace_size": (_SZ, [_I64, _BASIS]),
    "fagp_gram_x": (ctypes.c_int, [_P, _I64, _BASIS, _P, _D, _P, _P, _SZ, _P, _P]),
    "fagp_gram_x_chunks": (_I32, [_I64, _BASIS]),
    "fagp_gram_x_upload_chunk": (ctypes.c_int, [_P, _P, _I64, _BASIS, _I32, _P, _P, _P]),
    "fagp_gram_x_chunk": (ctypes.c_int, [_P, _I64, _BASIS, _P, _D, _I32, _P, _P, _SZ, _P, _P]),
    "fagp_gram_x_pipelined": (ctypes.c_int, [_P, _I64, _BASIS, _P, _D, _P, _P, _P, _SZ, _P, _P]),
    "fagp_gram_x_signal": (ctypes.c_int, [_P, _I32, _P]),
    "fagp_predict_x_wave_rows": (_I64, [_BASIS]),
    "fagp_route_info": (ctypes.c_int, [_I64, _I64, _BASIS, _P]),
    "fagp_host_copy": (ctypes.c_int, [_P, _P, _SZ, _I32]),
    "fagp_host_mapped": (ctypes.c_int, [_P, _SZ]),
    "fagp_host_copy_2d": (ctypes.c_int, [_P, _SZ, _P, _SZ, _SZ, _SZ, _I32]),
    "fagp_gram_x_stage_chunk": (ctypes.c_int, [_P, _P, _I64, _BASIS, _I32, _P, _P, _I32]),
    "fagp_predict_x_workspace_size": (_SZ, [_I64, _BASIS]),
    "fagp_predict_x": (ctypes.c_int, [_P, _I64, _BASIS, _P, _D, _D, _P, _P, _P, _P, _SZ, _P]),
    "fagp_factor_workspace_size": (_SZ, [_I64]),
    "fagp_predict_operand_len": (_I64, [_BASIS]),
    "fagp_factor": (ctypes.c_int, [_P, _BASIS, _P, _D, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "fagp_factor_inv": (ctypes.c_int, [_P, _BASIS, _P, _D, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "fagp_factor_inv_async": (ctypes.c_int, [_P, _BASIS, _P, _D, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "fagp_set_mean_weights": (ctypes.c_int, [_P, _P, _BASIS, _P]),
    "fagp_potrf_workspace_size": (_SZ, [_I64]),
    "fagp_potrf": (ctypes.c_int, [_P, _I64, _P, _P, _SZ, _P]),
    "fagp_potrs": (ctypes.c_int, [_P, _I64, _P, _I64, _P]),
    "fagp_spd_inverse_workspace_size": (_SZ, [_I64]),
    "fagp_spd_inverse": (ctypes.c_int, [_P, _I64, _P, _P, _P, _SZ, _P]),
    "fagp_dgemm": (ctypes.c_int, [_I32, _I32, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64, _P]),
    "fagp_trtri_workspace_size": (_SZ, [_I64]),
    "fagp_trtri": (ctypes.c_int, [_P, _P, _I64, _P, _P, _SZ, _P]),
    "fagp_predict": (ctypes.c_int, [_P, _I64, _BASIS, _P, _D, _D, _P, _P, _P, _P]),
    "fagp_phi_matvec": (ctypes.c_int, [_P, _I64, _BASIS, _P, _D, _P, _P, _P]),
    "fagp_phi_tmatvec_workspace_size": (ctypes.c_size_t, [_I64, _BASIS]),
    "fagp_phi_tmatvec": (ctypes.c_int, [_P, _I64, _BASIS, _P, _P, _P, ctypes.c_size_t, _P]),
    "fagp_vec_op": (ctypes.c_int, [ctypes.c_int32, _I64, _P, _P, _D, _P, _P]),
    "fagp_lambda_bar": (ctypes.c_int, [_P, _P, _I64, _D, _P, _P]),
    "fagp_literal_inner": (ctypes.c_int, [_P, _P, _I64, _P, _P]),
    "fagp_inner_operand_workspace_size": (ctypes.c_size_t, [_BASIS]),
    "fagp_inner_operand": (ctypes.c_int, [_P, _P, _BASIS, _P, _P, ctypes.c_size_t, _P]),
    "fagp_rowdot": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P]),
    "fagp_se_gram": (ctypes.c_int, [_P, _I64, _P, _I64, _I32, _P, _D, _P, _I64, _P]),
}

_LIB = None


class ExtensionMissing(RuntimeError):
    """The CUDA extension is not built or no CUDA device is present (no CPU fallback)."""


def load(path=None):
    """Load the shared library (no GPU needed) and bind every declared symbol."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path else Path(os.environ.get("FAGP_LIB_PATH", str(LIB_PATH)))
    if not p.exists():
        raise ExtensionMissing(
            f"{p} is missing: build it with `python -m paper_2403_12797_b200._build` "
            "(this package has no CPU fallback)"
        )
    # torch ships the CUDA runtime; import it first so libcudart.so.12 resolves
    try:
        import torch  # noqa: F401
    except ImportError:  # pragma: no cover
        pass
    handle = ctypes.CDLL(str(p), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.fagp_abi_version() != ABI_VERSION:
        raise ExtensionMissing(f"{p} has ABI {handle.fagp_abi_version()}, expected {ABI_VERSION}")
    if path is None:
        _LIB = handle
    return handle


def lib():
    """The loaded library, for a compute call: requires a CUDA device."""
    import torch

    if not torch.cuda.is_available():
        raise ExtensionMissing("no CUDA device: paper_2403_12797_b200 runs only on the GPU (no CPU fallback)")
    return load()


def strerror(status):
    return load().fagp_strerror(int(status)).decode()


def check(status, what="", pivot_index=None):
    """Raise the reference's exception type for a non-OK status."""
    if status == FAGP_OK:
        return
    msg = f"{what}: {strerror(status)}" if what else strerror(status)
    if status == FAGP_ENOTPD:
        raise NumericalError(msg, pivot_index=pivot_index)
    if status == FAGP_ENONFINITE:
        raise NumericalError(msg)
    if status == FAGP_EBUDGET:
        raise BudgetError(msg)
    if status in (FAGP_EINVAL, FAGP_EUNSUPPORTED):
        raise ValueError(msg)
    raise RuntimeError(msg)


def ptr(t):
    """Device (or host) address of a torch tensor / numpy array, or None."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(t.ctypes.data)


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)

# fagp_vec_op codes (include/fagp_b200.h)
VEC_DIV = 0
VEC_SUB_DIV = 1
VEC_MUL = 2
VEC_SUB = 3
VEC_SUB_SCALAR = 4
