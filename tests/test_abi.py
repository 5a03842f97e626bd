"""CPU: the C-ABI library loads and exports every symbol include/fagp_b200.h declares."""

import ctypes
import re
from pathlib import Path

from paper_2403_12797_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "fagp_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(fagp_[a-z0-9_]+)\s*\(", text))


def test_header_declares_expected_surface():
    names = declared_functions()
    for must in ("fagp_gram", "fagp_factor", "fagp_predict", "fagp_basis_eval", "fagp_multi_indices",
                 "fagp_eigenvalues", "fagp_potrf", "fagp_potrs", "fagp_trtri", "fagp_strerror"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_bindings_cover_header():
    assert declared_functions() == set(_lib.SIGNATURES)


def test_host_only_entry_points():
    lib = _lib.load()
    assert lib.fagp_abi_version() == _lib.ABI_VERSION
    assert lib.fagp_strerror(_lib.FAGP_ENOTPD) == b"matrix is not positive definite"
    assert lib.fagp_basis_table_len(3, 10) == 3 * 3 + 30 + 55 * 19  # + modal coefficients
    b3 = _lib.FagpBasis(3, 10, 1000, 8)  # table pointer is not dereferenced by host-only calls
    assert lib.fagp_gram_len(ctypes.byref(b3)) == 19**3 + 1000  # modal form [K | t]
    b1 = _lib.FagpBasis(1, 10, 10, 8)
    assert lib.fagp_gram_len(ctypes.byref(b1)) == 11 * 12 // 2  # p == 1: packed [Phi | r] SYRK
    assert lib.fagp_predict_operand_len(ctypes.byref(b1)) == 32 * 128
    assert lib.fagp_predict_operand_len(ctypes.byref(b3)) == 368 * 24 + 1000  # C'' (KP x NP) | w
    assert lib.fagp_factor_workspace_size(1000) > 0
    assert lib.fagp_table_width(3, 10) == 34 + 60  # phi-section | g-section
    assert lib.fagp_table_width(1, 10) == 14
    b = _lib.FagpBasis(3, 10, 1000, None)
    assert lib.fagp_gram_workspace_size(1000000, ctypes.byref(b)) == 0  # null table is rejected
    assert lib.fagp_gram_workspace_size(1000000, ctypes.byref(b3)) > 0
    buf = (ctypes.c_int64 * 24)()
    assert lib.fagp_multi_indices(2, 3, buf) == 0
    assert list(buf)[:6] == [1, 1, 1, 1, 1, 2]
    assert lib.fagp_multi_indices(0, 3, buf) == _lib.FAGP_EINVAL


def test_host_copy_streams_bitwise():
    """fagp_host_copy (threads + non-temporal stores: the host staging of numpy inputs) is a plain
    memcpy: bitwise, any length, any destination alignment, any thread count."""
    import numpy as np

    from paper_2403_12797_b200 import _lib

    L = _lib.load()
    rng = np.random.default_rng(5)
    for n, off, th in [(0, 0, 4), (1, 0, 1), (1001, 1, 3), (3_000_003, 0, 8), (5_000_001, 1, 16)]:
        a = rng.standard_normal(n)
        buf = np.zeros(n + 2)
        b = buf[off:off + n]
        assert L.fagp_host_copy(b.ctypes.data if n else None, a.ctypes.data if n else None, a.nbytes, th) == 0
        assert np.array_equal(a, b)
        assert buf[off + n:].sum() == 0.0 and (off == 0 or buf[0] == 0.0)
