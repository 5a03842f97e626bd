"""CPU: host-side logic (no GPU): bit-exact constants, validation, types, error mapping."""

import math
import os

import numpy as np
import pytest

import fagp_oracle as O
import paper_2403_12797_b200 as F
from paper_2403_12797_b200 import _lib
from paper_2403_12797_b200.backend import ENV_MAX_WORKERS, PHASES, TimingRecord, phase_scope


def test_shape_params_kats():
    sp = F.shape_params(F.KernelParams1D(1.0, 2.0), 2)
    assert sp.beta == pytest.approx(1.1892071150027211, rel=1e-15)
    assert sp.delta2 == pytest.approx(0.8284271247461901, rel=1e-15)
    assert sp.gamma[0] == pytest.approx(1.0905077326652577, rel=1e-15)
    sp0 = F.shape_params(F.KernelParams1D(0.0, 1.0), 3)
    assert sp0.beta == 1.0 and sp0.delta2 == 0.0
    with pytest.raises(ValueError, match="variant"):
        F.shape_params(F.KernelParams1D(1.0, 1.0), 1, delta2_variant="bogus")


@pytest.mark.parametrize("eps,rho,n", [(1.0, 1.0, 10), (1.0, 2.0, 7), (0.37, 0.81, 40), (0.0, 1.0, 4)])
def test_eigenvalues_1d_bit_exact_vs_oracle(eps, rho, n):
    for var in (F.DELTA2_RHO_SQUARED, F.DELTA2_RHO_LINEAR):
        assert np.array_equal(F.eigenvalues_1d(F.KernelParams1D(eps, rho), n, var), O.eigenvalues_1d(eps, rho, n, var))


def test_basis_table_layout_bit_exact(cases):
    for name in ("c1", "ard4", "lin2"):
        c = cases[name]
        tab = F.basis_table(c.kernel(), c.M, c.variant)
        p = c.p
        for d in range(p):
            beta, d2 = O.beta_delta2(c.eps[d], c.rho[d], c.variant)
            assert tab[d] == c.rho[d] * beta
            assert tab[p + d] == -d2
            assert tab[2 * p + d] == math.sqrt(beta)
            assert np.array_equal(tab[3 * p + d * c.M: 3 * p + (d + 1) * c.M],
                                  O.eigenvalues_1d(c.eps[d], c.rho[d], c.M, c.variant))
        assert tab.shape == (int(_lib.load().fagp_basis_table_len(p, c.M)),)


def test_bench_constants():
    """beta = 5^(1/4), delta2 = 0.618..., lam1 = 0.618..., ratio 0.381... at eps=rho=1"""
    sp = F.shape_params(F.KernelParams1D(1.0, 1.0), 1)
    assert sp.beta == pytest.approx(1.4953487812212205, rel=1e-15)
    assert sp.delta2 == pytest.approx(0.6180339887498947, rel=1e-15)
    lam = F.eigenvalues_1d(F.KernelParams1D(1.0, 1.0), 2)
    assert lam[0] == pytest.approx(0.6180339887498949, rel=1e-15)
    assert lam[1] / lam[0] == pytest.approx(0.38196601125010515, rel=1e-14)


def test_multi_indices_host_abi_bit_exact(golden):
    for key, ref in golden.items():
        if key.startswith("indices/"):
            n, p = (int(v) for v in key.split("/")[1].split("_"))
            got = F.multi_indices(n, p)
            assert got.dtype == np.int64 and np.array_equal(got, ref)
    with pytest.raises(F.BudgetError, match="4\\^3"):
        F.multi_indices(4, 3, max_count=63)


def test_estimate_bytes_formula():
    m = 3**2
    assert F.estimate_bytes(100, 3, 2) == 8 * (100 * m + m * m + 2 * m)


def test_types_validation():
    with pytest.raises(ValueError, match="epsilon"):
        F.KernelParams1D(-1.0)
    with pytest.raises(ValueError, match="rho"):
        F.KernelParams1D(1.0, 0.0)
    with pytest.raises(ValueError, match="at least one"):
        F.ArdKernelParams(())
    with pytest.raises(TypeError):
        F.ArdKernelParams((1.0,))
    k = F.ArdKernelParams.isotropic(3, 0.5, 2.0)
    assert k.p == 3 and np.array_equal(k.epsilons, [0.5] * 3) and np.array_equal(k.rhos, [2.0] * 3)
    with pytest.raises(ValueError, match="noise_var"):
        F.GpModel(k, noise_var=0.0)
    with pytest.raises(ValueError, match="n_eigen"):
        F.GpModel(k, noise_var=1.0, n_eigen=0)


def test_duck_typed_reference_params():
    from paper_2403_12797_b200.kernels import as_ard

    class P1:
        epsilon, rho = 0.7, 1.3

    class Ard:
        per_dim = (P1(), P1())

    k = as_ard(Ard())
    assert k == F.ArdKernelParams((F.KernelParams1D(0.7, 1.3),) * 2)


def test_backend_construction(monkeypatch):
    with pytest.raises(ValueError, match="mode"):
        F.Backend("gpu")
    with pytest.raises(ValueError, match="workers"):
        F.Backend("parallel", workers=0)
    monkeypatch.setenv(ENV_MAX_WORKERS, "2")
    assert F.Backend("parallel", workers=8).workers == 2
    monkeypatch.delenv(ENV_MAX_WORKERS)
    assert F.Backend("parallel", workers=8).workers == 8


def test_phase_timing():
    rec = TimingRecord()
    assert rec.total_s == 0.0
    with phase_scope(rec, "eigen"):
        pass
    with pytest.raises(RuntimeError, match="nest"):
        with phase_scope(rec, "setup"):
            with phase_scope(rec, "mean"):
                pass
    with pytest.raises(ValueError):
        rec.phase_seconds("bogus")
    assert PHASES == ("setup", "eigen", "mean", "retrieve")


def test_status_mapping():
    with pytest.raises(F.NumericalError) as ei:
        _lib.check(_lib.FAGP_ENOTPD, "x", pivot_index=7)
    assert ei.value.pivot_index == 7
    with pytest.raises(ValueError):
        _lib.check(_lib.FAGP_EINVAL)
    with pytest.raises(F.BudgetError):
        _lib.check(_lib.FAGP_EBUDGET)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.FAGP_ECUDA)
    _lib.check(_lib.FAGP_OK)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.ExtensionMissing):
        F.fagp_posterior(F.generate(10, 1, 0), np.zeros((2, 1)), F.GpModel(F.ArdKernelParams.isotropic(1, 1.0), 1.0,
                                                                           n_eigen=3))


def test_datagen_matches_reference_seeds(cases):
    # Case() already regenerates inputs and checks them against the reference's checksums
    assert cases["c1"].X.shape == (1000, 1)
    ds = F.generate(5, 2, seed=123)
    assert ds.X.shape == (5, 2) and ds.y.shape == (5,)
    with pytest.raises(ValueError):
        F.generate(0, 1, 1)


def test_package_imports_without_gpu():
    assert F.__version__ and callable(F.fagp_posterior)
    assert os.path.exists(_lib.LIB_PATH)
