"""GPU: method="literal" (the reference's cross-check route, posterior.py:236-262) and the
C-ABI pieces it is built from (fagp_phi_matvec / fagp_phi_tmatvec / fagp_vec_op /
fagp_lambda_bar / fagp_literal_inner / fagp_inner_operand / fagp_rowdot).

Tolerances: the elementwise pieces are bit-exact restatements of numpy expressions; the
Phi products match the oracle to 1e-13 (scaled); the literal posterior is ill-conditioned
by construction (LamBar carries 1/lam_f up to 1e14 on its diagonal), so its variance is
held to 10x the reference's OWN literal-vs-scaled disagreement on the same case (and never
looser than 1e-5 scaled), its mean to 1e-8 scaled.
"""

import numpy as np
import pytest

import fagp_oracle as O
import paper_2403_12797_b200 as F
from conftest import scaled_err
from paper_2403_12797_b200 import _device as dev
from paper_2403_12797_b200 import _lib
from paper_2403_12797_b200 import literal as lit
from paper_2403_12797_b200.mercer import Basis
from paper_2403_12797_b200.posterior import _stage_tables

pytestmark = pytest.mark.gpu

LITERAL_CASES = ["c1", "lin2", "ard4", "p1m40", "c5s"]


def _table(p, M, X, eps, rho):
    kernel = F.ArdKernelParams(tuple(F.KernelParams1D(float(e), float(r)) for e, r in zip(eps, rho)))
    basis = Basis(kernel, M, "rho_squared")
    Xd = dev.to_device(np.ascontiguousarray(X))
    return basis, _stage_tables(basis, Xd, None, _lib.stream_handle())


@pytest.mark.parametrize("p,M,N", [(1, 1, 7), (1, 12, 1001), (2, 5, 3333), (3, 10, 4097), (5, 4, 999), (8, 2, 300)])
def test_phi_products_against_oracle(p, M, N):
    rng = np.random.default_rng(p * 100 + M)
    X = rng.uniform(-1, 1, (N, p))
    eps, rho = rng.uniform(0.4, 1.5, p), rng.uniform(0.5, 2.0, p)
    basis, T = _table(p, M, X, eps, rho)
    phi = O.assemble_phi(X, list(eps), list(rho), M)
    x = rng.standard_normal(M**p)
    v = rng.standard_normal(N)
    y = dev.to_host(lit.phi_matvec(basis, T, dev.to_device(x), 0.75))
    assert scaled_err(y - 0.75, phi @ x) < 1e-13
    t = dev.to_host(lit.phi_tmatvec(basis, T, dev.to_device(v)))
    assert scaled_err(t, phi.T @ v) < 1e-13


def test_phi_tmatvec_empty_rows():
    basis, T = _table(2, 3, np.zeros((0, 2)), [1.0, 1.0], [1.0, 1.0])
    t = dev.to_host(lit.phi_tmatvec(basis, T, dev.empty((0,))))
    assert np.array_equal(t, np.zeros(9))


def test_vec_ops_bit_exact():
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal(1237) * 1e3, rng.standard_normal(1237)
    xd, yd = dev.to_device(x), dev.to_device(y)
    a = 0.0025
    assert np.array_equal(dev.to_host(lit.vec_op(_lib.VEC_DIV, xd, alpha=a)), x / a)
    assert np.array_equal(dev.to_host(lit.vec_op(_lib.VEC_SUB_DIV, xd, yd, alpha=a)), x - y / a)
    assert np.array_equal(dev.to_host(lit.vec_op(_lib.VEC_MUL, xd, yd)), x * y)
    assert np.array_equal(dev.to_host(lit.vec_op(_lib.VEC_SUB, xd, yd)), x - y)
    assert np.array_equal(dev.to_host(lit.vec_op(_lib.VEC_SUB_SCALAR, xd, alpha=-1.5)), x - (-1.5))
    with pytest.raises(ValueError):
        lit.vec_op(99, xd)


def test_lambda_bar_and_inner_bit_exact():
    rng = np.random.default_rng(4)
    m = 37
    A = rng.standard_normal((m, m))
    G = A @ A.T + 0.25 * rng.standard_normal((m, m))  # deliberately not symmetric
    lam_f = rng.uniform(1e-14, 1.0, m)
    s2 = 0.0025
    got = dev.to_host(lit.lambda_bar_matrix(dev.to_device(G), dev.to_device(lam_f), s2))
    ref = np.diag(1.0 / lam_f) + G / s2
    assert np.array_equal(got, 0.5 * (ref + ref.T))
    got = dev.to_host(lit.literal_inner(dev.to_device(G), dev.to_device(lam_f)))
    ref = np.diag(lam_f) - lam_f[:, None] * G * lam_f[None, :]
    assert np.array_equal(got, 0.5 * (ref + ref.T))


def test_rowdot():
    rng = np.random.default_rng(5)
    A, B = rng.standard_normal((301, 77)), rng.standard_normal((301, 77))
    got = dev.to_host(lit.rowdot(dev.to_device(A), dev.to_device(B)))
    np.testing.assert_allclose(got, np.einsum("ij,ij->i", A, B), rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("name", LITERAL_CASES)
def test_literal_posterior_parity(cases, name):
    c = cases[name]
    res = F.fagp_posterior(c.dataset(), c.Xs, c.model(), method="literal", delta2_variant=c.variant,
                           memory_cap=None)
    gap = scaled_err(c.ref["literal_var"], c.ref["var"])  # the reference's own route disagreement
    assert scaled_err(res.mean, c.ref["literal_mean"]) < 1e-8, scaled_err(res.mean, c.ref["literal_mean"])
    err = scaled_err(res.var, c.ref["literal_var"])
    assert err < max(1e-5, 10 * gap) and err < 1e-3, (err, gap)
    # and against the oracle's literal restatement
    ora = O.posterior_literal(c.X, c.y, c.Xs, c.eps, c.rho, c.M, c.noise_var, c.mean_const, c.variant)
    assert scaled_err(res.mean, ora["mean"]) < 1e-8


def test_scaled_and_literal_paths_agree():
    """test_posterior.py:106-113"""
    ds = F.generate(40, 1, seed=7, noise_std=0.1)
    rng = np.random.Generator(np.random.Philox(key=8))
    Xs = rng.uniform(-1.0, 1.0, size=(20, 1))
    model = F.GpModel(F.ArdKernelParams.isotropic(1, 1.0, 1.0), 1e-2, n_eigen=10)
    a = F.fagp_posterior(ds, Xs, model, want_cov=True, method="scaled")
    b = F.fagp_posterior(ds, Xs, model, want_cov=True, method="literal")
    scale = np.abs(a.mean).max()
    assert np.abs(a.mean - b.mean).max() / scale < 1e-8
    assert np.abs(a.cov - b.cov).max() / np.abs(a.cov).max() < 1e-8
    np.testing.assert_allclose(np.diag(b.cov), b.var, rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("p,M", [(2, 4), (3, 3)])
def test_literal_pair_form_cov_and_split_api(p, M):
    rng = np.random.default_rng(p)
    X = rng.uniform(-1, 1, (500, p))
    ds = F.Dataset(X=X, y=np.cos(X).sum(1), noise_std=0.0, seed=0, domain=((-1.0, 1.0),) * p)
    Xs = rng.uniform(-1, 1, (60, p))
    model = F.GpModel(F.ArdKernelParams.isotropic(p, 1.0, 1.0), 1e-2, mean_const=0.1, n_eigen=M)
    a = F.fagp_posterior(ds, Xs, model, want_cov=True, method="scaled")
    b = F.fagp_posterior(ds, Xs, model, want_cov=True, method="literal")
    assert np.abs(a.mean - b.mean).max() / np.abs(a.mean).max() < 1e-8
    assert np.abs(a.cov - b.cov).max() / np.abs(a.cov).max() < 1e-7
    np.testing.assert_allclose(np.diag(b.cov), b.var, rtol=1e-8, atol=1e-14)
    es, ess = F.eigensystem(X, model.kernel, M), F.eigensystem(Xs, model.kernel, M)
    c = F.fagp_posterior_from_eigensystems(es, ess, ds.y, model, method="literal")
    np.testing.assert_array_equal(c.mean, b.mean)
    np.testing.assert_array_equal(c.var, b.var)


def test_literal_fault_injection_flips_mean():
    ds = F.generate(200, 2, seed=1, noise_std=0.05)
    Xs = np.random.default_rng(0).uniform(-1, 1, (30, 2))
    model = F.GpModel(F.ArdKernelParams.isotropic(2, 1.0, 1.0), 1e-2, mean_const=0.0, n_eigen=5)
    a = F.fagp_posterior(ds, Xs, model, method="literal")
    F.set_fault_injection(True)
    try:
        b = F.fagp_posterior(ds, Xs, model, method="literal")
    finally:
        F.set_fault_injection(False)
    np.testing.assert_allclose(b.mean, -a.mean, rtol=1e-12)


def test_literal_rejects_nonfinite_x():
    ds = F.generate(50, 2, seed=1, noise_std=0.05)
    X = ds.X.copy()
    X[3, 1] = np.nan
    bad = F.Dataset(X=X, y=ds.y, noise_std=0.05, seed=1, domain=ds.domain)
    model = F.GpModel(F.ArdKernelParams.isotropic(2, 1.0, 1.0), 1e-2, n_eigen=4)
    with pytest.raises(ValueError, match="finite"):
        F.fagp_posterior(bad, np.zeros((3, 2)), model, method="literal")
