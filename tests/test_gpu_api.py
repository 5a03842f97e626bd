"""GPU: the reference's behavioural contract, exercised through this package's API.

Each test restates a check of /root/reference/pkg/tests (file:line in the docstring) against
the CUDA implementation.
"""

import numpy as np
import pytest

import paper_2403_12797_b200 as F
import paper_2403_12797_b200.posterior as post
from paper_2403_12797_b200 import (
    ArdKernelParams,
    Backend,
    BudgetError,
    GpModel,
    KernelParams1D,
    NumericalError,
    SpdFactor,
    spd_solve,
)

pytestmark = pytest.mark.gpu

UNIT_1D = ArdKernelParams.isotropic(1, 1.0, 1.0)


class DS:
    def __init__(self, X, y):
        self.X = np.atleast_2d(np.asarray(X, dtype=float))
        self.y = np.asarray(y, dtype=float)


def cos_problem(N, Ns, p=1, seed=42, noise_std=0.1):
    ds = F.generate(N, p, seed=seed, noise_std=noise_std)
    rng = np.random.Generator(np.random.Philox(key=seed + 1))
    return ds, rng.uniform(-1.0, 1.0, size=(Ns, p))


def test_rank_one_constant_kernel():
    """test_posterior.py:78-83"""
    res = F.fagp_posterior(DS([[0.0]], [1.0]), [[0.0]], GpModel(ArdKernelParams.isotropic(1, 0.0), 1.0, n_eigen=1))
    assert res.mean == pytest.approx([0.5], rel=1e-14)


def test_zero_residual_returns_prior_mean_bitwise():
    """test_posterior.py:85-91"""
    rng = np.random.default_rng(2)
    X = rng.uniform(-1, 1, size=(30, 1))
    model = GpModel(UNIT_1D, noise_var=1e-2, mean_const=-1.5, n_eigen=10)
    res = F.fagp_posterior(DS(X, np.full(30, -1.5)), rng.uniform(-1, 1, size=(9, 1)), model)
    assert np.array_equal(res.mean, np.full(9, -1.5))
    # same at a tensor-core-sized problem
    X3 = rng.uniform(-1, 1, size=(5000, 3))
    m3 = GpModel(ArdKernelParams.isotropic(3, 1.0), 0.0025, mean_const=3.25, n_eigen=10)
    r3 = F.fagp_posterior(DS(X3, np.full(5000, 3.25)), rng.uniform(-1, 1, size=(777, 3)), m3, memory_cap=None)
    assert np.array_equal(r3.mean, np.full(777, 3.25))


def test_requires_n_eigen():
    with pytest.raises(ValueError, match="n_eigen"):
        F.fagp_posterior(DS([[0.0]], [1.0]), [[0.0]], GpModel(UNIT_1D, 1.0))


def test_noise_var_validation():
    with pytest.raises(ValueError, match="noise_var"):
        GpModel(UNIT_1D, noise_var=0.0)


def test_dimension_checks():
    with pytest.raises(ValueError, match="columns"):
        F.fagp_posterior(DS(np.zeros((3, 2)), np.zeros(3)), np.zeros((2, 1)), GpModel(UNIT_1D, 1.0, n_eigen=3))
    with pytest.raises(ValueError, match="y has shape"):
        F.fagp_posterior(DS(np.zeros((3, 1)), np.zeros(4)), np.zeros((2, 1)), GpModel(UNIT_1D, 1.0, n_eigen=3))


def test_budget_propagates_and_cap_is_exact():
    """test_posterior.py:140-162"""
    ds, Xs = cos_problem(100, 10, p=2, seed=3)
    with pytest.raises(BudgetError):
        F.fagp_posterior(ds, Xs, GpModel(ArdKernelParams.isotropic(2, 1.0), 1e-2, n_eigen=20), memory_cap=1 << 10)
    N, n = 120, 7
    ds, Xs = cos_problem(N, 40, seed=21)
    model = GpModel(UNIT_1D, 1e-2, n_eigen=n)
    cap = F.estimate_bytes(N, n, 1)
    assert np.all(np.isfinite(F.fagp_posterior(ds, Xs, model, memory_cap=cap).mean))
    with pytest.raises(BudgetError):
        F.fagp_posterior(ds, Xs, model, memory_cap=cap - 1)


def test_eigensystem_budget_carries_n_features():
    """test_mercer.py:245-251"""
    with pytest.raises(BudgetError) as ei:
        F.eigensystem(np.zeros((10000, 4)), ArdKernelParams.isotropic(4, 1.0), 10, memory_cap=1 << 20)
    assert ei.value.n_features == 10**4 and "cap" in str(ei.value)


def test_nonfinite_x_rejected():
    """test_mercer.py:255-259"""
    with pytest.raises(ValueError, match="finite"):
        F.eigensystem(np.array([[np.inf]]), ArdKernelParams((KernelParams1D(1.0, 1.0),)), 2)
    with pytest.raises(ValueError, match="finite"):
        F.fagp_posterior(DS([[0.0], [np.nan]], [1.0, 2.0]), [[0.0]], GpModel(UNIT_1D, 1.0, n_eigen=3))


def test_nonfinite_feature_names_entry():
    """test_mercer.py:261-270: eps = 0 leaves degree-2 growth undamped -> overflow at row 1, col 2"""
    params = ArdKernelParams((KernelParams1D(0.0, 1.0),))
    with pytest.raises(NumericalError, match=r"row 1, column 2"):
        F.eigensystem(np.array([[0.0], [1e200]]), params, 3)
    with pytest.raises(NumericalError, match=r"row 1, column 2"):
        F.fagp_posterior(DS([[0.0], [1e200]], [1.0, 2.0]), [[0.0]], GpModel(params, 1.0, n_eigen=3))


def test_fault_injection_flips_mean():
    """test_posterior.py:164-173"""
    ds, Xs = cos_problem(30, 10, seed=5)
    model = GpModel(UNIT_1D, 1e-2, n_eigen=8)
    clean = F.fagp_posterior(ds, Xs, model)
    post.set_fault_injection(True)
    try:
        faulty = F.fagp_posterior(ds, Xs, model)
    finally:
        post.set_fault_injection(False)
    np.testing.assert_allclose(faulty.mean, -clean.mean, rtol=1e-12)


def test_covariance_sanity():
    """test_posterior.py:115-124"""
    ds, Xs = cos_problem(60, 40, seed=11)
    model = GpModel(UNIT_1D, 1e-2, n_eigen=15)
    res = F.fagp_posterior(ds, Xs, model, want_cov=True)
    assert np.abs(res.cov - res.cov.T).max() < 1e-9
    assert res.var.min() >= -1e-9
    es = F.eigensystem(Xs, UNIT_1D, 15)
    prior_var = np.einsum("ij,j,ij->i", es.phi, es.lam_floored, es.phi)
    assert np.all(res.var <= prior_var + 1e-9)


def test_lambda_bar_scalar_case():
    """test_posterior.py:177-184"""
    es = F.eigensystem(np.zeros((4, 1)), ArdKernelParams.isotropic(1, 0.0), 1)
    assert np.array_equal(es.phi, np.ones((4, 1)))
    h = F.lambda_bar(es, 1.0)
    np.testing.assert_allclose(h.matrix, [[5.0]], rtol=1e-15)
    assert h.solve(np.array([5.0])) == pytest.approx([1.0], rel=1e-12)


def test_lambda_bar_matrix_symmetric_and_solve():
    """test_posterior.py:186-201"""
    rng = np.random.default_rng(7)
    es = F.eigensystem(rng.uniform(-1, 1, size=(30, 1)), UNIT_1D, 5)
    for form in ("scaled", "literal"):
        h = F.lambda_bar(es, 0.3, form=form)
        m = h.matrix
        assert np.abs(m - m.T).max() == 0.0
        b = rng.normal(size=5)
        np.testing.assert_allclose(h.solve(b), np.linalg.inv(m) @ b, rtol=1e-10, atol=1e-12)


def test_woodbury_identity():
    """test_posterior.py:203-216"""
    rng = np.random.default_rng(8)
    for _ in range(3):
        es = F.eigensystem(rng.uniform(-1, 1, size=(30, 1)), UNIT_1D, 5)
        sigma2 = float(rng.uniform(0.1, 1.0))
        h = F.lambda_bar(es, sigma2)
        phi, lam = es.phi, es.lam_floored
        direct = np.linalg.inv(phi @ (lam[:, None] * phi.T) + sigma2 * np.eye(30))
        low_rank = np.eye(30) / sigma2 - (phi @ h.solve(phi.T)) / sigma2**2
        assert np.abs(low_rank - direct).max() / np.abs(direct).max() < 1e-8


def test_spd_solve_contract(golden):
    """test_backend.py:111-142"""
    rng = np.random.default_rng(7)
    b = rng.normal(size=(6, 3))
    assert np.array_equal(spd_solve(np.eye(6), b), b)
    np.testing.assert_allclose(spd_solve(np.diag([2.0, 4.0]), np.array([2.0, 4.0])), [1.0, 1.0], rtol=1e-15)
    a = rng.normal(size=(20, 20))
    m = a.T @ a + np.eye(20)
    bb = rng.normal(size=(20, 4))
    assert np.abs(m @ spd_solve(m, bb) - bb).max() / np.abs(bb).max() < 1e-10
    f = SpdFactor(golden["spd/near_singular"])
    assert f.jitter == float(golden["spd/near_singular_jitter"]) and f.jitter > 0
    assert np.all(np.isfinite(f.solve(np.ones(5))))
    with pytest.raises(NumericalError) as ei:
        spd_solve(np.diag([1.0, -1.0]), np.ones(2))
    assert ei.value.pivot_index == 2
    with pytest.raises(ValueError, match="symmetric"):
        spd_solve(np.array([[1.0, 0.5], [0.0, 1.0]]), np.ones(2))


def test_spd_large_pivot_index():
    """the pivot of a blocked factorisation is the global 1-based column (LAPACK info)"""
    rng = np.random.default_rng(1)
    n = 300
    q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    m = (q * rng.uniform(1, 2, n)) @ q.T
    m = 0.5 * (m + m.T)
    m[200:, :] = 0.0
    m[:, 200:] = 0.0
    m[200, 200] = -1.0
    np.fill_diagonal(m[201:, 201:], 1.0)
    with pytest.raises(NumericalError) as ei:
        SpdFactor(m, jitter_attempts=0)
    assert ei.value.pivot_index == 201


def test_backend_gemm_contract():
    """test_backend.py:18-91 on the device GEMM"""
    rng = np.random.default_rng(0)
    a = rng.normal(size=(17, 17))
    assert np.array_equal(Backend().gemm(a, np.eye(17)), a)
    a, b = rng.normal(size=(5, 9)), rng.normal(size=(7, 9))
    np.testing.assert_allclose(Backend().gemm(a, b, transpose_b=True), a @ b.T, rtol=1e-13)
    np.testing.assert_allclose(Backend().gemm(a, a, transpose_a=True), a.T @ a, rtol=1e-13, atol=1e-14)
    a, v = rng.normal(size=(40, 6)), rng.normal(size=6)
    got = Backend("parallel", workers=3, deterministic_reduction=True).gemm(a, v)
    assert got.shape == (40,)
    np.testing.assert_allclose(got, a @ v, rtol=1e-13)
    with pytest.raises(ValueError, match="conform"):
        Backend().gemm(np.zeros((2, 3)), np.zeros((2, 3)))
    a, b = rng.normal(size=(101, 37)), rng.normal(size=(37, 53))
    r = [Backend("serial", deterministic_reduction=True).gemm(a, b), Backend("parallel", workers=7).gemm(a, b)]
    assert np.array_equal(r[0], r[1])


def test_oracle_convergence_against_exact_gp():
    """test_posterior.py:93-104: FAGP converges to the exact GP, the exact GP on the device
    (exact_posterior, posterior.py:107-144)"""
    ds, Xs = cos_problem(50, 50)
    ex = F.exact_posterior(ds, Xs, GpModel(UNIT_1D, 1e-2), want_cov=True)
    exact_mean, exact_cov = ex.mean, ex.cov
    errs, cov_errs = [], []
    for n in (5, 10, 15, 20, 25):
        res = F.fagp_posterior(ds, Xs, GpModel(UNIT_1D, 1e-2, n_eigen=n), want_cov=True)
        errs.append(np.abs(res.mean - exact_mean).max())
        cov_errs.append(np.abs(res.cov - exact_cov).max())
    assert all(b <= a for a, b in zip(errs, errs[1:]))
    assert errs[-1] < 1e-4 * np.abs(ds.y).max()
    assert cov_errs[-1] < 1e-3


def test_empty_test_set():
    ds, _ = cos_problem(20, 1)
    res = F.fagp_posterior(ds, np.zeros((0, 1)), GpModel(UNIT_1D, 1e-2, n_eigen=4))
    assert res.mean.shape == (0,) and res.var.shape == (0,)
