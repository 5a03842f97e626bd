"""CPU: the oracle restatement is pinned to the reference (golden fixtures + reference KATs)."""

import math

import numpy as np
import pytest

import fagp_oracle as O
from conftest import CASE_NAMES, rel_err, scaled_err


@pytest.mark.parametrize("name", [n for n in CASE_NAMES if n != "c5s"])
def test_oracle_matches_reference_outputs(cases, name):
    c = cases[name]
    out = O.posterior(c.X, c.y, c.Xs, c.eps, c.rho, c.M, c.noise_var, c.mean_const, c.variant)
    # lam and the index order are bit-exact restatements
    assert np.array_equal(out["lam"], c.ref["lam"])
    assert np.array_equal(O.lam_floored(out["lam"]), c.ref["lam_floored"])
    assert scaled_err(out["t"], c.ref["t"]) < 1e-13
    assert scaled_err(np.diag(out["G"]), c.ref["G_diag"]) < 1e-13
    if "G" in c.ref:
        assert scaled_err(out["G"], c.ref["G"]) < 1e-13
    assert out["jitter"] == float(c.ref["jitter"])
    # mean identical evaluation order; var restated (diag of the reference covariance)
    assert rel_err(out["mean"], c.ref["mean"]) < 1e-12
    assert rel_err(out["var"], c.ref["var"]) < 1e-10


def test_oracle_blocked_gram_matches(cases):
    c = cases["c2s"]
    G0, t0 = O.gram(c.X, c.y, 0.0, c.eps, c.rho, c.M, c.variant)
    G1, t1 = O.gram(c.X, c.y, 0.0, c.eps, c.rho, c.M, c.variant, block=4096)
    assert scaled_err(G1, G0) < 2e-15 * 10 and scaled_err(t1, t0) < 1e-13


def test_oracle_phi_bit_exact_with_reference(cases):
    for name in ("c1", "c3s", "ard4"):
        c = cases[name]
        phi = O.assemble_phi(c.X[:8], c.eps, c.rho, c.M, c.variant)
        assert np.array_equal(phi, c.ref["phi_head"])


def test_multi_indices_golden(golden):
    for key, ref in golden.items():
        if key.startswith("indices/"):
            n, p = (int(v) for v in key.split("/")[1].split("_"))
            assert np.array_equal(O.multi_indices(n, p), ref)


# Known-answer values frozen in the reference test-suite (test_mercer.py)
def test_kat_shape_params_and_eigenvalues():
    beta, d2 = O.beta_delta2(1.0, 2.0)
    assert beta == pytest.approx(1.1892071150027211, rel=1e-15)
    assert d2 == pytest.approx(0.8284271247461901, rel=1e-15)
    assert O.gamma(1.0, 2.0, 1)[0] == pytest.approx(1.0905077326652577, rel=1e-15)
    lam = O.eigenvalues_1d(1.0, 2.0, 2)
    assert lam[0] == pytest.approx(0.8284271247461901, rel=1e-15)
    assert lam[1] == pytest.approx(0.14213562373095049, rel=1e-15)


def test_kat_hermite():
    assert O.normalized_hermite(np.array(0.75), 13)[12] == pytest.approx(-0.52375113515335598, rel=1e-13)
    assert O.normalized_hermite(np.array(-2.5), 41)[40] == pytest.approx(-8.0292666658136296, rel=1e-13)
    assert O.normalized_hermite(np.array(5.0), 91)[90] == pytest.approx(77354.543657580687, rel=1e-12)
    assert np.all(np.isfinite(O.normalized_hermite(np.linspace(-8, 8, 33), 300)))


def test_kat_eigenfunction():
    v = O.phi_1d(np.array([0.3]), 1.0, 2.0, 7)[0, 6]
    assert v == pytest.approx(0.61576462019268915, rel=1e-13)
    assert O.phi_1d(np.array([0.0]), 1.0, 2.0, 1)[0, 0] == pytest.approx(2 ** 0.125, rel=1e-15)


def test_spd_factor_jitter_and_pivot(golden):
    L, jit = O.spd_factor(golden["spd/near_singular"])
    assert jit == float(golden["spd/near_singular_jitter"]) and jit > 0
    with pytest.raises(ArithmeticError) as ei:
        O.spd_factor(np.diag([1.0, -1.0]))
    assert ei.value.args[1] == 2


def test_useful_flops_c3():
    assert O.useful_flops(10**6, 10**6, 1000) == pytest.approx(2.0087e12, rel=1e-4)
    assert math.isclose(O.useful_flops(1000, 1000, 10), 2.807e5, rel_tol=1e-3)


LITERAL_CASES = ["c1", "lin2", "ard4", "p1m40", "c5s"]


@pytest.mark.parametrize("name", LITERAL_CASES)
def test_oracle_literal_matches_reference(cases, name):
    """method='literal' restatement against the reference's own literal outputs."""
    c = cases[name]
    out = O.posterior_literal(c.X, c.y, c.Xs, c.eps, c.rho, c.M, c.noise_var, c.mean_const, c.variant)
    assert scaled_err(out["mean"], c.ref["literal_mean"]) < 1e-12
    # the reference takes diag(cov) after cov = Phi* inner Phi*^T; the restatement forms only
    # the diagonal (same products, different summation order) -- ill-conditioned route
    assert scaled_err(out["var"], c.ref["literal_var"]) < 1e-9


COV_CASES = ["c1", "ard4", "lin2", "p1m40", "c3s"]


@pytest.mark.parametrize("name", COV_CASES)
def test_oracle_covariance_matches_reference(cases, name):
    """The full covariance restatement (off-diagonal entries included) against the reference's
    own cov (posterior.py:249-263), on the first 200 test points."""
    c = cases[name]
    out = O.posterior(c.X, c.y, c.Xs[:200], c.eps, c.rho, c.M, c.noise_var, c.mean_const, c.variant)
    cov = O.covariance(c.Xs[:200], out, c.eps, c.rho, c.M, c.noise_var, c.variant)
    ref = c.ref["cov_head"]
    assert cov.shape == ref.shape
    assert scaled_err(cov, ref) < 1e-12
    assert np.array_equal(cov, cov.T)


@pytest.mark.parametrize("name", ["c1", "ard4", "lin2"])
def test_oracle_exact_gp_matches_reference(cases, name):
    """exact_posterior restatement (posterior.py:107-144) against the reference's outputs."""
    c = cases[name]
    out = O.exact_posterior(c.X, c.y, c.Xs, c.eps, c.noise_var, c.mean_const, want_cov=True)
    assert scaled_err(out["mean"], c.ref["exact_mean"]) < 1e-12
    assert scaled_err(out["cov"][:200, :200], c.ref["exact_cov_head"]) < 1e-12
    assert scaled_err(out["var"], c.ref["exact_var"]) < 1e-10
