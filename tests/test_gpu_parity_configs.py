"""GPU parity on the configurations and code paths round 1 left unpinned.

Every test compares the CUDA path with the CPU oracle (the reference algorithm: materialised
Phi, `phi.T @ phi`, LAPACK potrf; oracle/fagp_oracle.py) or with the reference's own golden
outputs, on identical seeded inputs:

  * ARD (eps, rho differing per dimension) and the `rho_linear` delta^2 variant at p = 3,
    M = 10 -- the shape served by fused_gram_split_kernel / fused_predict_split_kernel;
  * p = 3 at M = 9, 11, 12 -- fused_predict_split_kernel's other M, at the posterior level;
  * full-size C2 (N = N* = 1e5, p = 2, M = 10);
  * C4 (p 4, M 8, m 4096) at N = 1e6 and C5 (p 5, M 6, m 7776) at N = 1e5 train rows, blocked
    oracle Gram, test-row subsample;
  * prediction outside the training box (X* in [-3, 3], rho = 2);
  * the hot Gram entry (fagp_gram_x, fused, Phi never materialised) against the reference's
    G and t (golden.npz), not only against the table entry.

Tolerances (BASELINE.json north_star): mean / var elementwise relative <= 1e-9;
G, t max|d| / max|ref| <= 1e-12.  Reference: /root/reference/pkg/src/fagp/posterior.py:267-318,
mercer.py:276-292.
"""

import numpy as np
import pytest

import fagp_oracle as O
import paper_2403_12797_b200 as F
from conftest import CASE_NAMES, rel_err, scaled_err
from paper_2403_12797_b200 import _device as dev
from paper_2403_12797_b200.posterior import gram_unpack, gram_x_packed

pytestmark = pytest.mark.gpu

MEAN_VAR_RTOL = 1e-9
GRAM_TOL = 1e-12


class DS:
    def __init__(self, X, y):
        self.X, self.y = X, y


def _kernel(eps, rho):
    return F.ArdKernelParams(tuple(F.KernelParams1D(float(e), float(r)) for e, r in zip(eps, rho)))


def _data(N, Ns, p, seed, lo=-1.0, hi=1.0):
    rng = np.random.default_rng(seed)
    X = rng.uniform(-1, 1, (N, p))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    Xs = rng.uniform(lo, hi, (Ns, p))
    return X, y, Xs


def _check_posterior(X, y, Xs, eps, rho, M, noise_var, mean_const=0.0, variant="rho_squared", block=None,
                     predict_block=32768):
    model = F.GpModel(_kernel(eps, rho), noise_var, mean_const=mean_const, n_eigen=M)
    res = F.fagp_posterior(DS(X, y), Xs, model, memory_cap=None, delta2_variant=variant)
    ref = O.posterior(X, y, Xs, eps, rho, M, noise_var, mean_const, variant, block=block,
                      predict_block=predict_block)
    em, ev = rel_err(res.mean, ref["mean"]), rel_err(res.var, ref["var"])
    assert em <= MEAN_VAR_RTOL, em
    assert ev <= MEAN_VAR_RTOL, ev
    return res, ref


# ---- (i) ARD and rho_linear through the p = 3, M = 10 split kernels --------------------------
@pytest.mark.parametrize("variant", ["rho_squared", "rho_linear"])
def test_split_kernels_ard(variant):
    from paper_2403_12797_b200 import _lib

    eps, rho = [0.7, 1.0, 1.35], [0.8, 1.15, 1.6]
    X, y, Xs = _data(30_000, 7_001, 3, 31 + len(variant))
    basis = F.Basis(_kernel(eps, rho), 10, variant)
    # the shape really is served by the split layouts (the plan reports the same chunking as C3)
    assert int(_lib.lib().fagp_gram_x_chunks(30_000, basis.ref)) >= 1
    res, ref = _check_posterior(X, y, Xs, eps, rho, 10, 0.004, 0.2, variant)
    # and the hot Gram [K | t] itself against the oracle's G and t
    G, t = gram_unpack(basis, gram_x_packed(basis, dev.to_device(X), dev.to_device(y), 0.2))
    assert scaled_err(dev.to_host(G), ref["G"]) <= GRAM_TOL
    assert scaled_err(dev.to_host(t), ref["t"]) <= GRAM_TOL


# ---- (ii) p = 3, M = 9 / 11 / 12: the split predict's other shapes, posterior level ----------
@pytest.mark.parametrize("M", [9, 11, 12])
def test_split_predict_other_M(M):
    eps, rho = [1.0, 0.9, 1.2], [1.0, 1.3, 0.85]
    X, y, Xs = _data(12_000, 5_003, 3, 90 + M)
    _check_posterior(X, y, Xs, eps, rho, M, 0.0025, 0.0)


# ---- (iii) full-size C2 -------------------------------------------------------------------
@pytest.mark.slow
def test_c2_full_size_against_oracle():
    from paper_2403_12797_b200.datagen import generate, test_inputs, train_seed

    p, M, N = 2, 10, 100_000
    ds = generate(N, p, train_seed(p), 0.05)
    Xs = test_inputs(N, p)
    _check_posterior(ds.X, ds.y, Xs, [1.0] * p, [1.0] * p, M, 0.0025)


# ---- (iv) C4 at N = 1e6, C5 at N = 1e5 (blocked oracle Gram, test subsample) ---------------
@pytest.mark.slow
@pytest.mark.parametrize("p,M,N,Ns,block", [(4, 8, 1_000_000, 2_000, 16_384), (5, 6, 100_000, 1_000, 8_192)])
def test_c4_c5_train_sizes_against_oracle(p, M, N, Ns, block):
    from paper_2403_12797_b200.datagen import generate, test_inputs, train_seed

    ds = generate(N, p, train_seed(p), 0.05)
    Xs = test_inputs(Ns, p)
    res, ref = _check_posterior(ds.X, ds.y, Xs, [1.0] * p, [1.0] * p, M, 0.0025, block=block, predict_block=1000)
    assert np.all(res.var >= 0)


# ---- (v) prediction outside the training box --------------------------------------------
@pytest.mark.parametrize("p,M", [(3, 10), (2, 10), (3, 6)])
def test_predict_outside_training_box(p, M):
    """X* uniform in [-3, 3] with rho = 2 (the eigenfunctions grow like exp(rho^2 x^2 / 2)
    there); mean_const != 0 so the far-field mean (-> c) has no relative-error cancellation."""
    eps, rho = [1.0] * p, [2.0] * p
    X, y, Xs = _data(20_000, 4_001, p, 700 + p * 10 + M, lo=-3.0, hi=3.0)
    res, ref = _check_posterior(X, y, Xs, eps, rho, M, 0.0025, 0.5)
    assert np.all(np.isfinite(res.var))


# ---- (vi) the hot Gram entry against the reference's G and t ------------------------------
@pytest.mark.parametrize("name", CASE_NAMES)
def test_hot_gram_x_against_reference_G(cases, name):
    c = cases[name]
    basis = F.Basis(c.kernel(), c.M, c.variant)
    packed = gram_x_packed(basis, dev.to_device(c.X), dev.to_device(c.y), c.mean_const)
    G, t = (dev.to_host(a) for a in gram_unpack(basis, packed))
    assert scaled_err(t, c.ref["t"]) <= GRAM_TOL, scaled_err(t, c.ref["t"])
    assert scaled_err(np.diag(G), c.ref["G_diag"]) <= GRAM_TOL
    rows = [0, 1, basis.m // 2, basis.m - 1]
    assert scaled_err(G[rows], c.ref["G_rows"]) <= GRAM_TOL
    assert abs(np.linalg.norm(G) - float(c.ref["G_fro"])) <= GRAM_TOL * float(c.ref["G_fro"])
    if "G" in c.ref:
        assert scaled_err(G, c.ref["G"]) <= GRAM_TOL
    assert np.array_equal(G, G.T)


# ---- breakdown stress (the cholinv flag race) ---------------------------------
def test_spd_inverse_breakdown_stress():
    """Many indefinite matrices in a row, breakdown at every kind of column (first block,
    mid-matrix, the last pivot block, block boundaries): each returns LAPACK's info and the
    next SPD matrix still factors -- a CTA leaving the cooperative launch early would hang it."""
    import scipy.linalg as sla

    from paper_2403_12797_b200.linalg import spd_inverse

    rng = np.random.default_rng(77)
    for m in (40, 97, 256, 640, 1000):
        q, _ = np.linalg.qr(rng.standard_normal((m, m)))
        # A = U D U^T with U unit lower triangular: its Cholesky pivots are exactly D, so the
        # breakdown lands on the chosen column (LAPACK info = where + 1)
        U = np.eye(m) + np.tril(rng.standard_normal((m, m)), -1) / np.sqrt(m)
        for where in sorted({0, 1, 31, 32, 33, m // 3, m // 2, m - 33, m - 1}):
            if not 0 <= where < m:
                continue
            d = rng.uniform(1.0, 2.0, m)
            d[where] = -1.0
            Ai = (U * d) @ U.T
            Ai = 0.5 * (Ai + Ai.T)
            _, info_ref = sla.lapack.dpotrf(Ai, lower=1)
            _, info = spd_inverse(Ai)
            assert info == info_ref == where + 1, (m, where, info, info_ref)
        A = (q * np.linspace(1.0, 2.0, m)) @ q.T
        A = 0.5 * (A + A.T)
        inv, info = spd_inverse(A)
        assert info == 0
        assert scaled_err(dev.to_host(inv), np.linalg.inv(A)) < 1e-12


# ---- full covariance (off-diagonal entries) and the exact GP against the reference ----------
@pytest.mark.parametrize("name", ["c1", "ard4", "lin2", "p1m40", "c3s"])
def test_full_covariance_matches_reference(cases, name):
    """want_cov=True: the reference's full N* x N* covariance (posterior.py:249-263), every entry
    of its 200 x 200 head block, not only the diagonal."""
    c = cases[name]
    res = F.fagp_posterior(c.dataset(), c.Xs[:200], c.model(), want_cov=True, delta2_variant=c.variant,
                           memory_cap=None)
    ref = c.ref["cov_head"]
    assert res.cov.shape == ref.shape
    assert scaled_err(res.cov, ref) <= MEAN_VAR_RTOL, scaled_err(res.cov, ref)
    assert np.array_equal(res.cov, res.cov.T)
    assert rel_err(np.diag(res.cov), np.diag(ref)) <= MEAN_VAR_RTOL


@pytest.mark.parametrize("name", ["c1", "ard4", "lin2"])
def test_exact_posterior_on_device_matches_reference(cases, name):
    """exact_posterior (posterior.py:107-144) on the device: SE Gram kernel + Cholesky + solves."""
    c = cases[name]
    ex = F.exact_posterior(c.dataset(), c.Xs, c.model(), want_cov=True)
    assert scaled_err(ex.mean, c.ref["exact_mean"]) <= MEAN_VAR_RTOL
    assert rel_err(ex.mean, c.ref["exact_mean"]) <= 1e-8
    assert scaled_err(ex.cov[:200, :200], c.ref["exact_cov_head"]) <= MEAN_VAR_RTOL
    assert scaled_err(ex.var, c.ref["exact_var"]) <= MEAN_VAR_RTOL
    assert np.array_equal(ex.cov, ex.cov.T)
    # the SE Gram itself against the reference's gram_matrix restatement (CUDA exp: ulps)
    K = dev.to_host(F.se_gram(c.X[:300], c.X[:300], c.kernel()))
    Kref = O.se_gram(c.X[:300], c.X[:300], c.eps)
    assert np.all(np.diag(K) == 1.0) and np.max(np.abs(K - Kref) / Kref) <= 1e-15
