"""GPU parity: the CUDA path against the reference outputs (golden) and the oracle.

Tolerances (BASELINE.json north_star):
  * multi-indices, lam, lam_floored        bit-exact
  * Phi (exp differs by ulps, F5)          rtol 1e-13
  * G, t                                   max|d| / max|ref| <= 1e-12
  * mean, var                              elementwise relative <= 1e-9
"""

import numpy as np
import pytest
import torch

import fagp_oracle as O
import paper_2403_12797_b200 as F
from conftest import CASE_NAMES, rel_err, scaled_err
from paper_2403_12797_b200 import _device as dev
from paper_2403_12797_b200.posterior import _stage_tables, factor_packed, gram_packed, gram_unpack

pytestmark = pytest.mark.gpu

MEAN_VAR_RTOL = 1e-9
GRAM_TOL = 1e-12


def unpack(basis, packed):
    G, t = gram_unpack(basis, packed)
    return dev.to_host(G), dev.to_host(t)


def test_library_is_the_cuda_extension():
    from paper_2403_12797_b200 import _lib

    L = _lib.lib()
    assert L._name.endswith("libfagp_b200.so")
    assert torch.cuda.is_available()


@pytest.mark.parametrize("name", CASE_NAMES)
def test_posterior_mean_var_parity(cases, name):
    c = cases[name]
    res = F.fagp_posterior(c.dataset(), c.Xs, c.model(), delta2_variant=c.variant, memory_cap=None)
    assert res.mean.shape == (c.Ns,) and res.var.shape == (c.Ns,)
    assert rel_err(res.mean, c.ref["mean"]) <= MEAN_VAR_RTOL, rel_err(res.mean, c.ref["mean"])
    assert rel_err(res.var, c.ref["var"]) <= MEAN_VAR_RTOL, rel_err(res.var, c.ref["var"])


@pytest.mark.parametrize("name", CASE_NAMES)
def test_gram_and_t_parity(cases, name):
    c = cases[name]
    basis = F.Basis(c.kernel(), c.M, c.variant)
    X = dev.to_device(c.X)
    T = _stage_tables(basis, X, None, None)
    G, t = unpack(basis, gram_packed(basis, T, dev.to_device(c.y), c.mean_const))
    assert scaled_err(t, c.ref["t"]) <= GRAM_TOL
    assert scaled_err(np.diag(G), c.ref["G_diag"]) <= GRAM_TOL
    rows = [0, 1, basis.m // 2, basis.m - 1]
    assert scaled_err(G[rows], c.ref["G_rows"]) <= GRAM_TOL
    assert abs(np.linalg.norm(G) - float(c.ref["G_fro"])) <= GRAM_TOL * float(c.ref["G_fro"])
    if "G" in c.ref:
        assert scaled_err(G, c.ref["G"]) <= GRAM_TOL
    assert np.array_equal(G, G.T)


@pytest.mark.parametrize("name", ["c1", "c3s", "ard4", "lin2", "c5s"])
def test_eigenvalues_bit_exact(cases, name):
    c = cases[name]
    basis = F.Basis(c.kernel(), c.M, c.variant)
    from paper_2403_12797_b200 import _lib

    f, st, _ = factor_packed(basis, dev.zeros((int(_lib.lib().fagp_gram_len(basis.ref)),)), c.noise_var, 0.0, 0)
    assert np.array_equal(dev.to_host(f.lam), c.ref["lam"])
    assert np.array_equal(dev.to_host(f.lam_floored), c.ref["lam_floored"])
    assert np.array_equal(dev.to_host(f.sqrt_lam), np.sqrt(c.ref["lam_floored"]))


@pytest.mark.parametrize("name", ["c1", "c3s", "ard4", "lin2"])
def test_features_match_reference_phi(cases, name):
    c = cases[name]
    es = F.eigensystem(c.X[:8], c.kernel(), c.M, delta2_variant=c.variant)
    np.testing.assert_allclose(es.phi, c.ref["phi_head"], rtol=1e-13, atol=0)
    assert np.array_equal(es.lam, c.ref["lam"])


def test_multi_indices_bit_exact(golden):
    for key, ref in golden.items():
        if key.startswith("indices/"):
            n, p = (int(v) for v in key.split("/")[1].split("_"))
            got = F.multi_indices(n, p)
            assert got.dtype == np.int64 and np.array_equal(got, ref)


def test_factor_jitter_matches_reference(cases):
    for name in ("c1", "c2s", "c3s"):
        c = cases[name]
        basis = F.Basis(c.kernel(), c.M, c.variant)
        T = _stage_tables(basis, dev.to_device(c.X), None, None)
        packed = gram_packed(basis, T, dev.to_device(c.y), c.mean_const)
        f, st, piv = factor_packed(basis, packed, c.noise_var, c.mean_const, c.N)
        assert st == 0 and piv == 0
        assert f.jitter == float(c.ref["jitter"])


def test_weights_match_oracle(cases):
    c = cases["c2s"]
    basis = F.Basis(c.kernel(), c.M, c.variant)
    T = _stage_tables(basis, dev.to_device(c.X), None, None)
    packed = gram_packed(basis, T, dev.to_device(c.y), c.mean_const)
    f, st, _ = factor_packed(basis, packed, c.noise_var, c.mean_const, c.N, need_L=True)
    G, t = unpack(basis, packed)
    o = O.factor(G, t, c.ref["lam"], c.noise_var)
    assert scaled_err(dev.to_host(f.w), o["w"]) < 1e-10
    Lg = dev.to_host(f.L)
    assert scaled_err(Lg, o["L"]) < 1e-12
    assert np.all(np.triu(Lg, 1) == 0)
    # the fused inverse route (hot path): same weights, A^{-1} against the oracle's factor
    fi, st, _ = factor_packed(basis, packed, c.noise_var, c.mean_const, c.N)
    assert st == 0 and fi.L is None
    assert scaled_err(dev.to_host(fi.w), o["w"]) < 1e-10
    Li = np.linalg.inv(o["L"])
    assert scaled_err(dev.to_host(fi.Ainv), Li.T @ Li) < 1e-9


def test_run_to_run_bitwise_determinism(cases):
    c = cases["c3s"]
    a = F.fagp_posterior(c.dataset(), c.Xs, c.model(), memory_cap=None)
    b = F.fagp_posterior(c.dataset(), c.Xs, c.model(), memory_cap=None)
    assert np.array_equal(a.mean, b.mean) and np.array_equal(a.var, b.var)


def test_split_api_matches_one_shot(cases):
    c = cases["c2s"]
    full = F.fagp_posterior(c.dataset(), c.Xs, c.model(), memory_cap=None)
    es = F.eigensystem(c.X, c.kernel(), c.M, memory_cap=None)
    es_s = F.eigensystem(c.Xs, c.kernel(), c.M, memory_cap=None)
    split = F.fagp_posterior_from_eigensystems(es, es_s, c.y, c.model())
    assert np.array_equal(full.mean, split.mean) and np.array_equal(full.var, split.var)
    h = F.fit(c.dataset(), c.model(), memory_cap=None)
    pr = F.predict(h, c.Xs)
    assert np.array_equal(full.mean, pr.mean) and np.array_equal(full.var, pr.var)


def test_device_inputs_match_host_inputs(cases):
    c = cases["c1"]

    class DS:
        X = torch.as_tensor(c.X, device="cuda")
        y = torch.as_tensor(c.y, device="cuda")

    a = F.fagp_posterior(DS, torch.as_tensor(c.Xs, device="cuda"), c.model(), return_device=True)
    b = F.fagp_posterior(c.dataset(), c.Xs, c.model())
    assert a.mean.is_cuda and np.array_equal(dev.to_host(a.mean), b.mean)


def test_full_covariance_matches_reference_diag(cases):
    c = cases["ard4"]
    res = F.fagp_posterior(c.dataset(), c.Xs, c.model(), want_cov=True)
    assert res.cov.shape == (c.Ns, c.Ns)
    assert np.array_equal(res.cov, res.cov.T)
    assert rel_err(np.diag(res.cov), c.ref["var"]) < 1e-9


def test_hermite_kats_on_device():
    h = F.normalized_hermite(np.array([0.75, -2.5, 5.0]), 91)
    assert h[0, 12] == pytest.approx(-0.52375113515335598, rel=1e-13)
    assert h[1, 40] == pytest.approx(-8.0292666658136296, rel=1e-13)
    assert h[2, 90] == pytest.approx(77354.543657580687, rel=1e-12)
    z = np.array([0.0, 0.5, -1.25])
    hz = F.normalized_hermite(z, 3)
    assert np.array_equal(hz, O.normalized_hermite(z, 3))  # bit-exact recurrence
    assert np.all(np.isfinite(F.normalized_hermite(np.linspace(-8, 8, 33), 300)))
    zz = np.linspace(-3, 3, 1001)
    assert np.array_equal(F.normalized_hermite(zz, 40), O.normalized_hermite(zz, 40))


def test_eigenfunction_kats_on_device():
    p12 = F.KernelParams1D(1.0, 2.0)
    assert F.eigenfunction_1d(7, 0.3, p12) == pytest.approx(0.61576462019268915, rel=1e-13)
    assert F.eigenfunction_1d(1, 0.0, p12) == pytest.approx(2 ** 0.125, rel=1e-15)
    for params in (F.KernelParams1D(1.0, 1.0), p12, F.KernelParams1D(0.2, 0.7)):
        assert F.eigenfunction_1d(2, 0.0, params) == 0.0
    assert F.eigenfunction_1d(3, 1.0, F.KernelParams1D(0.0, 1.0)) == pytest.approx(0.7071067811865476, rel=1e-12)
    xs = np.linspace(0.05, 2.5, 9)
    for i in range(1, 13):
        np.testing.assert_allclose(F.eigenfunction_1d(i, -xs, F.KernelParams1D(1.0, 1.0)),
                                   (-1.0) ** (i - 1) * F.eigenfunction_1d(i, xs, F.KernelParams1D(1.0, 1.0)),
                                   rtol=1e-12)


@pytest.mark.parametrize("p,M,N,Ns", [(1, 1, 5, 3), (1, 7, 33, 129), (2, 3, 200, 257), (3, 4, 1000, 130),
                                      (6, 2, 500, 64), (1, 130, 2000, 50), (1, 200, 1500, 70)])
def test_ragged_shapes_against_oracle(p, M, N, Ns):
    rng = np.random.default_rng(p * 1000 + M)
    X = rng.uniform(-1, 1, (N, p))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    Xs = rng.uniform(-1, 1, (Ns, p))
    eps = rng.uniform(0.3, 1.5, p)
    rho = rng.uniform(0.5, 2.0, p)
    kernel = F.ArdKernelParams(tuple(F.KernelParams1D(float(e), float(r)) for e, r in zip(eps, rho)))
    model = F.GpModel(kernel, 0.01, mean_const=0.3, n_eigen=M)
    ref = O.posterior(X, y, Xs, eps, rho, M, 0.01, 0.3)

    class DS:
        pass

    DS.X, DS.y = X, y
    res = F.fagp_posterior(DS, Xs, model, memory_cap=None)
    assert rel_err(res.mean, ref["mean"]) <= MEAN_VAR_RTOL
    assert rel_err(res.var, ref["var"]) <= MEAN_VAR_RTOL


@pytest.mark.slow
def test_c3_full_size_properties():
    """BASELINE config C3 at full size: determinism, sanity bounds and subsample parity."""
    from paper_2403_12797_b200.datagen import generate, test_inputs, train_seed

    p, M, N = 3, 10, 1_000_000
    ds = generate(N, p, train_seed(p), 0.05)
    Xs = test_inputs(N, p)
    kernel = F.ArdKernelParams.isotropic(p, 1.0, 1.0)
    model = F.GpModel(kernel, 0.0025, n_eigen=M)
    a = F.fagp_posterior(ds, Xs, model, memory_cap=None)
    b = F.fagp_posterior(ds, Xs, model, memory_cap=None)
    assert np.array_equal(a.mean, b.mean) and np.array_equal(a.var, b.var)
    assert np.all(np.isfinite(a.mean)) and np.all(a.var >= 0)
    # oracle on the full train set (blocked Gram), test subsample
    idx = np.arange(0, N, 997)
    ref = O.posterior(ds.X, ds.y, Xs[idx], [1.0] * p, [1.0] * p, M, 0.0025, block=65536)
    assert rel_err(a.mean[idx], ref["mean"]) <= MEAN_VAR_RTOL
    assert rel_err(a.var[idx], ref["var"]) <= MEAN_VAR_RTOL


@pytest.mark.parametrize("impl", ["persistent", "blocked", "big"])
@pytest.mark.parametrize("m", [1, 5, 31, 32, 33, 64, 100, 257, 1000, 1100])
def test_potrf_matches_lapack(m, impl, monkeypatch):
    """fagp_potrf (persistent cooperative kernel, the blocked fallback, and the large-m route of
    512-column panels used from m = 3000 on -- forced here at small m) against LAPACK dpotrf on SPD
    matrices, and LAPACK's 1-based info on an indefinite one (breakdown inside a later panel for
    the large-m route at m = 1000, 1100)."""
    import scipy.linalg as sla

    from paper_2403_12797_b200.linalg import potrf

    if impl != "persistent":
        monkeypatch.setenv("FAGP_POTRF", impl)
    rng = np.random.default_rng(m)
    B = rng.standard_normal((m, m))
    A = B @ B.T + m * np.eye(m)
    L, info = potrf(A)
    assert info == 0
    Lh = dev.to_host(L)
    ref = np.linalg.cholesky(A)
    assert np.array_equal(np.triu(Lh, 1), np.zeros((m, m)))
    assert np.max(np.abs(Lh - ref)) / np.max(np.abs(ref)) < 1e-13
    if m >= 5:
        # indefinite: eigenvalue -1 placed so the breakdown lands mid-matrix
        q, _ = np.linalg.qr(rng.standard_normal((m, m)))
        ev = np.linspace(1.0, 2.0, m)
        ev[m // 2] = -1.0
        Ai = (q * ev) @ q.T
        Ai = 0.5 * (Ai + Ai.T)
        _, info_ref = sla.lapack.dpotrf(Ai, lower=1)
        _, info = potrf(Ai)
        assert info == info_ref > 0


# ---- the point-input (fused) entry points against the table path ----------------------
@pytest.mark.parametrize("p,M,N", [(2, 10, 1), (2, 10, 63), (2, 10, 5000), (3, 10, 1), (3, 10, 64), (3, 10, 4097),
                                   (3, 6, 777), (4, 4, 3001), (3, 10, 200_003),
                                   # output-tiled fused Gram (gram_tiled.cu): C4 / C5 shapes, ragged N
                                   (4, 8, 1), (4, 8, 3001), (4, 8, 70_001), (5, 6, 5), (5, 6, 2001), (6, 3, 999)])
def test_gram_x_matches_table_gram(p, M, N):
    from paper_2403_12797_b200.posterior import gram_x_packed

    rng = np.random.default_rng(1000 * p + M)
    X = rng.uniform(-1, 1, (N, p))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    kernel = F.ArdKernelParams.isotropic(p, 1.0, 1.0)
    basis = F.Basis(kernel, M)
    Xd, yd = dev.to_device(X), dev.to_device(y)
    ref = dev.to_host(gram_packed(basis, _stage_tables(basis, Xd, None, None), yd, 0.3))
    got = dev.to_host(gram_x_packed(basis, Xd, yd, 0.3))
    assert got.shape == ref.shape
    assert scaled_err(got, ref) <= 1e-13, scaled_err(got, ref)
    again = dev.to_host(gram_x_packed(basis, Xd, yd, 0.3))
    assert np.array_equal(got, again)  # deterministic


@pytest.mark.parametrize("p,M,Ns", [(2, 10, 1), (2, 10, 65), (3, 10, 1), (3, 10, 127), (3, 10, 100_001),
                                    (3, 6, 999), (4, 4, 3001),
                                    # output-tiled fused predict (predict_tiled.cu): C4 / C5 shapes, ragged N*
                                    (4, 8, 1), (4, 8, 3001), (4, 8, 70_001), (5, 6, 7), (5, 6, 2001), (6, 3, 999)])
def test_predict_x_matches_table_predict(p, M, Ns):
    from paper_2403_12797_b200.posterior import predict_x_device

    rng = np.random.default_rng(7 * p + M)
    N = 4000
    X = rng.uniform(-1, 1, (N, p))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    Xs = rng.uniform(-1.2, 1.2, (Ns, p))
    kernel = F.ArdKernelParams.isotropic(p, 1.0, 1.0)
    basis = F.Basis(kernel, M)
    Xd, yd, Xsd = dev.to_device(X), dev.to_device(y), dev.to_device(Xs)
    packed = gram_packed(basis, _stage_tables(basis, Xd, None, None), yd, 0.1)
    f, st, _ = factor_packed(basis, packed, 0.0025, 0.1, N)
    assert st == 0
    m_ref, v_ref = (dev.to_host(a) for a in predict_device_table(f, basis, Xsd))
    m_got, v_got = (dev.to_host(a) for a in predict_x_device(f, Xsd))
    assert rel_err(m_got, m_ref) <= 1e-11, rel_err(m_got, m_ref)
    assert rel_err(v_got, v_ref) <= 1e-9, rel_err(v_got, v_ref)
    m_only, none = predict_x_device(f, Xsd, want_var=False)
    assert none is None and np.array_equal(dev.to_host(m_only), m_got)


def predict_device_table(f, basis, Xsd):
    from paper_2403_12797_b200.posterior import predict_device

    return predict_device(f, _stage_tables(basis, Xsd, None, None))


def test_fused_path_flags_nonfinite_points():
    from paper_2403_12797_b200.posterior import gram_x_packed

    X = np.random.default_rng(0).uniform(-1, 1, (500, 3))
    X[123, 1] = np.nan
    basis = F.Basis(F.ArdKernelParams.isotropic(3, 1.0, 1.0), 10)
    flags = dev.zeros((1,), dtype="int32")
    from paper_2403_12797_b200 import _lib

    gram_x_packed(basis, dev.to_device(X), None, 0.0, flag_ptr=_lib.ptr(flags))
    assert int(dev.to_host(flags)[0]) & _lib.FLAG_X_NONFINITE


@pytest.mark.parametrize("N,Ns", [(200_003, 70_001), (5_000, 3_000)])
def test_host_pipeline_bitwise_equals_device_path(N, Ns):
    """fagp_posterior from host arrays (chunked uploads overlapped with the Gram sub-ranges,
    chunked predict + D2H) is bitwise identical to the device-resident path."""
    rng = np.random.default_rng(11)
    X = rng.uniform(-1, 1, (N, 3))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    Xs = rng.uniform(-1, 1, (Ns, 3))
    model = F.GpModel(F.ArdKernelParams.isotropic(3, 1.0, 1.0), 0.0025, n_eigen=10)

    class Host:
        pass

    class Dev:
        pass

    Host.X, Host.y = torch.from_numpy(X).pin_memory(), y
    Dev.X, Dev.y = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    a = F.fagp_posterior(Host, Xs, model, memory_cap=None)
    b = F.fagp_posterior(Dev, torch.from_numpy(Xs).cuda(), model, memory_cap=None)
    assert np.array_equal(a.mean, b.mean) and np.array_equal(a.var, b.var)
    c = F.fagp_posterior(Host, Xs, model, memory_cap=None)  # cached engine, second call
    assert np.array_equal(a.mean, c.mean) and np.array_equal(a.var, c.var)


@pytest.mark.parametrize("m", [1, 5, 31, 32, 33, 64, 100, 257, 1000])
def test_spd_inverse_sweep_matches_lapack(m):
    """fagp_spd_inverse (persistent Cholesky + trtri + lauum) against numpy's inverse on SPD
    matrices, Cholesky-grade accuracy on an ill-conditioned one, and LAPACK dpotrf's 1-based
    info on indefinite ones."""
    import scipy.linalg as sla

    from paper_2403_12797_b200.linalg import spd_inverse

    rng = np.random.default_rng(100 + m)
    B = rng.standard_normal((m, m))
    A = B @ B.T + m * np.eye(m)
    Ainv, info = spd_inverse(A)
    assert info == 0
    got = dev.to_host(Ainv)
    ref = np.linalg.inv(A)
    assert np.array_equal(got, got.T)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12
    # a badly conditioned SPD matrix (cond ~ 1e10) still matches to the conditioning
    q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    ev = np.logspace(0, -10, m)
    Ac = 0.5 * ((q * ev) @ q.T + ((q * ev) @ q.T).T)
    inv_c, info_c = spd_inverse(Ac)
    assert info_c == 0
    got_c = dev.to_host(inv_c)
    ref_c = np.linalg.inv(Ac)
    assert np.max(np.abs(got_c - ref_c)) / np.max(np.abs(ref_c)) < 1e-5
    if m >= 5:
        for where in (m // 2, m - 1, 1):
            ev = np.linspace(1.0, 2.0, m)
            ev[where] = -1.0
            Ai = (q * ev) @ q.T
            Ai = 0.5 * (Ai + Ai.T)
            _, info_ref = sla.lapack.dpotrf(Ai, lower=1)
            _, info = spd_inverse(Ai)
            assert info == info_ref > 0


def test_async_factor_falls_back_to_the_jitter_schedule():
    """A system whose attempt 0 breaks down (rank-deficient Gram, negligible noise): the async
    factor's retry path must give exactly what the blocking route (fit/predict) gives."""
    rng = np.random.default_rng(5)
    X = np.repeat(rng.uniform(-1, 1, (3, 2)), 40, axis=0)
    y = np.cos(X).sum(1)
    Xs = rng.uniform(-1, 1, (300, 2))
    model = F.GpModel(F.ArdKernelParams.isotropic(2, 1.0, 1.0), 1e-30, n_eigen=10)

    class DS:
        pass

    DS.X, DS.y = X, y
    f = F.fit(DS, model, memory_cap=None)
    assert f.jitter > 0.0  # the reference's schedule was needed
    ref = F.predict(f, Xs)
    got = F.fagp_posterior(DS, Xs, model, memory_cap=None)
    assert np.array_equal(got.mean, ref.mean) and np.array_equal(got.var, ref.var)
    dev_in = F.fagp_posterior(DS, torch.from_numpy(Xs).cuda(), model, memory_cap=None, return_device=True)
    assert np.array_equal(dev.to_host(dev_in.mean), ref.mean)


@pytest.mark.parametrize("N", [1, 4_097, 300_001])
def test_pipelined_gram_bitwise_equals_gram_x(N):
    """fagp_gram_x_pipelined: one launch waiting on per-chunk ready words, the chunks uploaded
    (in reverse order, to exercise the waits) and signalled from a copy stream -- bitwise the
    fagp_gram_x buffer, the ready words re-armed, twice in a row."""
    from paper_2403_12797_b200 import _lib
    from paper_2403_12797_b200.posterior import gram_x_packed

    rng = np.random.default_rng(N)
    X = rng.uniform(-1, 1, (N, 3))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    basis = F.Basis(F.ArdKernelParams.isotropic(3, 1.0, 1.0), 10)
    ref = dev.to_host(gram_x_packed(basis, dev.to_device(X), dev.to_device(y), 0.2))
    L = _lib.lib()
    nch = int(L.fagp_gram_x_chunks(N, basis.ref))
    Xh, yh = torch.from_numpy(X).pin_memory(), torch.from_numpy(y).pin_memory()
    Xd, yd = dev.empty((N, 3)), dev.empty((N,))
    ready = dev.zeros((nch,), dtype="int32")
    flags = dev.zeros((1,), dtype="int32")
    wsz = int(L.fagp_gram_x_workspace_size(N, basis.ref))
    ws = dev.empty((max(1, -(-wsz // 8)),))
    side = torch.cuda.Stream()
    for _ in range(2):
        out = dev.empty((int(L.fagp_gram_len(basis.ref)),))
        side.wait_stream(torch.cuda.current_stream())
        cs = _lib.stream_handle(torch.cuda.current_stream())
        _lib.check(L.fagp_gram_x_pipelined(_lib.ptr(Xd), N, basis.ref, _lib.ptr(yd), 0.2, _lib.ptr(ready),
                                           _lib.ptr(out), _lib.ptr(ws), wsz, _lib.ptr(flags), cs), "pipelined")
        sin = _lib.stream_handle(side)
        for k in reversed(range(nch)):
            _lib.check(L.fagp_gram_x_upload_chunk(_lib.ptr(Xh), _lib.ptr(yh), N, basis.ref, k, _lib.ptr(Xd),
                                                  _lib.ptr(yd), sin), "upload")
            _lib.check(L.fagp_gram_x_signal(_lib.ptr(ready), k, sin), "signal")
        torch.cuda.synchronize()
        assert int(dev.to_host(flags)[0]) == 0
        assert np.array_equal(dev.to_host(out), ref)
        assert not dev.to_host(ready).any()


def test_pipelined_gram_without_signal_reports_stall():
    """A ready word that is never set: the launch gives up after its bounded wait (~2 s) and
    raises FAGP_FLAG_STALLED instead of hanging the device."""
    from paper_2403_12797_b200 import _lib

    N = 50_000
    basis = F.Basis(F.ArdKernelParams.isotropic(3, 1.0, 1.0), 10)
    L = _lib.lib()
    nch = int(L.fagp_gram_x_chunks(N, basis.ref))
    Xd, yd = dev.zeros((N, 3)), dev.zeros((N,))
    ready = dev.zeros((nch,), dtype="int32")
    flags = dev.zeros((1,), dtype="int32")
    wsz = int(L.fagp_gram_x_workspace_size(N, basis.ref))
    ws = dev.empty((max(1, -(-wsz // 8)),))
    out = dev.empty((int(L.fagp_gram_len(basis.ref)),))
    _lib.check(L.fagp_gram_x_pipelined(_lib.ptr(Xd), N, basis.ref, _lib.ptr(yd), 0.0, _lib.ptr(ready), _lib.ptr(out),
                                       _lib.ptr(ws), wsz, _lib.ptr(flags), None), "pipelined")
    torch.cuda.synchronize()
    assert int(dev.to_host(flags)[0]) & _lib.FLAG_STALLED


@pytest.mark.parametrize("M", [4, 10, 11, 12])
def test_fused_mode_products_match_the_generic_kernels(M, monkeypatch):
    """p = 3 fused mode products against the generic per-mode kernels (FAGP_MODE_UNFUSED=1):
    expand3 (K -> pair Gram) keeps their stage and fma order -- bitwise the same G; ctc3 (the C''
    predict operand, folded and contracted in another order) agrees to rounding."""
    from paper_2403_12797_b200.posterior import gram_x_packed

    rng = np.random.default_rng(40 + M)
    N = 20_000
    X = rng.uniform(-1, 1, (N, 3))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    basis = F.Basis(F.ArdKernelParams.isotropic(3, 1.0, 1.0), M)
    packed = gram_x_packed(basis, dev.to_device(X), dev.to_device(y), 0.1)

    def run():
        G, t = gram_unpack(basis, packed)
        f, st, _ = factor_packed(basis, packed, 0.01, 0.1, N)
        assert st == 0
        return dev.to_host(G), dev.to_host(f.predict_op)

    G1, op1 = run()
    monkeypatch.setenv("FAGP_MODE_UNFUSED", "1")
    G0, op0 = run()
    assert np.array_equal(G1, G0)
    assert np.abs(op1 - op0).max() <= 1e-12 * np.abs(op0).max()


@pytest.mark.parametrize("subranges,chunks", [("1", 1), ("3", 7), ("27", 2)])
def test_host_pipeline_chunking_is_bitwise_invariant(subranges, chunks, monkeypatch):
    """The host path's upload chunking (Gram sub-ranges) and predict chunking change nothing:
    every split gives the device-resident path's bits."""
    from paper_2403_12797_b200.engine import PosteriorEngine

    rng = np.random.default_rng(5)
    N, Ns = 150_001, 90_017
    X = rng.uniform(-1, 1, (N, 3))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    Xs = rng.uniform(-1, 1, (Ns, 3))
    model = F.GpModel(F.ArdKernelParams.isotropic(3, 1.0, 1.0), 0.0025, n_eigen=10)

    class Dev:
        pass

    Dev.X, Dev.y = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    ref = F.fagp_posterior(Dev, torch.from_numpy(Xs).cuda(), model, memory_cap=None)
    monkeypatch.setenv("FAGP_GRAM_SUBRANGES", subranges)
    monkeypatch.setattr(PosteriorEngine, "PREDICT_CHUNKS", chunks)

    class Host:
        pass

    Host.X, Host.y = torch.from_numpy(X).pin_memory(), y
    got = F.fagp_posterior(Host, Xs, model, memory_cap=None)
    assert np.array_equal(got.mean, ref.mean) and np.array_equal(got.var, ref.var)


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (300, 257, 70), (513, 640, 129), (1000, 384, 1000)])
def test_dgemm_large_tile_matches_numpy(M, N, K, ta, tb):
    """The 128 x 128-tile DGEMM (both output sides >= 256, K >= 64: the m >= 3000 factor's GEMMs),
    every transpose combination, ragged edges, alpha / beta accumulation."""
    from paper_2403_12797_b200.linalg import dgemm

    rng = np.random.default_rng(M + 7 * N + 13 * K + 2 * ta + tb)
    a = rng.standard_normal((K, M) if ta else (M, K))
    b = rng.standard_normal((N, K) if tb else (K, N))
    c0 = rng.standard_normal((M, N))
    ref = -0.5 * ((a.T if ta else a) @ (b.T if tb else b)) + 2.0 * c0
    out = dev.to_device(c0)
    got = dev.to_host(dgemm(a, b, trans_a=bool(ta), trans_b=bool(tb), alpha=-0.5, beta=2.0, out=out))
    scale = np.abs(a).max() * np.abs(b).max() * K
    assert np.abs(got - ref).max() <= 1e-14 * scale


@pytest.mark.parametrize("zc_in,zc_out", [(True, True), (False, True), (True, False), (False, False)])
def test_host_path_zero_copy_is_bitwise_invariant(zc_in, zc_out, monkeypatch):
    """Pinned X, y, X*: the kernels read them in place and store mean / var straight into the
    pinned result buffer (zero-copy), or the copy pipelines run -- the same bits either way, equal
    to the device-resident path."""
    from paper_2403_12797_b200.engine import PosteriorEngine

    rng = np.random.default_rng(8)
    N, Ns = 120_007, 70_001
    X = rng.uniform(-1, 1, (N, 3))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    Xs = rng.uniform(-1, 1, (Ns, 3))
    model = F.GpModel(F.ArdKernelParams.isotropic(3, 1.0, 1.0), 0.0025, n_eigen=10)

    class Dev:
        pass

    Dev.X, Dev.y = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    ref = F.fagp_posterior(Dev, torch.from_numpy(Xs).cuda(), model, memory_cap=None)
    monkeypatch.setattr(PosteriorEngine, "ZERO_COPY_IN", zc_in)
    monkeypatch.setattr(PosteriorEngine, "ZERO_COPY_OUT", zc_out)

    class Host:
        pass

    Host.X, Host.y = torch.from_numpy(X).pin_memory(), torch.from_numpy(y).pin_memory()
    for _ in range(2):  # a second call reuses the engine and its pooled result buffers
        got = F.fagp_posterior(Host, torch.from_numpy(Xs).pin_memory(), model, memory_cap=None)
        assert np.array_equal(got.mean, ref.mean) and np.array_equal(got.var, ref.var)


@pytest.mark.gpu
@pytest.mark.parametrize("p,M,Ns", [(3, 10, 1), (3, 10, 63), (3, 10, 64), (3, 10, 65), (3, 10, 129), (3, 10, 3000),
                                    (3, 10, 148 * 128 + 5), (3, 9, 777), (3, 11, 4097), (3, 12, 200),
                                    # tiled predict: two groups where FB <= 2 (p = 4), one at p = 5
                                    (4, 8, 1), (4, 8, 33), (4, 8, 70_001), (5, 6, 2001)])
def test_predict_groups_bitwise(p, M, Ns, monkeypatch):
    """The two-warp-group predict kernels (split predict: 64-row blocks per group, named barriers,
    staggered start; tiled predict: 32-row blocks per group) against the one-group CTA, bitwise:
    each row's partial sums run the same k-steps in the same order.  Covers groups without a
    block (N* < 64, the last CTA's second group), one-CTA grids and ragged last blocks."""
    from paper_2403_12797_b200.posterior import gram_x_packed, predict_x_device

    rng = np.random.default_rng(11 * p + M)
    N = 3000
    X = rng.uniform(-1, 1, (N, p))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    Xs = rng.uniform(-1.5, 1.5, (Ns, p))
    basis = F.Basis(F.ArdKernelParams.isotropic(p, 1.0, 1.0), M)
    Xd, yd, Xsd = dev.to_device(X), dev.to_device(y), dev.to_device(Xs)
    f, st, _ = factor_packed(basis, gram_x_packed(basis, Xd, yd, 0.1), 0.0025, 0.1, N)
    assert st == 0
    out = {}
    for g in ("1", "2"):
        monkeypatch.setenv("FAGP_PREDICT_GROUPS", g)
        out[g] = [dev.to_host(a) for a in predict_x_device(f, Xsd)]
    for a, b in zip(out["1"], out["2"]):
        assert np.array_equal(a, b)
    assert np.all(np.isfinite(out["2"][0])) and np.all(out["2"][1] >= -1e-12)


@pytest.mark.parametrize("p,M,N", [(4, 8, 70_001), (5, 6, 50_003), (5, 6, 4096)])
def test_tiled_gram_span_deal(p, M, N, monkeypatch):
    """The tiled Gram's two CTA deals -- whole CTAs per tile, and CTAs cutting the tile-major work
    evenly (a CTA may finish one tile and start the next, two partial slots) -- agree with each
    other and with the table path, each deterministic."""
    from paper_2403_12797_b200.posterior import gram_x_packed

    rng = np.random.default_rng(31 * p + N)
    X = rng.uniform(-1, 1, (N, p))
    y = np.cos(X).sum(1) + 0.05 * rng.standard_normal(N)
    basis = F.Basis(F.ArdKernelParams.isotropic(p, 1.0, 1.0), M)
    Xd, yd = dev.to_device(X), dev.to_device(y)
    ref = dev.to_host(gram_packed(basis, _stage_tables(basis, Xd, None, None), yd, 0.3))
    got = {}
    for sp in ("0", "1"):
        monkeypatch.setenv("FAGP_TILED_SPAN", sp)
        got[sp] = dev.to_host(gram_x_packed(basis, Xd, yd, 0.3))
        assert np.array_equal(got[sp], dev.to_host(gram_x_packed(basis, Xd, yd, 0.3)))
        assert scaled_err(got[sp], ref) <= 1e-13, (sp, scaled_err(got[sp], ref))
    assert scaled_err(got["1"], got["0"]) <= 1e-13
