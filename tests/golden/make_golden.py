"""Generate golden fixtures by running the REFERENCE package itself (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Inputs are regenerated from seeds by the tests (numpy's
Philox is stable), so only seeds + input checksums + reference outputs are stored.  The
variance stored is np.diag(result.cov) -- exactly what `fagp predict` writes
(cli.py:222) -- from the reference's full covariance.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import fagp  # noqa: E402
from fagp.backend import SpdFactor  # noqa: E402
from fagp.bench import BenchConfig, _test_inputs, train_seed  # noqa: E402
from fagp.kernels import ArdKernelParams, KernelParams1D  # noqa: E402
from fagp.mercer import eigensystem, multi_indices  # noqa: E402
from fagp.posterior import GpModel, LambdaBarSolve, exact_posterior, fagp_posterior  # noqa: E402

OUT = Path(__file__).with_name("golden.npz")

# name: (p, M, N, Ns, eps per dim, rho per dim, noise_var, mean_const, delta2 variant, full G?)
CASES = {
    "c1": (1, 10, 1000, 1000, None, None, 0.0025, 0.0, "rho_squared", True),
    "c2s": (2, 10, 20000, 2000, None, None, 0.0025, 0.0, "rho_squared", True),
    "c3s": (3, 10, 4000, 600, None, None, 0.0025, 0.0, "rho_squared", False),
    "ard4": (4, 3, 700, 150, (1.0, 0.5, 2.0, 0.7), (1.0, 2.0, 0.5, 1.5), 0.01, 0.25, "rho_squared", True),
    "lin2": (2, 7, 900, 200, (0.8, 1.3), (0.6, 1.7), 0.05, -0.5, "rho_linear", True),
    "p1m40": (1, 40, 3000, 400, (1.5,), (1.2,), 0.001, 1.0, "rho_squared", True),
    "c5s": (5, 6, 600, 80, None, None, 0.0025, 0.0, "rho_squared", False),
    "c4s": (4, 8, 3000, 300, None, None, 0.0025, 0.0, "rho_squared", False),
}

LITERAL_CASES = ("c1", "lin2", "ard4", "p1m40", "c5s")
COV_CASES = ("c1", "ard4", "lin2", "p1m40", "c3s")  # store the reference's full covariance (head block)
EXACT_CASES = ("c1", "ard4", "lin2")  # the exact dense GP (posterior.py:107-144)
COV_HEAD = 200  # cov[:200, :200]: the covariance of the first 200 test points


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {}
    for name, (p, M, N, Ns, eps, rho, nv, c, var_kind, full_g) in CASES.items():
        cfg = BenchConfig(n_samples=N, n_test=Ns)
        seed = train_seed(cfg, p, 0)
        ds = fagp.generate(N, p, seed, 0.05, domain=(-1.0, 1.0))
        Xs = _test_inputs(cfg, p, 0)
        if eps is None:
            kernel = ArdKernelParams.isotropic(p, 1.0, 1.0)
        else:
            kernel = ArdKernelParams(tuple(KernelParams1D(e, r) for e, r in zip(eps, rho)))
        model = GpModel(kernel, noise_var=nv, mean_const=c, n_eigen=M)
        res = fagp_posterior(ds, Xs, model, want_cov=True, delta2_variant=var_kind, memory_cap=1 << 40)
        es = eigensystem(ds.X, kernel, M, delta2_variant=var_kind, memory_cap=1 << 40)
        handle = LambdaBarSolve(es, nv)
        G = handle._gram
        t = es.phi.T @ (ds.y - c)
        pre = f"{name}/"
        out[pre + "meta"] = np.array([p, M, N, Ns, seed])
        out[pre + "eps"] = np.array([k.epsilon for k in kernel.per_dim])
        out[pre + "rho"] = np.array([k.rho for k in kernel.per_dim])
        out[pre + "noise_var"] = np.array(nv)
        out[pre + "mean_const"] = np.array(c)
        out[pre + "variant"] = np.array(var_kind)
        out[pre + "x_sha"] = np.array(digest(ds.X) + digest(ds.y) + digest(Xs))
        out[pre + "mean"] = res.mean
        out[pre + "var"] = np.diag(res.cov).copy()
        out[pre + "lam"] = es.lam
        out[pre + "lam_floored"] = es.lam_floored
        out[pre + "t"] = t
        out[pre + "G_diag"] = np.diag(G).copy()
        out[pre + "G_rows"] = G[[0, 1, G.shape[0] // 2, G.shape[0] - 1]].copy()
        out[pre + "G_fro"] = np.array(np.linalg.norm(G))
        out[pre + "jitter"] = np.array(handle._factor.jitter)
        out[pre + "phi_head"] = es.phi[:8].copy()
        if full_g:
            out[pre + "G"] = G
        if name in COV_CASES:  # off-diagonal entries of the reference covariance (posterior.py:249-263)
            out[pre + "cov_head"] = res.cov[:COV_HEAD, :COV_HEAD].copy()
        if name in EXACT_CASES:
            ex = exact_posterior(ds, Xs, model, want_cov=True)
            out[pre + "exact_mean"] = ex.mean
            out[pre + "exact_var"] = np.diag(ex.cov).copy()
            out[pre + "exact_cov_head"] = ex.cov[:COV_HEAD, :COV_HEAD].copy()
        if name in LITERAL_CASES:  # the cross-check route (posterior.py:236-244, 256-260)
            lit = fagp_posterior(ds, Xs, model, want_cov=True, method="literal", delta2_variant=var_kind,
                                 memory_cap=1 << 40)
            out[pre + "literal_mean"] = lit.mean
            out[pre + "literal_var"] = np.diag(lit.cov).copy()
        print(name, "m =", es.size, "mean[0] =", res.mean[0], file=sys.stderr)
    # multi-index enumerations (bit-exact check)
    for n, p in [(1, 1), (3, 1), (2, 2), (4, 3), (10, 3), (8, 4), (6, 5), (3, 7)]:
        out[f"indices/{n}_{p}"] = multi_indices(n, p)
    # SpdFactor contract: jitter on a near-singular matrix (test_backend.py:128-137)
    rng = np.random.default_rng(10)
    q, _ = np.linalg.qr(rng.normal(size=(5, 5)))
    mm = (q * np.array([1.0, 0.9, 0.5, 0.2, -1e-15])) @ q.T
    mm = 0.5 * (mm + mm.T)
    out["spd/near_singular"] = mm
    out["spd/near_singular_jitter"] = np.array(SpdFactor(mm).jitter)
    # CSV schema of the bench / plotdata files (the reference's own golden headers)
    from fagp.bench import PLOTDATA_HEADER, RESULTS_HEADER

    out["headers/results"] = np.array(RESULTS_HEADER)
    out["headers/plotdata"] = np.array(PLOTDATA_HEADER)
    gold = Path("/root/reference/pkg/tests/golden")
    assert (gold / "results_header.txt").read_text().strip() == RESULTS_HEADER
    assert (gold / "plotdata_header.txt").read_text().strip() == PLOTDATA_HEADER
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, OUT.stat().st_size, "bytes", file=sys.stderr)


if __name__ == "__main__":
    main()
