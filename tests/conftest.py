"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` runs on a B200 via gpurun.

GPU tests do NOT skip when the extension or the device is missing: the package has no
CPU fallback, so a missing libfagp_b200.so must fail the GPU suite loudly.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfagp_b200.so")
    config.addinivalue_line("markers", "slow: large-size GPU checks (seconds each)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN, allow_pickle=False))


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class Case:
    """A golden case: regenerated inputs (checked against the stored checksums) + outputs."""

    def __init__(self, g, name):
        from paper_2403_12797_b200.datagen import generate, test_inputs

        pre = name + "/"
        self.name = name
        self.p, self.M, self.N, self.Ns, self.seed = (int(v) for v in g[pre + "meta"])
        self.eps = g[pre + "eps"]
        self.rho = g[pre + "rho"]
        self.noise_var = float(g[pre + "noise_var"])
        self.mean_const = float(g[pre + "mean_const"])
        self.variant = str(g[pre + "variant"])
        ds = generate(self.N, self.p, self.seed, 0.05, domain=(-1.0, 1.0))
        self.X, self.y = ds.X, ds.y
        self.Xs = test_inputs(self.Ns, self.p, 0)
        assert _digest(self.X) + _digest(self.y) + _digest(self.Xs) == str(g[pre + "x_sha"]), name
        self.ref = {k[len(pre):]: v for k, v in g.items() if k.startswith(pre)}

    @property
    def m(self):
        return self.M**self.p

    def kernel(self):
        from paper_2403_12797_b200 import ArdKernelParams, KernelParams1D

        return ArdKernelParams(tuple(KernelParams1D(float(e), float(r)) for e, r in zip(self.eps, self.rho)))

    def model(self):
        from paper_2403_12797_b200 import GpModel

        return GpModel(self.kernel(), noise_var=self.noise_var, mean_const=self.mean_const, n_eigen=self.M)

    def dataset(self):
        from paper_2403_12797_b200 import Dataset

        return Dataset(X=self.X, y=self.y, noise_std=0.05, seed=self.seed, domain=((-1.0, 1.0),) * self.p)


CASE_NAMES = ["c1", "c2s", "c3s", "ard4", "lin2", "p1m40", "c5s", "c4s"]


@pytest.fixture(scope="session")
def cases(golden):
    return {n: Case(golden, n) for n in CASE_NAMES}


def rel_err(a, b):
    """Elementwise relative error max |a-b|/|b| (b nonzero)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b) / np.abs(b)))


def scaled_err(a, b):
    """max |a-b| / max |b| (the reference tests' measure, test_posterior.py:132)."""
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b)))
