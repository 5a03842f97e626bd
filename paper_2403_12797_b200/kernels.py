"""Kernel hyper-parameter types (mirror of /root/reference/pkg/src/fagp/kernels.py:28-81).

Same names, fields and validation as the reference, so code written against
``fagp.KernelParams1D`` / ``fagp.ArdKernelParams`` runs unchanged.  Every function in this
package also accepts the reference's own objects (anything with ``per_dim`` entries that
carry ``epsilon`` and ``rho``), see :func:`as_ard`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["KernelParams1D", "ArdKernelParams", "as_ard"]


@dataclass(frozen=True)
class KernelParams1D:
    """Univariate SE kernel exp(-eps^2 (x - x')^2) with eigen-decay scale rho (kernels.py:28-49)."""

    epsilon: float
    rho: float = 1.0

    def __post_init__(self):
        if not np.isfinite(self.epsilon) or self.epsilon < 0:
            raise ValueError(f"epsilon must be finite and >= 0, got {self.epsilon!r}")
        if not np.isfinite(self.rho) or self.rho <= 0:
            raise ValueError(f"rho must be finite and > 0, got {self.rho!r}")


@dataclass(frozen=True)
class ArdKernelParams:
    """Per-dimension SE parameters for p-variate inputs (kernels.py:52-81)."""

    per_dim: tuple

    def __post_init__(self):
        per_dim = tuple(self.per_dim)
        if len(per_dim) < 1:
            raise ValueError("ArdKernelParams needs at least one dimension")
        if not all(isinstance(k, KernelParams1D) for k in per_dim):
            raise TypeError("per_dim entries must be KernelParams1D")
        object.__setattr__(self, "per_dim", per_dim)

    @classmethod
    def isotropic(cls, p, epsilon, rho=1.0):
        return cls(tuple(KernelParams1D(epsilon, rho) for _ in range(p)))

    @property
    def p(self):
        return len(self.per_dim)

    @property
    def epsilons(self):
        return np.array([k.epsilon for k in self.per_dim])

    @property
    def rhos(self):
        return np.array([k.rho for k in self.per_dim])


def as_ard(params):
    """Normalise ours or the reference's parameter object (duck-typed) to ArdKernelParams."""
    if isinstance(params, ArdKernelParams):
        return params
    per_dim = getattr(params, "per_dim", None)
    if per_dim is None:
        if hasattr(params, "epsilon") and hasattr(params, "rho"):
            per_dim = (params,)
        else:
            raise TypeError(f"expected kernel parameters with per_dim, got {type(params).__name__}")
    return ArdKernelParams(tuple(KernelParams1D(float(k.epsilon), float(k.rho)) for k in per_dim))
