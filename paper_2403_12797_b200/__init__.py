"""paper_2403_12797_b200 -- B200-native FAGP posterior (arXiv 2403.12797).

Drop-in for the fit/predict surface of the reference package ``fagp``
(/root/reference/pkg/src/fagp/__init__.py:13-69) on the hot path: eigen-decomposition,
fused feature generation + Gram on FP64 tensor cores, Cholesky/solves, and the fused
predictive mean + variance, all in hand-written sm_100a kernels (libfagp_b200.so, C ABI in
include/fagp_b200.h).  Importing works without a GPU; every compute call requires one.
"""

from .backend import PHASES, Backend, SpdFactor, TimingRecord, phase_scope, spd_solve
from .datagen import Dataset, generate
from .exact import exact_posterior, se_gram
from .errors import BudgetError, ConfigError, CsvFormatError, NumericalError
from .kernels import ArdKernelParams, KernelParams1D
from .mercer import (
    DEFAULT_MEMORY_CAP,
    DELTA2_RHO_LINEAR,
    DELTA2_RHO_SQUARED,
    LAMBDA_FLOOR_REL,
    Basis,
    EigenSystem,
    ShapeParams,
    basis_table,
    eigenfunction_1d,
    eigensystem,
    eigenvalues_1d,
    estimate_bytes,
    multi_indices,
    normalized_hermite,
    reconstruct_kernel,
    shape_params,
)
from .posterior import (
    Fit,
    GpModel,
    LambdaBarSolve,
    PosteriorResult,
    fagp_posterior,
    fagp_posterior_from_eigensystems,
    fit,
    lambda_bar,
    predict,
    set_fault_injection,
)

__version__ = "0.1.0"

__all__ = [
    "ArdKernelParams", "Backend", "Basis", "BudgetError", "ConfigError", "CsvFormatError", "Dataset",
    "DEFAULT_MEMORY_CAP", "DELTA2_RHO_LINEAR", "DELTA2_RHO_SQUARED", "EigenSystem", "Fit", "GpModel",
    "KernelParams1D", "LAMBDA_FLOOR_REL", "LambdaBarSolve", "NumericalError", "PHASES", "PosteriorResult",
    "ShapeParams", "SpdFactor", "TimingRecord", "basis_table", "eigenfunction_1d", "eigensystem",
    "eigenvalues_1d", "estimate_bytes", "exact_posterior", "fagp_posterior", "fagp_posterior_from_eigensystems", "fit",
    "generate", "lambda_bar", "multi_indices", "normalized_hermite", "phase_scope", "predict",
    "reconstruct_kernel", "se_gram", "set_fault_injection", "shape_params", "spd_solve", "__version__",
]
