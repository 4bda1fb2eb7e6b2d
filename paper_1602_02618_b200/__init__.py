"""B200-native Chebyshev-Jacobi transform (arXiv 1602.02618).

Drop-in for the forward / inverse transform path of the reference package
``chebjac`` (plan / forward / inverse on coefficient vectors and (alpha, beta)),
plus batched variants.  Planning runs on the host (bit-compatible with the
reference planner); execution runs in hand-written sm_100a kernels behind the
C ABI of include/cjt.h.  See DESIGN.md.
"""

from .backend import available_backends, kernel_backend, register_with, set_kernel_backend
from .engine import (
    CHEBYSHEV,
    JACOBI,
    AngleGrid,
    CoefficientVector,
    TransformPlan,
    chebyshev,
    forward,
    forward_batched,
    inverse,
    inverse_batched,
    jacobi,
    pipeline,
    plan,
)
from .planner import DEFAULT_EPS, DEFAULT_M, JacobiParameters, ParameterRangeError

__version__ = "0.1.0"

__all__ = [
    "AngleGrid", "CHEBYSHEV", "CoefficientVector", "DEFAULT_EPS", "DEFAULT_M", "JACOBI",
    "JacobiParameters", "ParameterRangeError", "TransformPlan", "available_backends",
    "chebyshev", "forward", "forward_batched", "inverse", "inverse_batched", "jacobi",
    "kernel_backend", "pipeline", "plan", "register_with", "set_kernel_backend",
]
