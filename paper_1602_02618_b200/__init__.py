"""B200-native Chebyshev-Jacobi transform (arXiv 1602.02618).

Drop-in for the forward / inverse transform path of the reference package
``chebjac`` (plan / forward / inverse on coefficient vectors and (alpha, beta)),
its integer parameter shifts and jacobi_to_jacobi, the expansion-evaluation API
(evaluate_expansion, Clenshaw-Smith, forward recurrences), plus batched variants.  Planning runs on the host (bit-compatible with the
reference planner); execution runs in hand-written sm_100a kernels behind the
C ABI of include/cjt.h.  See DESIGN.md.
"""

from .backend import available_backends, kernel_backend, register_with, set_kernel_backend
from .engine import (
    CHEBYSHEV,
    JACOBI,
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
from .recurrences import (
    AngleGrid,
    clenshaw_smith,
    clenshaw_smith_reinsch,
    evaluate_expansion,
    evaluate_expansion_batched,
    jacobi_forward,
    jacobi_forward_reinsch,
)
from .shifts import (
    decrement_alpha,
    decrement_beta,
    from_core,
    from_core_batched,
    increment_alpha,
    increment_beta,
    jacobi_to_jacobi,
    jacobi_to_jacobi_batched,
    shift_batched,
    to_core,
    to_core_batched,
)

__version__ = "0.1.0"

__all__ = [
    "AngleGrid", "CHEBYSHEV", "CoefficientVector", "DEFAULT_EPS", "DEFAULT_M", "JACOBI",
    "JacobiParameters", "ParameterRangeError", "TransformPlan", "available_backends",
    "chebyshev", "forward", "forward_batched", "inverse", "inverse_batched", "jacobi",
    "kernel_backend", "pipeline", "plan", "register_with", "set_kernel_backend",
    "decrement_alpha", "decrement_beta", "from_core", "from_core_batched", "increment_alpha",
    "increment_beta", "jacobi_to_jacobi", "jacobi_to_jacobi_batched", "shift_batched", "to_core",
    "to_core_batched", "clenshaw_smith", "clenshaw_smith_reinsch", "evaluate_expansion",
    "evaluate_expansion_batched", "jacobi_forward", "jacobi_forward_reinsch",
]
