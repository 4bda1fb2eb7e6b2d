"""Public API: same names, argument meaning and error behaviour as the
reference's engine (chebjac/engine.py:36-227, parameters.py)."""
import numpy as np
import pytest

import paper_1602_02618_b200 as cj
from paper_1602_02618_b200 import backend


def test_public_names():
    for name in ("plan", "forward", "inverse", "jacobi", "chebyshev", "CoefficientVector",
                 "TransformPlan", "JacobiParameters", "ParameterRangeError", "CHEBYSHEV", "JACOBI",
                 "forward_batched", "inverse_batched", "set_kernel_backend", "kernel_backend",
                 "available_backends"):
        assert hasattr(cj, name), name
    assert issubclass(cj.ParameterRangeError, ValueError)


def test_coefficient_vector_validation():
    p = cj.JacobiParameters(0.0, 0.0)
    with pytest.raises(ValueError):
        cj.jacobi(p, [])
    with pytest.raises(ValueError):
        cj.jacobi(p, np.ones((2, 2)))
    with pytest.raises(ValueError):
        cj.jacobi(p, [1.0, np.nan])
    with pytest.raises(ValueError):
        cj.CoefficientVector(cj.JACOBI, np.ones(3))
    with pytest.raises(ValueError):
        cj.CoefficientVector(cj.CHEBYSHEV, np.ones(3), p)
    with pytest.raises(ValueError):
        cj.CoefficientVector("legendre", np.ones(3))
    assert cj.chebyshev([1, 2, 3]).n == 2


def test_plan_errors_and_attributes():
    p = cj.JacobiParameters(-0.25, 0.4)
    with pytest.raises(cj.ParameterRangeError):
        cj.plan("forward", cj.JacobiParameters(0.75, 0.0), 16)
    with pytest.raises(ValueError):
        cj.plan("both", p, 16)
    fp = cj.plan("forward", p, 255)
    ip = cj.plan("inverse", p, 255)
    assert fp.grid_n == 255 and ip.grid_n == 510
    assert fp.weights is None and ip.weights is not None and ip.scalings.shape == (256,)
    assert len(fp.cuts) == 256 and len(ip.cuts) == 511


def test_execution_input_checks_precede_device_use():
    p = cj.JacobiParameters(-0.25, 0.4)
    fp = cj.plan("forward", p, 15)
    ip = cj.plan("inverse", p, 15)
    with pytest.raises(ValueError):
        cj.inverse(fp, cj.chebyshev(np.ones(16)))
    with pytest.raises(ValueError):
        cj.forward(fp, cj.chebyshev(np.ones(16)))
    with pytest.raises(ValueError):
        cj.forward(fp, cj.jacobi(cj.JacobiParameters(0.0, 0.0), np.ones(16)))
    with pytest.raises(ValueError):
        cj.forward(fp, cj.jacobi(p, np.ones(15)))
    with pytest.raises(ValueError):
        cj.forward_batched(ip, np.ones((2, 16)))
    with pytest.raises(ValueError):
        cj.forward_batched(fp, np.ones((2, 15)))
    with pytest.raises(ValueError):
        cj.inverse_batched(ip, np.full((2, 16), np.inf))


def test_backend_registry_contract():
    assert set(cj.available_backends()) == {"cuda"}
    assert cj.kernel_backend() == "cuda"
    assert cj.set_kernel_backend("cuda") == "cuda"
    with pytest.raises(ValueError):
        cj.set_kernel_backend("cython")
    import inspect
    sig = inspect.signature(backend.clenshaw_points)
    assert list(sig.parameters) == ["A", "B", "C", "rb_plus", "rb_minus", "rb_plus_inv",
                                    "rb_minus_inv", "coeffs", "thetas", "cuts", "regions", "out"]
    sig = inspect.signature(backend.transpose_accumulate)
    assert list(sig.parameters) == ["A", "B", "C", "rf_plus", "rf_minus", "rf_plus_inv",
                                    "rf_minus_inv", "wv", "thetas", "cuts", "regions", "out"]


def test_register_with_reference_registry():
    import types
    fake = types.SimpleNamespace(_BACKENDS={"numpy": object()})
    assert cj.register_with(fake) == "cuda"
    assert fake._BACKENDS["cuda"] is backend.cuda_kernels
