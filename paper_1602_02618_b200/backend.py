"""Kernel-backend plugin with the reference's contract (chebjac/backend.py:13-53).

The reference engine looks kernels up in ``backend._BACKENDS[name]``; a module
there must export

    clenshaw_points(A, B, C, rb_plus, rb_minus, rb_plus_inv, rb_minus_inv,
                    coeffs, thetas, cuts, regions, out)        # overwrites out
    transpose_accumulate(A, B, C, rf_plus, rf_minus, rf_plus_inv, rf_minus_inv,
                         wv, thetas, cuts, regions, out)       # accumulates into out

with C-contiguous 1-d float64 arrays (int64 cuts, int8 regions)
(_kernels_cy.pyx:83-88, 201-206).  ``cuda_kernels`` implements both on the GPU
through libcjt_b200.so (cjt_clenshaw_points / cjt_transpose_accumulate), so a
reference installation can run its own engine with the B200 recurrence by
``register_with(chebjac.backend)`` followed by ``set_kernel_backend("cuda")``.
"""

from __future__ import annotations

import types

import numpy as np

from . import _native as nat


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def clenshaw_points(A, B, C, rb_plus, rb_minus, rb_plus_inv, rb_minus_inv,
                    coeffs, thetas, cuts, regions, out):
    """out[i] = sum_{n < cuts[i]} coeffs[n] P_n(cos thetas[i]) on the GPU."""
    if out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array")
    A, B, C = _f64(A), _f64(B), _f64(C)
    rbp, rbm, rbpi, rbmi = _f64(rb_plus), _f64(rb_minus), _f64(rb_plus_inv), _f64(rb_minus_inv)
    coeffs, thetas = _f64(coeffs), _f64(thetas)
    cuts = np.ascontiguousarray(cuts, dtype=np.int64)
    regions = np.ascontiguousarray(regions, dtype=np.int8)
    npts = len(thetas)
    if not (len(cuts) == len(regions) == len(out) == npts):
        raise ValueError("thetas, cuts, regions and out must have equal length")
    if npts and int(cuts.max()) + 1 > min(len(A), len(B), len(C)):
        raise ValueError("recurrence tables are shorter than the largest cut + 1")
    nat.check(nat.lib().cjt_clenshaw_points(
        A.ctypes.data, B.ctypes.data, C.ctypes.data, rbp.ctypes.data, rbm.ctypes.data,
        rbpi.ctypes.data, rbmi.ctypes.data, coeffs.ctypes.data, len(coeffs),
        thetas.ctypes.data, cuts.ctypes.data, regions.ctypes.data, out.ctypes.data, npts),
        "cjt_clenshaw_points")
    return None


def transpose_accumulate(A, B, C, rf_plus, rf_minus, rf_plus_inv, rf_minus_inv,
                         wv, thetas, cuts, regions, out):
    """out[n] += sum_i wv[i] P_n(cos thetas[i]) over i with n < cuts[i] on the GPU."""
    if out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array")
    A, B, C = _f64(A), _f64(B), _f64(C)
    rfp, rfm, rfpi, rfmi = _f64(rf_plus), _f64(rf_minus), _f64(rf_plus_inv), _f64(rf_minus_inv)
    wv, thetas = _f64(wv), _f64(thetas)
    cuts = np.ascontiguousarray(cuts, dtype=np.int64)
    regions = np.ascontiguousarray(regions, dtype=np.int8)
    npts = len(thetas)
    if not (len(cuts) == len(regions) == len(wv) == npts):
        raise ValueError("thetas, cuts, regions and wv must have equal length")
    tl = min(len(A), len(B), len(C), len(rfp), len(rfm), len(rfpi), len(rfmi))
    nat.check(nat.lib().cjt_transpose_accumulate(
        A.ctypes.data, B.ctypes.data, C.ctypes.data, rfp.ctypes.data, rfm.ctypes.data,
        rfpi.ctypes.data, rfmi.ctypes.data, wv.ctypes.data, thetas.ctypes.data,
        cuts.ctypes.data, regions.ctypes.data, out.ctypes.data, len(out), npts, tl),
        "cjt_transpose_accumulate")
    return None


cuda_kernels = types.ModuleType("cuda_kernels")
cuda_kernels.clenshaw_points = clenshaw_points
cuda_kernels.transpose_accumulate = transpose_accumulate

_BACKENDS = {"cuda": cuda_kernels}
_active_name = "cuda"


def available_backends():
    return dict(_BACKENDS)


def kernel_backend() -> str:
    return _active_name


def set_kernel_backend(name: str) -> str:
    """Same contract as chebjac.backend.set_kernel_backend (backend.py:42-49)."""
    global _active_name
    if name not in _BACKENDS:
        raise ValueError(f"unknown backend {name!r}; available: {sorted(_BACKENDS)}")
    prev = _active_name
    _active_name = name
    return prev


def kernels():
    return _BACKENDS[_active_name]


def register_with(reference_backend_module, name: str = "cuda"):
    """Insert the GPU kernels into a reference installation's backend registry
    (chebjac.backend._BACKENDS, backend.py:13-15)."""
    reference_backend_module._BACKENDS[name] = cuda_kernels
    return name
