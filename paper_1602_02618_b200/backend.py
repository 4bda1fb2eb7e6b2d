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

import collections
import ctypes
import hashlib
import threading
import types

import numpy as np

from . import _native as nat


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class _KernelPlan:
    """One cjt_kernel_plan (device tables + rows of one plugin call site)."""

    def __init__(self, kind, tables, thetas, cuts, regions, n_len):
        tabs = [_f64(t) for t in tables]
        thetas = _f64(thetas)
        cuts = np.ascontiguousarray(cuts, dtype=np.int64)
        regions = np.ascontiguousarray(regions, dtype=np.int8)
        npts = len(thetas)
        if not (len(cuts) == len(regions) == npts):
            raise ValueError("thetas, cuts and regions must have equal length")
        tl = min(len(t) for t in tabs)
        if kind == nat.CJT_KERNEL_CLENSHAW and npts and int(cuts.max()) + 1 > min(len(t) for t in tabs[:3]):
            raise ValueError("recurrence tables are shorter than the largest cut + 1")
        h = ctypes.c_void_p()
        nat.check(nat.lib().cjt_kernel_plan_create(
            kind, *[t.ctypes.data for t in tabs], tl, thetas.ctypes.data, cuts.ctypes.data,
            regions.ctypes.data, npts, int(n_len), ctypes.byref(h)), "cjt_kernel_plan_create")
        self.handle = h
        self.n_points = npts
        self.n_len = int(n_len)

    def execute(self, x, out):
        nat.check(nat.lib().cjt_kernel_plan_execute(self.handle, x.ctypes.data, out.ctypes.data),
                  "cjt_kernel_plan_execute")

    def __del__(self):
        h = getattr(self, "handle", None)
        lib_ = getattr(nat, "_lib", None) if nat is not None else None   # None at interpreter exit
        if h is not None and h.value and lib_ is not None:
            try:
                lib_.cjt_kernel_plan_destroy(h)
            except Exception:
                pass


# Plugin call sites -> device state.  The reference engine passes the same
# read-only plan arrays (tables, angles, cuts, regions; engine.py:118-119,
# kernels.py:362-363) on every forward / inverse, so the key is their identity
# (the cache holds references, so identities cannot be recycled while cached);
# a writeable array also contributes a digest of its contents.
_KCACHE: "collections.OrderedDict" = collections.OrderedDict()
_KCACHE_MAX = 16
_KLOCK = threading.Lock()


def _ident(a):
    a_ = np.asarray(a)
    key = (id(a), a_.shape, a_.dtype.str)
    if a_.flags.writeable:
        key += (hashlib.blake2b(np.ascontiguousarray(a_).tobytes(), digest_size=16).digest(),)
    return key


def _kernel_plan(kind, tables, thetas, cuts, regions, n_len) -> _KernelPlan:
    args = (*tables, thetas, cuts, regions)
    key = (kind, int(n_len), nat.current_device(), tuple(_ident(a) for a in args))
    with _KLOCK:
        hit = _KCACHE.get(key)
        if hit is not None:
            _KCACHE.move_to_end(key)
            return hit[0]
    kp = _KernelPlan(kind, tables, thetas, cuts, regions, n_len)
    with _KLOCK:
        _KCACHE[key] = (kp, args)
        while len(_KCACHE) > _KCACHE_MAX:
            _KCACHE.popitem(last=False)
    return kp


def clenshaw_points(A, B, C, rb_plus, rb_minus, rb_plus_inv, rb_minus_inv,
                    coeffs, thetas, cuts, regions, out):
    """out[i] = sum_{n < cuts[i]} coeffs[n] P_n(cos thetas[i]) on the GPU."""
    if out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array")
    if not (len(thetas) == len(out)):
        raise ValueError("thetas, cuts, regions and out must have equal length")
    coeffs = _f64(coeffs)
    kp = _kernel_plan(nat.CJT_KERNEL_CLENSHAW, (A, B, C, rb_plus, rb_minus, rb_plus_inv, rb_minus_inv),
                      thetas, cuts, regions, len(coeffs))
    kp.execute(coeffs, out)
    return None


def transpose_accumulate(A, B, C, rf_plus, rf_minus, rf_plus_inv, rf_minus_inv,
                         wv, thetas, cuts, regions, out):
    """out[n] += sum_i wv[i] P_n(cos thetas[i]) over i with n < cuts[i] on the GPU."""
    if out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array")
    wv = _f64(wv)
    if len(wv) != len(thetas):
        raise ValueError("thetas, cuts, regions and wv must have equal length")
    kp = _kernel_plan(nat.CJT_KERNEL_TRANSPOSE, (A, B, C, rf_plus, rf_minus, rf_plus_inv, rf_minus_inv),
                      thetas, cuts, regions, len(out))
    kp.execute(wv, out)
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
