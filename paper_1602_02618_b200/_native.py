"""ctypes binding of the C ABI in include/cjt.h (libcjt_b200.so).

The library is the only compute path of the package: there is no CPU
fallback.  Loading fails loudly (ImportError / RuntimeError) when the shared
object is missing or no CUDA device is visible.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_lib" / "libcjt_b200.so"

CJT_OK, CJT_EINVAL, CJT_ECUDA, CJT_ENOMEM, CJT_ENODEV = 0, 1, 2, 3, 4
CJT_FORWARD, CJT_INVERSE = 0, 1

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_dp = ctypes.POINTER(ctypes.c_double)


class ChirpZDesc(ctypes.Structure):
    _fields_ = [
        ("p0", _i64), ("width", _i64), ("q0", _i64), ("count", _i64), ("length", _i64),
        ("m_count", _i32), ("accumulate", _i32),
        ("pre", _p), ("post", _p),
        ("n_tiles_in", _i32), ("n_tiles_out", _i32), ("tiles_in", _p), ("tiles_out", _p),
        ("kernel_hat", _p), ("out_shift", _i64),
        ("device_tables", _i32), ("pre_kind", _i32), ("post_kind", _i32),
        ("grid_g", _i64), ("pre_row0", _i64), ("post_row0", _i64),
    ]


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("direction", _i32), ("m_terms", _i32), ("n", _i64), ("grid_n", _i64),
        ("x", _p), ("xm", _p), ("regions", _p), ("cuts", _p),
        ("table_len", _i64),
        ("A", _p), ("B", _p), ("C", _p),
        ("rf_plus", _p), ("rf_minus", _p), ("rf_plus_inv", _p), ("rf_minus_inv", _p),
        ("n_blocks", _i32), ("blocks", ctypes.POINTER(ChirpZDesc)),
        ("edge", ChirpZDesc),
        ("scalings", _p), ("half_k", _p),
        ("thetas", _p), ("alpha", ctypes.c_double), ("beta", ctypes.c_double),
        ("half_gemm", _i32),
    ]


class PlanStats(ctypes.Structure):
    _fields_ = [
        ("launches_per_execute", _i64), ("rec_steps", _i64), ("checkpoint_bytes", _i64),
        ("workspace_bytes", _i64), ("reserved_batch", _i64),
        ("rec_flops_per_vector", ctypes.c_double), ("fft_points_per_vector", ctypes.c_double),
        ("rec_steps_executed", _i64),
    ]


class NativeError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libcjt_b200.so (once)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the package has no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    L.cjt_version.restype = ctypes.c_int
    L.cjt_last_error.restype = ctypes.c_char_p
    L.cjt_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
    L.cjt_plan_create.argtypes = [ctypes.POINTER(PlanDesc), ctypes.POINTER(_p)]
    L.cjt_plan_destroy.argtypes = [_p]
    L.cjt_plan_reserve.argtypes = [_p, _i64]
    L.cjt_plan_stats_get.argtypes = [_p, ctypes.POINTER(PlanStats)]
    L.cjt_execute.argtypes = [_p, _p, _p, _i64, _p]
    L.cjt_execute_host.argtypes = [_p, _p, _p, _i64, _p]
    L.cjt_execute_stage.argtypes = [_p, _p, _p, _i64, _i32, _p]
    L.cjt_probe_fp64_peak.argtypes = [ctypes.POINTER(ctypes.c_double), _p]
    L.cjt_clenshaw_points.argtypes = [_p] * 8 + [_i64, _p, _p, _p, _p, _i64]
    L.cjt_transpose_accumulate.argtypes = [_p] * 12 + [_i64, _i64, _i64]
    L.cjt_host_angles.argtypes = [_p, _p, _i64, _p, _p]
    L.cjt_host_half_exact.argtypes = [_p, _p, _p, _i64, _i64, _p, _p, _p]
    L.cjt_host_moments.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, _i64, _p]
    L.cjt_jacobi_shift.argtypes = [_i32, ctypes.c_double, ctypes.c_double, _p, _p, _i64, _i64, _p]
    L.cjt_clenshaw_points_dev.argtypes = [_p] * 7 + [_i64, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _i64, _p]
    L.cjt_jacobi_values.argtypes = [_p] * 5 + [_i64, _i64, _p, _p, _i64, _p]
    L.cjt_clenshaw_smith_points.argtypes = [_p] * 6 + [_i64, _p, _p, _i64, _p]
    L.cjt_chirpz_create.argtypes = [ctypes.POINTER(ChirpZDesc), ctypes.POINTER(_p)]
    L.cjt_chirpz_execute.argtypes = [_p, _p, _i64, _p, _i64, _i64, _p]
    L.cjt_chirpz_destroy.argtypes = [_p]
    L.cjt_kernel_plan_create.argtypes = [_i32] + [_p] * 7 + [_i64, _p, _p, _p, _i64, _i64, ctypes.POINTER(_p)]
    L.cjt_kernel_plan_execute.argtypes = [_p, _p, _p]
    L.cjt_kernel_plan_destroy.argtypes = [_p]
    for name in ("cjt_device_count", "cjt_plan_create", "cjt_plan_destroy", "cjt_plan_reserve",
                 "cjt_plan_stats_get", "cjt_execute", "cjt_execute_host", "cjt_clenshaw_points",
                 "cjt_transpose_accumulate", "cjt_host_angles", "cjt_host_moments", "cjt_host_half_exact",
                 "cjt_jacobi_shift", "cjt_execute_stage", "cjt_probe_fp64_peak",
                 "cjt_clenshaw_points_dev", "cjt_jacobi_values", "cjt_clenshaw_smith_points",
                 "cjt_chirpz_create", "cjt_chirpz_execute", "cjt_chirpz_destroy",
                 "cjt_kernel_plan_create", "cjt_kernel_plan_execute", "cjt_kernel_plan_destroy"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


EXPORTED_SYMBOLS = (
    "cjt_version", "cjt_last_error", "cjt_device_count", "cjt_plan_create", "cjt_plan_destroy",
    "cjt_plan_reserve", "cjt_plan_stats_get", "cjt_execute", "cjt_execute_host",
    "cjt_clenshaw_points", "cjt_transpose_accumulate", "cjt_host_angles", "cjt_host_moments",
    "cjt_jacobi_shift", "cjt_execute_stage", "cjt_probe_fp64_peak", "cjt_clenshaw_points_dev",
    "cjt_jacobi_values", "cjt_clenshaw_smith_points", "cjt_chirpz_create", "cjt_chirpz_execute",
    "cjt_chirpz_destroy", "cjt_host_half_exact", "cjt_kernel_plan_create", "cjt_kernel_plan_execute",
    "cjt_kernel_plan_destroy",
)
CJT_KERNEL_CLENSHAW, CJT_KERNEL_TRANSPOSE = 0, 1
CJT_DIAG_ARRAY, CJT_DIAG_MODULATION = 0, 1
SHIFT_INC_BETA, SHIFT_DEC_BETA, SHIFT_INC_ALPHA, SHIFT_DEC_ALPHA = 0, 1, 2, 3
STAGE_REC, STAGE_BLOCKS, STAGE_EDGE, STAGE_ALL = 1, 2, 4, 7


def check(rc: int, what: str = "cjt"):
    if rc == CJT_OK:
        return
    msg = lib().cjt_last_error().decode(errors="replace")
    if rc == CJT_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if rc == CJT_ENOMEM:
        raise MemoryError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")


def current_device() -> int:
    """The calling thread's current CUDA device (0 without torch / CUDA)."""
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except ImportError:
        pass
    return 0


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = lib().cjt_device_count(ctypes.byref(n))
    return n.value if rc == CJT_OK else 0


def ptr(arr) -> int:
    """Address of a C-contiguous numpy array or a torch tensor."""
    if hasattr(arr, "data_ptr"):
        return arr.data_ptr()
    return arr.ctypes.data


def env_flag(name: str) -> bool:
    return os.environ.get(name, "").strip() not in ("", "0")
