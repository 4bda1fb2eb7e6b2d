"""Jacobi polynomial / expansion evaluation at angles, on the GPU.

Mirrors the reference module ``chebjac.recurrences`` (recurrences.py:1-171):
``AngleGrid``, ``classify_region(s)``, ``jacobi_forward``,
``jacobi_forward_reinsch``, ``clenshaw_smith``, ``clenshaw_smith_reinsch`` and
``evaluate_expansion`` keep the reference's names, argument meaning, checks
and exceptions.  Every evaluation runs in libcjt_b200.so:

* ``jacobi_forward[_reinsch]``  -> ``cjt_jacobi_values`` (k_jacobi_values);
* ``clenshaw_smith[_reinsch]`` -> ``cjt_clenshaw_smith_points`` (the scalar
  helpers' operation order: the Reinsch step divides by rb_n);
* ``evaluate_expansion`` -> the active kernel backend's ``clenshaw_points``
  (the GPU plugin, ``cjt_clenshaw_points``), exactly as the reference
  dispatches (recurrences.py:155-171);
* ``evaluate_expansion_batched`` -> ``cjt_clenshaw_points_dev`` on CUDA
  tensors (B expansions of one degree at once, stream ordered).

All of them use the reference's operation order, so results are
bit-identical to the reference's Cython kernel / Python loops (the host libm
supplies cos(theta) and the half-angle x -+ 1, as in the reference).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import backend
from . import planner as pl
from .planner import (BREAK_HI, BREAK_LO, INTERIOR, NEAR_MINUS_ONE, NEAR_PLUS_ONE, JacobiParameters,
                      RecurrenceTables, recurrence_tables)

__all__ = [
    "AngleGrid", "BREAK_HI", "BREAK_LO", "INTERIOR", "NEAR_MINUS_ONE", "NEAR_PLUS_ONE",
    "classify_region", "classify_regions", "clenshaw_smith", "clenshaw_smith_reinsch",
    "evaluate_expansion", "evaluate_expansion_batched", "jacobi_forward", "jacobi_forward_reinsch",
]


def classify_region(theta: float) -> int:
    """Region code of one angle (recurrences.py:32-38)."""
    if theta < BREAK_LO:
        return NEAR_PLUS_ONE
    if theta > BREAK_HI:
        return NEAR_MINUS_ONE
    return INTERIOR


def classify_regions(thetas: np.ndarray) -> np.ndarray:
    """Region codes of an angle array (recurrences.py:41-45)."""
    return pl.region_codes(np.asarray(thetas))


@dataclass(frozen=True)
class AngleGrid:
    """theta_j = pi j / N, j = 0..N (recurrences.py:48-66); read-only angles.

    ``AngleGrid(n)`` as in the reference; plans pass their own (identical)
    angle array to skip recomputing it."""

    n: int
    angles: np.ndarray = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if self.angles is None:
            object.__setattr__(self, "angles", pl.angle_grid(self.n))
        elif self.n < 1:
            raise ValueError("grid parameter N must be >= 1")

    def __len__(self):
        return self.n + 1


def _check_theta(theta):
    if not 0.0 <= theta <= math.pi:
        raise ValueError(f"theta must lie in [0, pi], got {theta}")


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _values(t: RecurrenceTables, n_max: int, theta: float, mode: int) -> np.ndarray:
    if n_max < 0:
        raise ValueError("n_max must be >= 0")
    A, B, C, rfp, rfm = (_f64(v) for v in (t.A, t.B, t.C, t.rf_plus, t.rf_minus))
    tl = min(len(A), len(B), len(C), len(rfp), len(rfm))
    if tl < n_max:
        raise ValueError("recurrence tables are shorter than n_max")
    th = np.array([theta], dtype=np.float64)
    md = np.array([mode], dtype=np.int8)
    out = np.empty(n_max + 1)
    nat.check(nat.lib().cjt_jacobi_values(A.ctypes.data, B.ctypes.data, C.ctypes.data, rfp.ctypes.data,
                                          rfm.ctypes.data, tl, n_max, th.ctypes.data, md.ctypes.data, 1,
                                          out.ctypes.data), "cjt_jacobi_values")
    return out


def jacobi_forward(p: JacobiParameters, n_max: int, theta: float,
                   tables: RecurrenceTables | None = None) -> np.ndarray:
    """P_0 .. P_{n_max} at cos(theta) by the unmodified forward recurrence
    (recurrences.py:74-87)."""
    _check_theta(theta)
    t = tables if tables is not None else recurrence_tables(p, max(n_max, 1))
    return _values(t, n_max, theta, 0)


def jacobi_forward_reinsch(p: JacobiParameters, n_max: int, theta: float, end: int,
                           tables: RecurrenceTables | None = None) -> np.ndarray:
    """P_0 .. P_{n_max} at cos(theta) by Reinsch's modified forward recurrence
    anchored at x0 = end (+1 or -1) (recurrences.py:90-112)."""
    _check_theta(theta)
    t = tables if tables is not None else recurrence_tables(p, max(n_max, 1))
    if end not in (1, -1):
        raise ValueError("end must be +1 or -1")
    return _values(t, n_max, theta, end)


def _clenshaw_one(p, coeffs, theta, mode, tables):
    coeffs = np.asarray(coeffs, dtype=float)
    if coeffs.ndim != 1:
        raise ValueError("coeffs must be a 1-d sequence")
    if coeffs.size == 0:
        if mode == INTERIOR:
            return 0.0   # the reference's empty backward loop returns u1 = 0
        raise IndexError("index 0 is out of bounds for axis 0 with size 0")
    n_max = len(coeffs) - 1
    t = tables if tables is not None else recurrence_tables(p, n_max + 1)
    A, B, C, rbp, rbm = (_f64(v) for v in (t.A, t.B, t.C, t.rb_plus, t.rb_minus))
    if min(len(A), len(B), len(C), len(rbp), len(rbm)) < n_max + 2:
        raise ValueError("recurrence tables are shorter than len(coeffs) + 1")
    c = _f64(coeffs)
    th = np.array([theta], dtype=np.float64)
    md = np.array([mode], dtype=np.int8)
    out = np.empty(1)
    nat.check(nat.lib().cjt_clenshaw_smith_points(A.ctypes.data, B.ctypes.data, C.ctypes.data,
                                                  rbp.ctypes.data, rbm.ctypes.data, c.ctypes.data,
                                                  len(c), th.ctypes.data, md.ctypes.data, 1,
                                                  out.ctypes.data), "cjt_clenshaw_smith_points")
    return float(out[0])


def clenshaw_smith(p: JacobiParameters, coeffs, theta: float,
                   tables: RecurrenceTables | None = None) -> float:
    """sum_n coeffs[n] P_n(cos theta) by the backward inhomogeneous recurrence
    (recurrences.py:115-127)."""
    _check_theta(theta)
    return _clenshaw_one(p, coeffs, theta, INTERIOR, tables)


def clenshaw_smith_reinsch(p: JacobiParameters, coeffs, theta: float, end: int,
                           tables: RecurrenceTables | None = None) -> float:
    """The same sum by the Reinsch-modified algorithm with the backward
    endpoint ratios (recurrences.py:130-152)."""
    _check_theta(theta)
    if end not in (1, -1):
        raise ValueError("end must be +1 or -1")
    return _clenshaw_one(p, coeffs, theta, end, tables)


def evaluate_expansion(p: JacobiParameters, coeffs, grid: AngleGrid,
                       tables: RecurrenceTables | None = None) -> np.ndarray:
    """sum_n coeffs[n] P_n at every grid angle, per-angle dispatch to the
    unmodified or Reinsch-modified Clenshaw-Smith algorithm
    (recurrences.py:155-171), through the active kernel backend."""
    coeffs = np.ascontiguousarray(coeffs, dtype=float)
    n_max = len(coeffs) - 1
    t = tables if tables is not None else recurrence_tables(p, n_max + 1)
    thetas = grid.angles
    cuts = np.full(len(thetas), n_max + 1, dtype=np.int64)
    regions = classify_regions(thetas)
    out = np.empty(len(thetas))
    backend.kernels().clenshaw_points(
        t.A, t.B, t.C, t.rb_plus, t.rb_minus, t.rb_plus_inv, t.rb_minus_inv,
        coeffs, np.ascontiguousarray(thetas), cuts, regions, out,
    )
    return out


class _GridDev:
    """Device copies of one (p, n_max, grid) evaluation setup (cached)."""

    def __init__(self, p, n_max, grid, device):
        import torch

        t = recurrence_tables(p, n_max + 1)
        thetas = np.ascontiguousarray(grid.angles, dtype=np.float64)
        regions = classify_regions(thetas)
        x = np.empty(len(thetas))
        xm = np.empty(len(thetas))
        nat.check(nat.lib().cjt_host_angles(thetas.ctypes.data, regions.ctypes.data, len(thetas),
                                            x.ctypes.data, xm.ctypes.data), "cjt_host_angles")

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(device)

        self.tabs = [up(_f64(v)) for v in (t.A, t.B, t.C, t.rb_plus, t.rb_minus, t.rb_plus_inv,
                                            t.rb_minus_inv)]
        self.table_len = min(len(v) for v in self.tabs)
        self.x, self.xm = up(x), up(xm)
        self.cuts = up(np.full(len(thetas), n_max + 1, dtype=np.int64))
        self.regions = up(regions)
        self.npts = len(thetas)


_GRID_CACHE: dict = {}


def evaluate_expansion_batched(p: JacobiParameters, coeffs, grid: AngleGrid, out=None, stream=None):
    """Batched ``evaluate_expansion``: ``coeffs`` (B, n+1) float64 CUDA tensor
    (or NumPy array -> NumPy result); returns (B, len(grid)) values, each row
    bit-identical to ``evaluate_expansion`` of that row.  Device path only
    (cjt_clenshaw_points_dev); stream ordered on ``stream`` or torch's current
    stream."""
    import torch

    host = isinstance(coeffs, np.ndarray)
    if host:
        if not torch.cuda.is_available():
            raise RuntimeError("evaluate_expansion_batched needs a CUDA device (no CPU fallback)")
        c = torch.from_numpy(np.ascontiguousarray(coeffs, dtype=np.float64)).cuda()
    else:
        c = coeffs
        if not c.is_cuda:
            raise ValueError("coeffs must be a CUDA tensor or a NumPy array")
        if c.dtype != torch.float64:
            raise ValueError("coeffs must be float64")
    if c.dim() != 2 or c.shape[1] == 0:
        raise ValueError("coeffs must be (batch, n+1) with n >= 0")
    c = c.contiguous()
    batch, n1 = c.shape
    dev = c.device
    key = (p.alpha, p.beta, n1 - 1, grid.n, dev.index)
    g = _GRID_CACHE.get(key)
    if g is None:
        if len(_GRID_CACHE) >= 16:
            _GRID_CACHE.pop(next(iter(_GRID_CACHE)))
        g = _GRID_CACHE[key] = _GridDev(p, n1 - 1, grid, dev)
    if out is None:
        out = torch.empty((batch, g.npts), dtype=torch.float64, device=dev)
    elif tuple(out.shape) != (batch, g.npts) or out.dtype != torch.float64 or not out.is_contiguous():
        raise ValueError("out must be a contiguous float64 (batch, len(grid)) tensor")
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    L = nat.lib()
    done = 0
    while done < batch:   # the grid's y dimension caps one launch at 65535 vectors
        nb = min(65535, batch - done)
        nat.check(L.cjt_clenshaw_points_dev(
            *[t.data_ptr() for t in g.tabs], g.table_len, c[done].data_ptr(), n1, g.x.data_ptr(),
            g.xm.data_ptr(), g.cuts.data_ptr(), g.regions.data_ptr(), out[done].data_ptr(), g.npts,
            g.npts, nb, st.cuda_stream), "cjt_clenshaw_points_dev")
        done += nb
    if host:
        return out.cpu().numpy()
    return out
