"""Integer parameter shifts and Jacobi-to-Jacobi conversion on the GPU
(reference engine.py:232-354).

Same names, arguments, results and errors as the reference:
``increment_beta / decrement_beta / increment_alpha / decrement_alpha``
(bidiagonal change of basis, O(N)), ``to_core / from_core`` (integer shifts
into / out of the core square (-1/2, 1/2]^2) and ``jacobi_to_jacobi``
(shifts -> forward CJT -> inverse CJT at the target's core pair -> shifts).
Every operation runs in the native library (``cjt_jacobi_shift`` and the
transform plans); the ``*_batched`` variants take (B, N+1) float64 CUDA
tensors and stay on the device, stream ordered.
"""

from __future__ import annotations

import collections
import math
import threading

import numpy as np

from . import _native as nat
from . import engine
from .engine import JACOBI, CoefficientVector, jacobi
from .planner import DEFAULT_EPS, DEFAULT_M, JacobiParameters, ParameterRangeError

_OPS = {"increment_beta": (nat.SHIFT_INC_BETA, 0, 1), "decrement_beta": (nat.SHIFT_DEC_BETA, 0, -1),
        "increment_alpha": (nat.SHIFT_INC_ALPHA, 1, 0), "decrement_alpha": (nat.SHIFT_DEC_ALPHA, -1, 0)}


def _shifted(p: JacobiParameters, dalpha: int = 0, dbeta: int = 0) -> JacobiParameters:
    """engine.py:232-236 (same message and exception chaining)."""
    try:
        return JacobiParameters(p.alpha + dalpha, p.beta + dbeta)
    except ParameterRangeError as exc:
        raise ParameterRangeError(f"inadmissible shift target: {exc}") from exc


def _require_jacobi(c: CoefficientVector):
    if c.basis != JACOBI:
        raise ValueError("parameter shifts require Jacobi coefficients")


def _raw_stream(stream, device):
    """cudaStream_t handle of a torch stream, a raw handle, or the current stream."""
    import torch
    if stream is None:
        return torch.cuda.current_stream(device).cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _cuda_2d(x):
    import torch
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.dim() == 2):
        raise ValueError("expected a (B, N+1) float64 CUDA tensor")
    return x.contiguous()


def shift_batched(op: str, p: JacobiParameters, x, out=None, stream=None):
    """Apply one shift (`op` = 'increment_beta', ...) to every row of the
    (B, N+1) CUDA tensor `x` in basis `p`.  Returns (out, shifted params)."""
    import torch
    if op not in _OPS:
        raise ValueError(f"unknown shift {op!r}")
    code, da, db = _OPS[op]
    target = _shifted(p, da, db)
    x = _cuda_2d(x)
    if out is None:
        out = engine.empty_on_stream(x, stream)
    elif out.shape != x.shape or not out.is_contiguous() or out.dtype != torch.float64:
        raise ValueError("out must be a contiguous float64 tensor shaped like x")
    st = _raw_stream(stream, x.device)
    b, n1 = x.shape
    with torch.cuda.device(x.device):
        for b0 in range(0, b, 65535):   # the decrement kernel runs one CTA per row
            b1 = min(b, b0 + 65535)
            nat.check(nat.lib().cjt_jacobi_shift(code, p.alpha, p.beta, x[b0:b1].data_ptr(),
                                                 out[b0:b1].data_ptr(), n1 - 1, b1 - b0, st), op)
    return out, target


def _one(op: str, c: CoefficientVector) -> CoefficientVector:
    import torch
    _require_jacobi(c)
    code, da, db = _OPS[op]
    _shifted(c.params, da, db)   # raise before touching the device
    dev = torch.device("cuda", engine._current_device())
    x = torch.from_numpy(c.data).to(dev).view(1, -1)
    y, target = shift_batched(op, c.params, x)
    return jacobi(target, y.view(-1).cpu().numpy())


def increment_beta(c: CoefficientVector) -> CoefficientVector:
    """(alpha, beta) -> (alpha, beta + 1) basis, O(N) (engine.py:239-248)."""
    return _one("increment_beta", c)


def decrement_beta(c: CoefficientVector) -> CoefficientVector:
    """Inverse of increment_beta (engine.py:251-267)."""
    return _one("decrement_beta", c)


def increment_alpha(c: CoefficientVector) -> CoefficientVector:
    """Alpha shift by the parity symmetry (engine.py:277-282)."""
    return _one("increment_alpha", c)


def decrement_alpha(c: CoefficientVector) -> CoefficientVector:
    """engine.py:285-288."""
    return _one("decrement_alpha", c)


def _core_offsets(p: JacobiParameters) -> tuple:
    """Integer (da, db) with (alpha - da, beta - db) in the core square (engine.py:296-302)."""
    return math.ceil(p.alpha - 0.5), math.ceil(p.beta - 0.5)


def _to_core_ops(p: JacobiParameters):
    da, db = _core_offsets(p)
    return (["decrement_alpha"] * max(da, 0) + ["increment_alpha"] * max(-da, 0)
            + ["decrement_beta"] * max(db, 0) + ["increment_beta"] * max(-db, 0))


def _from_core_ops(target: JacobiParameters):
    da, db = _core_offsets(target)
    return (["increment_alpha"] * max(da, 0) + ["decrement_alpha"] * max(-da, 0)
            + ["increment_beta"] * max(db, 0) + ["decrement_beta"] * max(-db, 0))


def _apply_ops(ops, p: JacobiParameters, x, stream=None):
    """Run a shift chain on a CUDA batch, ping-ponging two buffers."""
    import torch
    if not ops:
        return x, p
    # temporaries recorded on `stream` (kernels run there, not on the current stream)
    bufs = [engine.empty_on_stream(x, stream), engine.empty_on_stream(x, stream)]
    cur = x
    for k, op in enumerate(ops):
        cur, p = shift_batched(op, p, cur, out=bufs[k % 2], stream=stream)
    return cur, p


def to_core_batched(p: JacobiParameters, x, stream=None):
    """Shift a (B, N+1) CUDA batch into the core square (engine.py:305-318)."""
    return _apply_ops(_to_core_ops(p), p, _cuda_2d(x), stream)


def from_core_batched(p: JacobiParameters, x, target: JacobiParameters, stream=None):
    """Shift core-square coefficients out to `target` (engine.py:321-338)."""
    y, q = _apply_ops(_from_core_ops(target), p, _cuda_2d(x), stream)
    if q != target:
        raise ParameterRangeError(f"shift chain reached {q}, expected {target}")
    return y


def to_core(c: CoefficientVector) -> CoefficientVector:
    """engine.py:305-318."""
    import torch
    _require_jacobi(c)
    ops = _to_core_ops(c.params)
    if not ops:
        return c
    dev = torch.device("cuda", engine._current_device())
    y, q = _apply_ops(ops, c.params, torch.from_numpy(c.data).to(dev).view(1, -1))
    return jacobi(q, y.view(-1).cpu().numpy())


def from_core(c: CoefficientVector, target: JacobiParameters) -> CoefficientVector:
    """engine.py:321-338."""
    import torch
    _require_jacobi(c)
    ops = _from_core_ops(target)
    if not ops:
        if c.params != target:
            raise ParameterRangeError(f"shift chain reached {c.params}, expected {target}")
        return c
    dev = torch.device("cuda", engine._current_device())
    y, q = _apply_ops(ops, c.params, torch.from_numpy(c.data).to(dev).view(1, -1))
    if q != target:
        raise ParameterRangeError(f"shift chain reached {q}, expected {target}")
    return jacobi(q, y.view(-1).cpu().numpy())


# plans are expensive; conversions between the same pairs reuse them
_PLAN_CACHE: "collections.OrderedDict" = collections.OrderedDict()
_PLAN_LOCK = threading.Lock()
_PLAN_CACHE_SIZE = 8


def _cached_plan(direction, p, n, m_terms, eps):
    key = (direction, p.alpha, p.beta, n, m_terms, eps)
    with _PLAN_LOCK:
        tp = _PLAN_CACHE.get(key)
        if tp is not None:
            _PLAN_CACHE.move_to_end(key)
            return tp
    tp = engine.plan(direction, p, n, m_terms, eps)
    with _PLAN_LOCK:
        _PLAN_CACHE[key] = tp
        while len(_PLAN_CACHE) > _PLAN_CACHE_SIZE:
            _PLAN_CACHE.popitem(last=False)
    return tp


def jacobi_to_jacobi_batched(p: JacobiParameters, x, target: JacobiParameters,
                             m_terms: int = DEFAULT_M, eps: float = DEFAULT_EPS, stream=None):
    """(B, N+1) CUDA batch in basis `p` -> basis `target` (engine.py:341-354):
    shifts into the core square, forward CJT, inverse CJT at the target's core
    pair, shifts out; all on the device."""
    x = _cuda_2d(x)
    n = x.shape[1] - 1
    core, cp = to_core_batched(p, x, stream)
    fwd = _cached_plan("forward", cp, n, m_terms, eps)
    raw = None if stream is None else _raw_stream(stream, x.device)
    cheb = engine.forward_batched(fwd, core, stream=raw)
    da, db = _core_offsets(target)
    core_target = JacobiParameters(target.alpha - da, target.beta - db)
    inv = _cached_plan("inverse", core_target, n, m_terms, eps)
    out = engine.inverse_batched(inv, cheb, stream=raw)
    return from_core_batched(core_target, out, target, stream)


def jacobi_to_jacobi(c: CoefficientVector, target: JacobiParameters,
                     m_terms: int = DEFAULT_M, eps: float = DEFAULT_EPS) -> CoefficientVector:
    """Convert between Jacobi expansions of differing parameters (engine.py:341-354)."""
    import torch
    _require_jacobi(c)
    dev = torch.device("cuda", engine._current_device())
    x = torch.from_numpy(np.ascontiguousarray(c.data)).to(dev).view(1, -1)
    y = jacobi_to_jacobi_batched(c.params, x, target, m_terms, eps)
    return jacobi(target, y.view(-1).cpu().numpy())
