"""Plan / execute API of the B200 Chebyshev-Jacobi transform.

Mirrors the reference's public engine API (chebjac/engine.py:36-227,
chebjac/__init__.py:12-31): ``plan``, ``forward``, ``inverse``, ``jacobi``,
``chebyshev``, ``CoefficientVector``, ``TransformPlan`` with the same argument
meaning and error behaviour (ValueError / ParameterRangeError), and adds the
batched entry points ``forward_batched`` / ``inverse_batched`` over (B, N+1)
float64 arrays or CUDA tensors.  All execution happens in libcjt_b200.so on
the GPU; a missing library or device raises instead of falling back.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import planner as pl
from .planner import DEFAULT_EPS, DEFAULT_M, JacobiParameters, ParameterRangeError
from .recurrences import AngleGrid

CHEBYSHEV = "cheb"
JACOBI = "jac"


@dataclass(frozen=True)
class CoefficientVector:
    """Expansion coefficients tagged with their basis (engine.py:36-62)."""

    basis: str
    data: np.ndarray
    params: JacobiParameters | None = None

    def __post_init__(self):
        data = np.ascontiguousarray(self.data, dtype=float)
        if data.ndim != 1 or data.size == 0:
            raise ValueError("coefficient data must be a nonempty 1-d vector")
        if not np.all(np.isfinite(data)):
            raise ValueError("coefficient data must be finite")
        object.__setattr__(self, "data", data)
        if self.basis == CHEBYSHEV:
            if self.params is not None:
                raise ValueError("Chebyshev coefficients carry no parameters")
        elif self.basis == JACOBI:
            if self.params is None:
                raise ValueError("Jacobi coefficients require parameters")
        else:
            raise ValueError(f"unknown basis {self.basis!r}")

    @property
    def n(self) -> int:
        return len(self.data) - 1


def chebyshev(data) -> CoefficientVector:
    return CoefficientVector(CHEBYSHEV, np.asarray(data, dtype=float))


def jacobi(p: JacobiParameters, data) -> CoefficientVector:
    return CoefficientVector(JACOBI, np.asarray(data, dtype=float), p)


class _DevicePlan:
    """One uploaded plan on one CUDA device (owns a cjt_plan*)."""

    def __init__(self, hp: pl.HostPlan):
        L = nat.lib()
        keep = []

        def arr(a, dtype=np.float64):
            a = np.ascontiguousarray(a, dtype=dtype)
            keep.append(a)
            return a.ctypes.data

        g1 = hp.grid_n + 1
        x = np.empty(g1)
        xm = np.empty(g1)
        regions = np.ascontiguousarray(hp.regions, dtype=np.int8)
        thetas = np.ascontiguousarray(hp.thetas, dtype=np.float64)
        nat.check(L.cjt_host_angles(thetas.ctypes.data, regions.ctypes.data, g1,
                                    x.ctypes.data, xm.ctypes.data), "cjt_host_angles")
        cuts = hp.device_cuts

        def cz_desc(cz: pl.ChirpZ) -> nat.ChirpZDesc:
            d = nat.ChirpZDesc()
            d.p0, d.width, d.q0, d.count, d.length = cz.p0, cz.width, cz.q0, cz.count, cz.length
            d.m_count = cz.m_count
            d.accumulate = 1 if cz.accumulate else 0
            d.n_tiles_in = len(cz.tiles_in)
            d.n_tiles_out = len(cz.tiles_out)
            d.tiles_in = arr(cz.tiles_in, np.int64)
            d.tiles_out = arr(cz.tiles_out, np.int64)
            d.out_shift = cz.out_shift
            if cz.device_tables:
                # bare diagonals; chirps, modulation and spectra built on the device
                d.device_tables = 1
                d.grid_g = cz.g
                for which, diag in (("pre", cz.pre_diag), ("post", cz.post_diag)):
                    if isinstance(diag, pl.Modulation):
                        setattr(d, which + "_kind", nat.CJT_DIAG_MODULATION)
                        setattr(d, which + "_row0", diag.row0)
                    else:
                        setattr(d, which, arr(np.atleast_2d(diag), np.complex128))
            else:
                d.pre = arr(cz.pre, np.complex128)
                d.post = arr(cz.post, np.complex128)
                d.kernel_hat = arr(cz.kernel_hat, np.complex128)
            return d

        desc = nat.PlanDesc()
        desc.direction = nat.CJT_FORWARD if hp.direction == "forward" else nat.CJT_INVERSE
        desc.m_terms = hp.m_terms
        desc.n = hp.n
        desc.grid_n = hp.grid_n
        desc.x = arr(x)
        desc.xm = arr(xm)
        desc.regions = arr(regions, np.int8)
        desc.cuts = arr(cuts, np.int64)
        t = hp.tables
        desc.table_len = len(t.A)
        desc.A, desc.B, desc.C = arr(t.A), arr(t.B), arr(t.C)
        desc.rf_plus, desc.rf_minus = arr(t.rf_plus), arr(t.rf_minus)
        desc.rf_plus_inv, desc.rf_minus_inv = arr(t.rf_plus_inv), arr(t.rf_minus_inv)
        blocks = (nat.ChirpZDesc * max(1, len(hp.blocks)))()
        for k, cz in enumerate(hp.blocks):
            blocks[k] = cz_desc(cz)
        desc.n_blocks = len(hp.blocks)
        desc.blocks = blocks
        edge = hp.analysis if hp.direction == "forward" else hp.synthesis
        if edge is not None:
            desc.edge = cz_desc(edge)
        desc.scalings = arr(hp.scalings) if hp.scalings is not None else None
        desc.half_k = arr(hp.half_k) if hp.half_k is not None else None
        desc.thetas = arr(thetas)
        desc.half_gemm = 1 if hp.half_gemm else 0
        desc.alpha, desc.beta = hp.p.alpha, hp.p.beta
        handle = ctypes.c_void_p()
        nat.check(L.cjt_plan_create(ctypes.byref(desc), ctypes.byref(handle)), "cjt_plan_create")
        self.handle = handle
        self.x = x
        self.xm = xm

    def reserve(self, batch: int):
        nat.check(nat.lib().cjt_plan_reserve(self.handle, int(batch)), "cjt_plan_reserve")

    def stats(self) -> nat.PlanStats:
        s = nat.PlanStats()
        nat.check(nat.lib().cjt_plan_stats_get(self.handle, ctypes.byref(s)), "cjt_plan_stats_get")
        return s

    def __del__(self):
        h = getattr(self, "handle", None)
        lib_ = getattr(nat, "_lib", None) if nat is not None else None   # None at interpreter exit
        if h is not None and h.value and lib_ is not None:
            try:
                lib_.cjt_plan_destroy(h)
            except Exception:
                pass


class TransformPlan:
    """Immutable precomputation for one transform direction and size
    (engine.py:73-93); device uploads are created per CUDA device on first use."""

    def __init__(self, hp: pl.HostPlan):
        self._hp = hp
        self.direction = hp.direction
        self.p = hp.p
        self.n = hp.n
        self.m_terms = hp.m_terms
        self.eps = hp.eps
        self.grid = AngleGrid(hp.grid_n, hp.thetas)
        self.layout = hp.layout
        self.tables = hp.tables
        self.cuts = hp.cuts
        self.regions = hp.regions
        self.weights = hp.weights
        self.scalings = hp.scalings
        self._dev = {}
        self._lock = threading.Lock()

    @property
    def grid_n(self) -> int:
        return self.grid.n

    @property
    def host(self) -> pl.HostPlan:
        return self._hp

    def device_plan(self, device: int | None = None) -> _DevicePlan:
        if device is None:
            device = _current_device()
        with self._lock:
            dp = self._dev.get(device)
            if dp is None:
                with _on_device(device):
                    dp = _DevicePlan(self._hp)
                self._dev[device] = dp
            return dp

    def __repr__(self):
        return (f"TransformPlan(direction={self.direction!r}, p={self.p}, n={self.n}, "
                f"m_terms={self.m_terms}, eps={self.eps})")


def _current_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except ImportError:
        pass
    return 0


class _on_device:
    def __init__(self, dev: int):
        self.dev = dev
        self.prev = None

    def __enter__(self):
        try:
            import torch
            if torch.cuda.is_available():
                self.prev = torch.cuda.current_device()
                torch.cuda.set_device(self.dev)
        except ImportError:
            pass

    def __exit__(self, *exc):
        if self.prev is not None:
            import torch
            torch.cuda.set_device(self.prev)


def plan(direction: str, p: JacobiParameters, n: int,
         m_terms: int = DEFAULT_M, eps: float = DEFAULT_EPS) -> TransformPlan:
    """Reusable plan for the forward (Jacobi -> Chebyshev) or inverse
    (Chebyshev -> Jacobi) transform of degree-N vectors (engine.py:96-130)."""
    return TransformPlan(pl.build(direction, p, n, m_terms, eps))


def _check_input(tp: TransformPlan, c: CoefficientVector, basis: str):
    if c.basis != basis:
        raise ValueError(f"plan expects {basis!r} input, got {c.basis!r}")
    if basis == JACOBI and c.params != tp.p:
        raise ValueError("coefficient parameters do not match the plan")
    if c.n != tp.n:
        raise ValueError(f"plan expects degree {tp.n}, got {c.n}")


def _run_host(tp: TransformPlan, data: np.ndarray) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.float64)
    batch = 1 if data.ndim == 1 else data.shape[0]
    out = np.empty_like(data)
    dp = tp.device_plan()
    nat.check(nat.lib().cjt_execute_host(dp.handle, data.ctypes.data, out.ctypes.data, batch, None),
              "cjt_execute_host")
    return out


def forward(tp: TransformPlan, c: CoefficientVector) -> CoefficientVector:
    """Jacobi -> Chebyshev coefficients of the same polynomial (engine.py:153-186)."""
    if tp.direction != "forward":
        raise ValueError("not a forward plan")
    _check_input(tp, c, JACOBI)
    return chebyshev(_run_host(tp, c.data))


def inverse(tp: TransformPlan, c: CoefficientVector) -> CoefficientVector:
    """Chebyshev -> Jacobi coefficients (engine.py:189-227)."""
    if tp.direction != "inverse":
        raise ValueError("not an inverse plan")
    _check_input(tp, c, CHEBYSHEV)
    return jacobi(tp.p, _run_host(tp, c.data))


def empty_on_stream(like, stream=None):
    """torch.empty_like(like) for use by kernels on `stream` (a torch stream or
    a raw cudaStream_t handle): when that is not the current stream, the block
    is recorded on it, so the caching allocator cannot hand it out again while
    work queued there may still touch it."""
    import torch
    out = torch.empty_like(like)
    if stream is not None:
        s = stream if isinstance(stream, torch.cuda.Stream) else torch.cuda.ExternalStream(
            int(stream), device=like.device)
        if s.cuda_stream != torch.cuda.current_stream(like.device).cuda_stream:
            out.record_stream(s)
    return out


def _execute_batched(tp: TransformPlan, data, out=None, check_finite: bool = True, stream=None):
    n1 = tp.n + 1
    if hasattr(data, "data_ptr"):  # torch tensor
        import torch
        if data.dtype != torch.float64:
            raise ValueError("batched input must be float64")
        if data.dim() != 2 or data.shape[1] != n1:
            raise ValueError(f"batched input must have shape (B, {n1}), got {tuple(data.shape)}")
        if data.shape[0] == 0:
            raise ValueError("batch must be nonempty")
        if not data.is_cuda:
            res = _execute_batched(tp, data.numpy(), None, check_finite)
            return torch.from_numpy(res)
        data = data.contiguous()
        if check_finite and not bool(torch.isfinite(data).all()):
            raise ValueError("coefficient data must be finite")
        dev = data.device.index
        if out is None:
            out = empty_on_stream(data, stream)
        elif out.shape != data.shape or out.dtype != torch.float64 or not out.is_contiguous():
            raise ValueError("out must be a contiguous float64 tensor shaped like the input")
        dp = tp.device_plan(dev)
        st = stream if stream is not None else torch.cuda.current_stream(data.device).cuda_stream
        with torch.cuda.device(dev):
            nat.check(nat.lib().cjt_execute(dp.handle, data.data_ptr(), out.data_ptr(),
                                            data.shape[0], st), "cjt_execute")
        return out
    arr = np.ascontiguousarray(data, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[1] != n1 or arr.shape[0] == 0:
        raise ValueError(f"batched input must have shape (B, {n1}), got {arr.shape}")
    if check_finite and not np.all(np.isfinite(arr)):
        raise ValueError("coefficient data must be finite")
    return _run_host(tp, arr)


def forward_batched(tp: TransformPlan, c, out=None, check_finite: bool = True, stream=None):
    """Forward transform of a (B, N+1) batch of Jacobi coefficient vectors.
    CUDA tensors stay on the device (stream-ordered, no host sync); NumPy arrays
    are copied in and out."""
    if tp.direction != "forward":
        raise ValueError("not a forward plan")
    return _execute_batched(tp, c, out, check_finite, stream)


def inverse_batched(tp: TransformPlan, c, out=None, check_finite: bool = True, stream=None):
    """Inverse transform of a (B, N+1) batch of Chebyshev coefficient vectors."""
    if tp.direction != "inverse":
        raise ValueError("not an inverse plan")
    return _execute_batched(tp, c, out, check_finite, stream)


_PIPE_CACHE: dict = {}


_PIPE_NEXT = {}


def pipeline(plans, host_in, host_out=None, chunk: int | None = None, streams: int = 2,
             device: int | None = None, sync: bool = True):
    """Apply `plans` in sequence (e.g. ``(forward_plan, inverse_plan)``) to a
    (B, N+1) float64 host array, with host<->device copies overlapped with the
    transforms: the batch is cut into chunks that flow through a
    host->device copy stream, two transform streams (alternating chunks) and
    a device->host copy stream over a ring of `streams` device buffer slots,
    linked by events, so the two copy directions and the transforms proceed
    independently (chunk k+1 arrives and chunk k-1 leaves while chunk k is
    transformed; compute-bound batches overlap the transforms of consecutive
    chunks -- two at a time, more only contend: config 2 5.5e8 coeffs/s with
    two, 4.7e8 with three).  Pinned host memory (e.g.
    ``torch.empty(..., pin_memory=True)``) is required for the copies to be
    asynchronous.  Returns host_out.

    ``sync=False`` returns as soon as the work is enqueued (host_out is valid
    after ``torch.cuda.synchronize()``); consecutive calls continue the slot
    rotation, so one call's copies overlap the neighbouring calls' transforms
    (streaming many batches through the GPU).  The caller must not modify
    host_in / read host_out of a call before synchronizing."""
    import torch
    if not plans:
        raise ValueError("no plans")
    n1 = plans[0].n + 1
    for i, tp in enumerate(plans):
        if tp.n + 1 != n1:
            raise ValueError("plans must share the degree N")
        if i and plans[i - 1].direction == tp.direction:
            raise ValueError("consecutive plans must alternate direction")
    hin = host_in if hasattr(host_in, "data_ptr") else torch.from_numpy(np.ascontiguousarray(host_in))
    if hin.dtype != torch.float64 or hin.dim() != 2 or hin.shape[1] != n1:
        raise ValueError(f"host input must be float64 with shape (B, {n1})")
    if host_out is None:
        host_out = torch.empty_like(hin, pin_memory=True)
    hout = host_out if hasattr(host_out, "data_ptr") else torch.from_numpy(host_out)
    batch = hin.shape[0]
    chunk = batch if chunk is None else max(1, min(int(chunk), batch))
    dev = torch.device("cuda", _current_device() if device is None else device)
    nslots = max(1, int(streams))
    # streams, events and device buffers are cached: plan workspaces are per
    # (compute) stream, so fresh streams would re-allocate them on every call
    key = (dev.index, nslots, chunk, n1)
    cached = _PIPE_CACHE.get(key)
    if cached is None:
        h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        comp = [torch.cuda.Stream(dev) for _ in range(min(nslots, 2))]
        bufs = [(torch.empty((chunk, n1), dtype=torch.float64, device=dev),
                 torch.empty((chunk, n1), dtype=torch.float64, device=dev)) for _ in range(nslots)]
        ev_in = [torch.cuda.Event() for _ in range(nslots)]     # slot filled
        ev_done = [torch.cuda.Event() for _ in range(nslots)]   # slot transformed
        ev_free = [torch.cuda.Event() for _ in range(nslots)]   # slot's result copied out
        cached = _PIPE_CACHE[key] = (h2d, comp, d2h, bufs, ev_in, ev_done, ev_free)
    h2d, comp, d2h, bufs, ev_in, ev_done, ev_free = cached
    cur = torch.cuda.current_stream(dev)
    for s in (h2d, d2h, *comp):
        s.wait_stream(cur)
    k0 = _PIPE_NEXT.get(key, 0) if not sync else 0
    for k, r0 in enumerate(range(0, batch, chunk), start=k0):
        r1 = min(batch, r0 + chunk)
        slot = k % nslots
        a, b = bufs[slot]
        h2d.wait_event(ev_free[slot])          # the slot's previous chunk has left (no-op if unused)
        with torch.cuda.stream(h2d):
            a[: r1 - r0].copy_(hin[r0:r1], non_blocking=True)
            ev_in[slot].record(h2d)
        cs = comp[k % len(comp)]
        cs.wait_event(ev_in[slot])
        src, dst = a[: r1 - r0], b[: r1 - r0]
        with torch.cuda.stream(cs):
            for tp in plans:
                _execute_batched(tp, src, out=dst, check_finite=False)
                src, dst = dst, src
            ev_done[slot].record(cs)
        d2h.wait_event(ev_done[slot])
        with torch.cuda.stream(d2h):
            hout[r0:r1].copy_(src, non_blocking=True)
            ev_free[slot].record(d2h)
    if not sync:
        _PIPE_NEXT[key] = (k0 + -(-batch // chunk)) % nslots
        return host_out
    cur.wait_stream(d2h)
    torch.cuda.synchronize(dev)
    return host_out
