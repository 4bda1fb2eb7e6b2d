"""DCT-I / bordered DST-I and the Chebyshev synthesis / analysis maps, on the GPU.

Mirrors the reference module ``chebjac.trig`` (trig.py:1-70): the kernel
convention is unnormalized and unhalved,

    dct1:  y_j = sum_{k=0}^{N} cos(pi j k / N) x_k
    dst1:  y_j = sum_{k=0}^{N} sin(pi j k / N) x_k   (rows 0, N exactly zero)

``TrigPlanWorkspace(n)`` keeps the reference's methods (dct1, dst1_bordered,
chebyshev_synthesis, chebyshev_analysis, clone) and length checks; the
module-level functions take the workspace first, as in the reference.  Each
transform is one batched chirp-z product (the same Bluestein kernels as the
transform blocks, planner.chirpz with M = 1) behind cjt_chirpz_create /
cjt_chirpz_execute; ``*_batched`` variants take (B, N+1) CUDA tensors.
The reference calls scipy.fft; results agree to rounding (test_trig.py's
dense-equivalence bound, 1e-13).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native as nat
from . import planner as pl

__all__ = ["TrigPlanWorkspace", "dct1", "dst1_bordered", "chebyshev_synthesis", "chebyshev_analysis",
           "trig_batched"]

KINDS = ("dct1", "dst1_bordered", "chebyshev_synthesis", "chebyshev_analysis")


def _scalings(kind: str, n: int):
    """pre / post diagonals of z_q = sum_p e^{i pi p q / N} pre_p x_p,
    y_q = Re(post_q z_q)."""
    pre = np.ones(n + 1)
    post = np.ones(n + 1, dtype=np.complex128)
    if kind == "dst1_bordered":
        pre[0] = pre[-1] = 0.0         # the reference transforms x[1:-1] only (trig.py:42-47)
        post[:] = -1j                  # Re(-i z) = Im(z) = the sine sum
        post[0] = post[-1] = 0.0       # rows 0 and N exactly zero
    elif kind == "chebyshev_analysis":
        pre[0] = pre[-1] = 0.5         # trig.py:53-63: dct(0.5 v), then 2/N, ends halved
        post[:] = 2.0 / n
        post[0] *= 0.5
        post[-1] *= 0.5
    return pre, post


class _DeviceChirpZ:
    """One uploaded chirp-z product on one device (owns a cjt_chirpz_plan*)."""

    def __init__(self, kind: str, n: int):
        pre, post = _scalings(kind, n)
        cz = pl.chirpz(n, 0, n + 1, 0, n + 1, pre[None, :], post[None, :], accumulate=False)
        keep = []

        def arr(a, dtype):
            a = np.ascontiguousarray(a, dtype=dtype)
            keep.append(a)
            return a.ctypes.data

        d = nat.ChirpZDesc()
        d.p0, d.width, d.q0, d.count, d.length = cz.p0, cz.width, cz.q0, cz.count, cz.length
        d.m_count = cz.m_count
        d.accumulate = 0
        d.pre = arr(cz.pre, np.complex128)
        d.post = arr(cz.post, np.complex128)
        d.n_tiles_in = len(cz.tiles_in)
        d.n_tiles_out = len(cz.tiles_out)
        d.tiles_in = arr(cz.tiles_in, np.int64)
        d.tiles_out = arr(cz.tiles_out, np.int64)
        d.kernel_hat = arr(cz.kernel_hat, np.complex128)
        h = ctypes.c_void_p()
        nat.check(nat.lib().cjt_chirpz_create(ctypes.byref(d), ctypes.byref(h)), "cjt_chirpz_create")
        self.handle = h
        self.n = n

    def run(self, x, out, stream):
        batch = x.shape[0]
        done = 0
        while done < batch:   # the combine grid caps one call at 65535 vectors
            nb = min(65535, batch - done)
            nat.check(nat.lib().cjt_chirpz_execute(self.handle, x[done].data_ptr(), self.n + 1,
                                                   out[done].data_ptr(), self.n + 1, nb,
                                                   stream.cuda_stream), "cjt_chirpz_execute")
            done += nb

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and nat._lib is not None:
            try:
                nat._lib.cjt_chirpz_destroy(h)
            except Exception:
                pass


_CACHE: dict = {}
_LOCK = threading.Lock()


def _device_plan(kind: str, n: int, device: int) -> _DeviceChirpZ:
    import torch
    key = (kind, n, device)
    with _LOCK:
        dp = _CACHE.get(key)
        if dp is None:
            if len(_CACHE) >= 32:
                _CACHE.pop(next(iter(_CACHE)))
            with torch.cuda.device(device):
                dp = _CACHE[key] = _DeviceChirpZ(kind, n)
        return dp


def trig_batched(kind: str, x, out=None, stream=None):
    """Batched trig transform ``kind`` (one of KINDS) of a (B, N+1) float64
    CUDA tensor (or NumPy array -> NumPy result); stream ordered."""
    import torch
    if kind not in KINDS:
        raise ValueError(f"unknown transform {kind!r}; one of {KINDS}")
    host = isinstance(x, np.ndarray)
    if host:
        if not torch.cuda.is_available():
            raise RuntimeError("trig transforms need a CUDA device (no CPU fallback)")
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    else:
        t = x
        if not t.is_cuda or t.dtype != torch.float64:
            raise ValueError("x must be a float64 CUDA tensor or a NumPy array")
    if t.dim() != 2 or t.shape[1] < 2:
        raise ValueError("x must be (batch, N+1) with N >= 1")
    t = t.contiguous()
    n = t.shape[1] - 1
    if out is None:
        out = torch.empty_like(t)
    elif tuple(out.shape) != tuple(t.shape) or out.dtype != torch.float64 or not out.is_contiguous():
        raise ValueError("out must be a contiguous float64 tensor shaped like x")
    if t.shape[0] == 0:
        return out.cpu().numpy() if host else out
    st = stream if stream is not None else torch.cuda.current_stream(t.device)
    _device_plan(kind, n, t.device.index).run(t, out, st)
    if host:
        return out.cpu().numpy()
    return out


class TrigPlanWorkspace:
    """Size-(N+1) trigonometric transforms (trig.py:15-63); the device plans
    are shared and per-stream workspaces make concurrent use safe, so
    ``clone()`` is cheap as in the reference."""

    def __init__(self, n: int):
        if n < 1:
            raise ValueError("grid parameter N must be >= 1")
        self.n = n

    def clone(self) -> "TrigPlanWorkspace":
        return TrigPlanWorkspace(self.n)

    def _check(self, x):
        if len(x) != self.n + 1:
            raise ValueError(f"expected length {self.n + 1}, got {len(x)}")

    def _run(self, kind, x):
        x = np.asarray(x, dtype=np.float64)
        self._check(x)
        return trig_batched(kind, x[None, :])[0]

    def dct1(self, x: np.ndarray) -> np.ndarray:
        return self._run("dct1", x)

    def dst1_bordered(self, x: np.ndarray) -> np.ndarray:
        return self._run("dst1_bordered", x)

    def chebyshev_synthesis(self, c: np.ndarray) -> np.ndarray:
        """Values sum_n c_n T_n at the Chebyshev-Lobatto points cos(pi j / N)."""
        return self._run("chebyshev_synthesis", c)

    def chebyshev_analysis(self, v: np.ndarray) -> np.ndarray:
        """Chebyshev coefficients from Lobatto-point values (exact inverse)."""
        return self._run("chebyshev_analysis", v)


def dct1(w: TrigPlanWorkspace, x: np.ndarray) -> np.ndarray:
    return w.dct1(x)


def dst1_bordered(w: TrigPlanWorkspace, x: np.ndarray) -> np.ndarray:
    return w.dst1_bordered(x)


def chebyshev_synthesis(w: TrigPlanWorkspace, c: np.ndarray) -> np.ndarray:
    return w.chebyshev_synthesis(c)


def chebyshev_analysis(w: TrigPlanWorkspace, v: np.ndarray) -> np.ndarray:
    return w.chebyshev_analysis(v)
