"""Host-side planning for the B200 Chebyshev-Jacobi transform.

Everything here runs once per plan on the host and produces the read-only
tables the device executes against.  The numerics follow the reference
package ``chebjac`` operation-for-operation wherever the device result depends
on the exact bits (grid angles, region codes, partition, recurrence tables,
asymptotic coefficients, modulation functions, quadrature weights,
orthonormality constants), so a plan built here describes exactly the
reference's transform:

  * angle grid           chebjac/recurrences.py:48-66
  * region classifier    chebjac/recurrences.py:24-45
  * Stirling factors     chebjac/kernels.py:20-106
  * recurrence tables    chebjac/kernels.py:336-364
  * C_{n,m}              chebjac/kernels.py:186-252
  * 1/A_n                chebjac/kernels.py:255-307
  * modulation u_m, v_m  chebjac/asymptotics.py:22-75
  * envelope g_m, n_M    chebjac/asymptotics.py:86-138
  * partition            chebjac/asymptotics.py:147-255
  * moments, CC weights  chebjac/quadrature.py:35-78

On top of that the planner lays every trigonometric transform of the
reference execution (engine.py:163-227, trig.py:35-63) out as a *chirp-z*
problem with power-of-two cyclic length: for input indices p in [p0, p0+W)
and output indices q in [q0, q0+R),

    z_q = sum_p x_p exp(i pi p q / G)
        = chirp(q) * sum_p (x_p chirp(p)) * conj(chirp(q - p)),
    chirp(k) = exp(i pi k^2 / (2G)),

so every DCT-I / bordered DST-I of the reference becomes one real part of a
Bluestein convolution whose diagonal scalings (C_{n,m}, u_m - i v_m, the
Clenshaw-Curtis weights, the analysis 2/G) are folded into per-plan complex
pre/post tables.  G = 2^k - 1 and 2G = 2(2^k - 1) have large prime factors
(8191 is prime), so the power-of-two Bluestein length keeps one FFT code path
for every configuration.
"""

from __future__ import annotations

import dataclasses
import math
import threading
from dataclasses import dataclass, field

import functools

import numpy as np
import scipy.fft

DEFAULT_M = 7
DEFAULT_EPS = float(np.finfo(np.float64).eps)

# region codes (chebjac/recurrences.py:27-29)
INTERIOR = 0
NEAR_PLUS_ONE = 1
NEAR_MINUS_ONE = -1
BREAK_LO = 0.25 * math.pi
BREAK_HI = 0.75 * math.pi


class ParameterRangeError(ValueError):
    """(alpha, beta) outside the range an operation supports
    (chebjac/parameters.py:6)."""


@dataclass(frozen=True)
class JacobiParameters:
    """Weight exponents (alpha, beta); alpha, beta > -1 (parameters.py:11-44)."""

    alpha: float
    beta: float

    def __post_init__(self):
        if not (self.alpha > -1.0 and self.beta > -1.0):
            raise ParameterRangeError(
                f"Jacobi parameters require alpha, beta > -1, got ({self.alpha}, {self.beta})")

    @property
    def core(self) -> bool:
        return (-0.5 < self.alpha <= 0.5) and (-0.5 < self.beta <= 0.5)

    def swapped(self) -> "JacobiParameters":
        return JacobiParameters(self.beta, self.alpha)

    def require_core(self, context: str = "this operation"):
        if not self.core:
            raise ParameterRangeError(
                f"{context} requires (alpha, beta) in (-1/2, 1/2]^2, got "
                f"({self.alpha}, {self.beta}); reduce the parameters with "
                f"integer increments/decrements first")


# ---------------------------------------------------------------------------
# Stirling series (kernels.py:20-106).  Coefficients are exact rationals of the
# classical numerator/denominator sequences, rounded once.
_STIRLING_NUM_DEN = (
    (1, 1), (1, 12), (1, 288), (-139, 51840), (-571, 2488320),
    (163879, 209018880), (5246819, 75246796800), (-534703531, 902961561600),
    (-4483131259, 86684309913600), (432261921612371, 514904800886784000),
    (6232523202521089, 86504006548979712000),
    (-25834629665134204969, 13494625021640835072000),
    (-1579029138854919086429, 9716130015581401251840000),
    (746590869962651602203151, 116593560186976815022080000),
    (1511513601028097903631961, 2798245444487443560529920000),
    (-8849272268392873147705987190261, 299692087104605205332754432000000),
    (-142801712490607530608130701097701, 57540880724084199423888850944000000),
)
STIRLING = tuple(num / den for num, den in _STIRLING_NUM_DEN)
# smallest z for which k terms reach eps/20 (kernels.py:46-61), ascending in z
_STIRLING_CUTS = np.array([9.0, 10.0, 11.0, 12.0, 14.0, 17.0, 20.0, 26.0, 35.0, 53.0,
                           92.0, 196.0, 591.0, 3275.0])
_STIRLING_TERMS = np.array([17, 16, 15, 14, 13, 12, 11, 10, 9, 8, 7, 6, 5, 4], dtype=np.int64)


def stirling_series(z):
    """S(z) = Gamma(z) e^z z^(1/2-z) / sqrt(2 pi), truncated per argument."""
    z = np.asarray(z, dtype=float)
    if np.any(z < 9.0):
        raise ValueError("Stirling series requires z >= 9")
    idx = np.searchsorted(_STIRLING_CUTS, z, side="right") - 1
    res = np.empty_like(z)
    if z.ndim == 1 and z.size > 1 and np.all(z[1:] >= z[:-1]):
        # ascending arguments (the planner's degree ranges): contiguous runs of
        # equal term counts, no masks
        bounds = np.flatnonzero(np.diff(idx)) + 1
        runs = zip(np.concatenate([[0], bounds]), np.concatenate([bounds, [z.size]]))
        groups = [(int(_STIRLING_TERMS[idx[a]]), slice(int(a), int(b))) for a, b in runs]
    else:
        terms = _STIRLING_TERMS[idx]
        groups = [(int(k), terms == k) for k in np.unique(terms)]
    for k, pick in groups:
        zz = z[pick]
        horner = np.zeros_like(zz)
        for j in range(k - 1, 0, -1):
            horner = (horner + STIRLING[j]) / zz
        res[pick] = horner + 1.0
    return res


def _pow1p(x, y):
    # (1+x)^y as exp(y log1p x) (kernels.py:118-119)
    return np.exp(y * np.log1p(x))


# ---------------------------------------------------------------------------
# C_{n,m} (kernels.py:186-252)

def _cnm_switch(a: float, b: float) -> int:
    lo = min(a, b)
    return 8 + math.ceil(abs(lo)) if lo != 0.0 else 8


def _cnm_stirling(a, b, n, m):
    """Closed Stirling form of C_{n,m}; n scalar or array."""
    d = 2.0 * n + (a + b) + m + 2.0
    lead = math.exp(m) / (4.0**m * math.sqrt(math.pi))
    f1 = _pow1p((a - b - m) / d, n + a + 0.5)
    f2 = _pow1p((b - a - m) / d, n + b + 0.5)
    den = np.power(np.asarray(n, dtype=float), m + 0.5) * _pow1p(
        ((a + b) + m + 2.0) / (2.0 * n), m + 0.5)
    ratio = (stirling_series(n + a + 1.0) * stirling_series(n + b + 1.0)
             / stirling_series(2.0 * n + m + (a + b) + 2.0))
    return lead * f1 * f2 / den * ratio


def cnm_scalar(p: JacobiParameters, n: int, m: int) -> float:
    """C_{n,m} at one degree (kernels.py:210-228)."""
    if n < 0 or m < 0:
        raise ValueError("n and m must be nonnegative")
    a, b = p.alpha, p.beta
    if n + min(a, b) >= 8.0:
        return float(_cnm_stirling(a, b, n, m))
    n0 = _cnm_switch(a, b)
    val = float(_cnm_stirling(a, b, n0, m))
    s = a + b
    for k in range(n0, n, -1):
        val *= (k + (s + m + 1) / 2) * (k + (s + m) / 2) / ((k + a) * (k + b))
    return val


def _cnm_table(p: JacobiParameters, nmax: int, m_count: int) -> np.ndarray:
    """C_{n,m}, n = 0..nmax, m < m_count, shape (nmax+1, m_count)
    (kernels.py:231-252)."""
    a, b = p.alpha, p.beta
    s = a + b
    n0 = min(_cnm_switch(a, b), nmax)
    col = np.empty(nmax + 1)
    if n0 < nmax or n0 + min(a, b) >= 8.0:
        col[n0:] = _cnm_stirling(a, b, np.arange(n0, nmax + 1, dtype=float), 0)
    else:
        col[n0] = cnm_scalar(p, n0, 0)
    for k in range(n0, 0, -1):
        col[k - 1] = col[k] * (k + (s + 1) / 2) * (k + s / 2) / ((k + a) * (k + b))
    out = np.empty((nmax + 1, m_count))
    out[:, 0] = col
    deg = np.arange(nmax + 1, dtype=float)
    for m in range(1, m_count):
        out[:, m] = out[:, m - 1] / (2.0 * (2.0 * deg + s + m + 1.0))
    return out


# ---------------------------------------------------------------------------
# A_n (kernels.py:255-307)

def _an_direct(a, b, n):
    g = math.gamma(n + a + 1.0) * math.gamma(n + b + 1.0)
    return (2.0 ** ((a + b) + 1.0) * g
            / ((2.0 * n + (a + b) + 1.0) * math.gamma(n + (a + b) + 1.0) * math.gamma(n + 1.0)))


def _an_stirling(a, b, n):
    n = np.asarray(n, dtype=float)
    front = 2.0 ** ((a + b) + 1.0) / (2.0 * n + (a + b) + 1.0)
    g1 = _pow1p(-b / (n + (a + b) + 1.0), n / 2 + a + 0.25) * _pow1p(
        -a / (n + (a + b) + 1.0), n / 2 + b + 0.25)
    g2 = _pow1p(a / (n + 1.0), n / 2 + 0.25) * _pow1p(b / (n + 1.0), n / 2 + 0.25)
    rat = (stirling_series(n + a + 1.0) * stirling_series(n + b + 1.0)
           / (stirling_series(n + (a + b) + 1.0) * stirling_series(n + 1.0)))
    return front * g1 * g2 * rat


def _orthonormality(p: JacobiParameters, nmax: int) -> np.ndarray:
    """A_n = ||P_n||^2 for n = 0..nmax (kernels.py:298-307)."""
    a, b = p.alpha, p.beta
    lo = min(a, b, a + b, 0.0)
    switch = 8 + math.ceil(-lo) if lo < 0.0 else 8
    n0 = min(switch, nmax + 1)
    out = np.empty(nmax + 1)
    for n in range(n0):
        out[n] = _an_direct(a, b, n)
    if n0 <= nmax:
        out[n0:] = _an_stirling(a, b, np.arange(n0, nmax + 1))
    return out


# ---------------------------------------------------------------------------
# Recurrence tables (kernels.py:336-364)

@dataclass(frozen=True)
class RecurrenceTables:
    A: np.ndarray
    B: np.ndarray
    C: np.ndarray
    rf_plus: np.ndarray
    rf_minus: np.ndarray
    rb_plus: np.ndarray
    rb_minus: np.ndarray
    rf_plus_inv: np.ndarray
    rf_minus_inv: np.ndarray
    rb_plus_inv: np.ndarray
    rb_minus_inv: np.ndarray


def _recurrence_tables(p: JacobiParameters, nmax: int) -> RecurrenceTables:
    a, b = p.alpha, p.beta
    s = a + b
    deg = np.arange(nmax + 1, dtype=float)
    t = 2.0 * deg + s
    den = 2.0 * (deg + 1.0) * (deg + s + 1.0)
    A = (t + 1.0) * (t + 2.0) / den
    with np.errstate(divide="ignore", invalid="ignore"):
        B = (a - b) * (a + b) * (t + 1.0) / (den * t)
        C = 2.0 * (deg + a) * (deg + b) * (t + 2.0) / (den * t)
    A[0] = s / 2 + 1.0
    B[0] = (a - b) / 2
    C[0] = 0.0
    rfp = (deg + a + 1.0) / (deg + 1.0)
    rfm = -(deg + b + 1.0) / (deg + 1.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        core = (deg + 1.0) * (s + deg + 1.0) * (s + 2.0 * deg) / (deg * (s + 2.0 * deg + 2.0))
        rbp = core / (deg + b)
        rbm = -core / (deg + a)
    rbp[0] = rbm[0] = np.nan
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = [1.0 / v for v in (rfp, rfm, rbp, rbm)]
    arrays = (A, B, C, rfp, rfm, rbp, rbm, *inv)
    for arr in arrays:
        arr.flags.writeable = False
    return RecurrenceTables(*arrays)


# ---------------------------------------------------------------------------
# Per-(alpha, beta) prefix caches.  Every entry of these tables is a function
# of its degree alone (elementwise formulas; the downward recursions stop at
# the Stirling switch degree, below any length the planner asks for), so a
# shorter table is bit-for-bit the prefix of a longer one (checked for the
# configuration-5 parameter set in tests/test_planner.py).  Ragged batches
# (configuration 5: 25 parameter pairs x 9 degrees x 2 directions) then build
# each table once per pair.

_PREFIX_CACHE: dict = {}
_PREFIX_LOCK = threading.Lock()
_PREFIX_MIN = 64            # below this the tables are cheap: no caching


def _prefix(kind: str, p: JacobiParameters, n: int, extra, build):
    if n + 1 < _PREFIX_MIN:
        return n, build(n)
    key = (kind, p.alpha, p.beta, extra)
    with _PREFIX_LOCK:
        hit = _PREFIX_CACHE.get(key)
    if hit is None or hit[0] < n:
        val = build(n)
        if isinstance(val, np.ndarray):
            val.flags.writeable = False
        hit = (n, val)
        with _PREFIX_LOCK:
            cur = _PREFIX_CACHE.get(key)
            if cur is None or cur[0] < n:
                _PREFIX_CACHE[key] = hit
    return hit


def cnm_table(p: JacobiParameters, nmax: int, m_count: int) -> np.ndarray:
    """C_{n,m}, n = 0..nmax, m < m_count, shape (nmax+1, m_count)
    (kernels.py:231-252); prefix-cached per (alpha, beta, M)."""
    if nmax < _cnm_switch(p.alpha, p.beta):
        return _cnm_table(p, nmax, m_count)
    top, tab = _prefix("cnm", p, nmax, m_count, lambda n: _cnm_table(p, n, m_count))
    return tab if top == nmax else tab[: nmax + 1]


def orthonormality(p: JacobiParameters, nmax: int) -> np.ndarray:
    """A_n = ||P_n||^2 for n = 0..nmax (kernels.py:298-307); prefix-cached."""
    top, tab = _prefix("an", p, nmax, None, lambda n: _orthonormality(p, n))
    return tab if top == nmax else tab[: nmax + 1]


def recurrence_tables(p: JacobiParameters, nmax: int) -> RecurrenceTables:
    """Three-term and Reinsch tables for degrees 0..nmax (kernels.py:336-364);
    prefix-cached per (alpha, beta)."""
    top, t = _prefix("rec", p, nmax, None, lambda n: _recurrence_tables(p, n))
    if top == nmax:
        return t
    return RecurrenceTables(*(getattr(t, f.name)[: nmax + 1] for f in dataclasses.fields(t)))


def prewarm(p: JacobiParameters, n_max: int, m_terms: int = 7) -> None:
    """Build the prefix-cached tables of `p` once at the largest size plans of
    degree <= n_max ask for (forward and inverse), so those plans slice them
    (ragged batches: one build per parameter pair instead of one per plan)."""
    g = 2 * n_max
    recurrence_tables(p, g + 1)
    orthonormality(p, n_max)
    cnm_table(p, min(g, max(n_max, _cnm_switch(p.alpha, p.beta))), m_terms)


# ---------------------------------------------------------------------------
# Grid and regions (recurrences.py:41-66)

def angle_grid(g: int) -> np.ndarray:
    if g < 1:
        raise ValueError("grid parameter N must be >= 1")
    th = np.pi * np.arange(g + 1) / g
    th.flags.writeable = False
    return th


def region_codes(thetas: np.ndarray) -> np.ndarray:
    reg = np.zeros(len(thetas), dtype=np.int8)
    reg[thetas < BREAK_LO] = NEAR_PLUS_ONE
    reg[thetas > BREAK_HI] = NEAR_MINUS_ONE
    return reg


# ---------------------------------------------------------------------------
# Modulation / envelope (asymptotics.py:22-138)

def _pair_weights(gamma: float, count: int) -> np.ndarray:
    w = np.empty(count)
    w[0] = 1.0
    for l in range(1, count):
        w[l] = w[l - 1] * (0.5 + gamma + l - 1) * (0.5 - gamma + l - 1) / l
    return w


def modulation(p: JacobiParameters, m_count: int, thetas: np.ndarray):
    """u_m(theta), v_m(theta), shape (m_count, len(thetas))
    (asymptotics.py:36-75)."""
    a, b = p.alpha, p.beta
    thetas = np.asarray(thetas, dtype=float)
    sh = np.sin(0.5 * thetas)
    ch = np.cos(0.5 * thetas)
    wa = _pair_weights(a, m_count)
    wb = _pair_weights(b, m_count)
    phase = (a + b + 1.0) * 0.5 * thetas - (a + 0.5) * 0.5 * math.pi
    re = np.cos(phase)
    im = np.sin(phase)
    u = np.empty((m_count, len(thetas)))
    v = np.empty((m_count, len(thetas)))
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        scale0 = 1.0 / (sh ** (a + 0.5) * ch ** (b + 0.5))
        for m in range(m_count):
            cr, ci = re.copy(), im.copy()
            scale = scale0 * ch ** (-float(m))
            um = np.zeros(len(thetas))
            vm = np.zeros(len(thetas))
            for l in range(m + 1):
                rho = wa[l] * wb[m - l]
                if rho != 0.0:
                    um += rho * cr * scale
                    vm -= rho * ci * scale
                if l < m:
                    cr, ci = ci, -cr
                    scale = scale * ch / sh
            u[m] = um
            v[m] = vm
            re, im = re * ch - im * sh, re * sh + im * ch
    return u, v


def envelope(p: JacobiParameters, m: int, thetas: np.ndarray) -> np.ndarray:
    """g_m over angles (asymptotics.py:86-103)."""
    a, b = p.alpha, p.beta
    thetas = np.asarray(thetas, dtype=float)
    sh = np.sin(0.5 * thetas)
    ch = np.cos(0.5 * thetas)
    wa = _pair_weights(a, m + 1)
    wb = _pair_weights(b, m + 1)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        scale = 1.0 / (sh ** (a + 0.5) * ch ** (float(m) + b + 0.5))
        g = np.zeros(len(thetas))
        for l in range(m + 1):
            w = wa[l] * wb[m - l]
            if w != 0.0:
                g += w * scale
            if l < m:
                scale = scale * ch / sh
    return g


def _degree_from_bound(g: float, m_terms: int, eps: float) -> int:
    if g == 0.0:
        return 0
    val = (eps * 2.0 ** (2 * m_terms - 1) * math.sqrt(math.pi) / g) ** (-1.0 / (m_terms + 0.5))
    return int(math.floor(val))


def n_m(p: JacobiParameters, m_terms: int, eps: float) -> int:
    """asymptotics.py:131-138"""
    if m_terms < 2:
        raise ValueError("M >= 2 required")
    if eps <= 0:
        raise ValueError("eps must be positive")
    g = float(envelope(p, m_terms, np.array([0.5 * math.pi]))[0])
    return _degree_from_bound(g, m_terms, eps)


@dataclass(frozen=True)
class Block:
    j: int
    i1: int
    i2: int


@dataclass(frozen=True)
class Partition:
    """Certified rectangles (asymptotics.py:156-200)."""

    n: int
    m_terms: int
    eps: float
    n_m: int
    alpha_n: float
    k: int
    blocks: tuple
    theta_bar_index: int

    def column_strips(self):
        out, top = [], self.n
        for blk in self.blocks:
            out.append((blk.j, top))
            top = blk.j - 1
        return out

    def row_cuts(self) -> np.ndarray:
        cuts = np.full(self.n + 1, self.n + 1, dtype=np.int64)
        for blk in self.blocks:
            cuts[blk.i1: blk.i2 + 1] = blk.j
        return cuts


def partition(p: JacobiParameters, g: int, m_terms: int, eps: float,
              thetas: np.ndarray | None = None) -> Partition:
    """asymptotics.py:203-255"""
    p.require_core("partition construction")
    if m_terms < 2:
        raise ValueError("M >= 2 required")
    if thetas is None:
        thetas = angle_grid(g)
    nm = n_m(p, m_terms, eps)
    env = envelope(p, m_terms, thetas)
    tbar = int(np.argmin(env))
    if g <= nm:
        return Partition(g, m_terms, eps, nm, 0.5, 0, (), tbar)
    ratio = math.log(g / max(nm, 1))
    alpha_n = min(1.0 / ratio, 0.5) if ratio > 0 else 0.5
    blocks = []
    lo_prev, hi_prev = 1, g - 1
    k = 1
    while True:
        jk = int(math.floor(alpha_n ** k * g))
        if jk <= nm or jk < 2:
            break
        bad = ~(2.0 * cnm_scalar(p, jk, m_terms) * env < eps)
        if bad[tbar]:
            break
        left = bad[1:tbar][::-1]
        i1 = tbar - (int(np.argmax(left)) if left.any() else left.size)
        right = bad[tbar + 1: g]
        i2 = tbar + (int(np.argmax(right)) if right.any() else right.size)
        i1 = max(i1, lo_prev)
        i2 = min(i2, hi_prev)
        if not i1 < tbar < i2:
            break
        blocks.append(Block(jk, i1, i2))
        lo_prev, hi_prev = i1, i2
        k += 1
    return Partition(g, m_terms, eps, nm, alpha_n, len(blocks), tuple(blocks), tbar)


# ---------------------------------------------------------------------------
# Quadrature (quadrature.py:35-78)

def moments(p: JacobiParameters, g: int) -> np.ndarray:
    p.require_core("the moment recurrence")
    a, b = p.alpha, p.beta
    s = a + b
    mu = np.empty(g + 1)
    mu0 = 2.0 ** (s + 1.0) * math.gamma(a + 1.0) * math.gamma(b + 1.0) / math.gamma(s + 2.0)
    # the serial recurrence (quadrature.py:35-53) runs in the native library,
    # same operation order and rounding as the reference's loop
    from . import _native as nat
    nat.check(nat.lib().cjt_host_moments(a, b, mu0, g, mu.ctypes.data), "moments")
    return mu


def dct1_host(x: np.ndarray) -> np.ndarray:
    """sum_k cos(pi j k / G) x_k with the reference's staging (trig.py:35-40).
    Plan-time only (quadrature weights)."""
    st = np.array(x, dtype=float)
    st[1:-1] *= 0.5
    return scipy.fft.dct(st, type=1)


def cc_weights(p: JacobiParameters, g: int, mu: np.ndarray) -> np.ndarray:
    st = np.empty(g + 1)
    st[0] = mu[0]
    st[-1] = mu[g]
    st[1:-1] = 2.0 * mu[1:g]
    w = dct1_host(st)
    w /= g
    w[0] *= 0.5
    w[-1] *= 0.5
    return w


# ---------------------------------------------------------------------------
# Exact unit phases for the chirp-z layout

_PI_LD = np.longdouble("3.14159265358979323846264338327950288419716939937510")


_PHASE_B = 2048


@functools.lru_cache(maxsize=32)
def _phase_tables(den: int):
    """exp(2 pi i a B / den) and exp(2 pi i b / den), b < B, in 80-bit extended."""
    def tab(idx):
        ang = (2 * _PI_LD) * idx.astype(np.longdouble) / np.longdouble(den)
        return np.cos(ang) + np.clongdouble(1j) * np.sin(ang)
    hi = tab(np.arange(den // _PHASE_B + 1, dtype=np.int64) * _PHASE_B)
    lo = tab(np.arange(_PHASE_B, dtype=np.int64))
    return hi, lo


def unit_phase(num, den: int) -> np.ndarray:
    """exp(2 pi i num/den) for integer num: num reduced exactly mod den, the
    phase as the 80-bit product of two tabulated 80-bit phases, rounded to
    double (|error| <= ~0.5 ulp + 2^-63)."""
    r = np.mod(np.asarray(num, dtype=np.int64), den)
    hi, lo = _phase_tables(int(den))
    return (hi[r // _PHASE_B] * lo[r % _PHASE_B]).astype(np.complex128)


def chirp(k, g: int) -> np.ndarray:
    """exp(i pi k^2 / (2G)) with k^2 reduced exactly mod 4G."""
    k = np.asarray(k, dtype=np.int64)
    return unit_phase(np.mod(k * k, 4 * g), 4 * g)


def _next_pow2(v: int) -> int:
    return 1 << max(4, int(v - 1).bit_length())


class Modulation:
    """A diagonal of u_m - i v_m (asymptotics.py:36-75, endpoint rows zeroed as
    engine.py:138-139) over grid rows row0 .. row0 + len - 1; built on the
    device by the library (cjt_plan_dev.cu) or on the host on demand."""

    def __init__(self, p: "JacobiParameters", m_count: int, thetas: np.ndarray, row0: int, length: int):
        self.p, self.m_count, self.thetas, self.row0, self.length = p, m_count, thetas, row0, length

    def host(self) -> np.ndarray:
        g = len(self.thetas) - 1
        rows = np.arange(self.row0, self.row0 + self.length)
        u, v = modulation(self.p, self.m_count, self.thetas[rows])
        edge = (rows == 0) | (rows == g)
        u[:, edge] = 0.0
        v[:, edge] = 0.0
        return u - 1j * v


class ChirpZ:
    """One batched chirp-z product with fused diagonal scalings:

        out[b, q0+s-out_shift] (+)= sum_m Re(post[m, s] * z_{b,m}[s]),
        z_{b,m}[s] = sum_t exp(i pi (p0+t)(q0+s)/G) pre[m, t] x[b, p0+t].

    The index rectangle (input t < width) x (output s < count) may be tiled:
    tile (j, i) covers inputs tiles_in[i] and outputs tiles_out[j] and is one
    Bluestein convolution of length `length` with spectrum kernel_hat[j, i].

    `pre_diag` / `post_diag` are the bare diagonals (arrays, or Modulation);
    with device_tables the library builds the chirps, folded tables and
    spectra on the GPU.  `pre`, `post` and `kernel_hat`
    are the host-built equivalents, computed on first access (tests, the
    standalone trigonometric transforms, $CJT_DEVICE_PLAN=0)."""

    def __init__(self, g, p0, width, q0, count, length, pre_diag, post_diag, accumulate,
                 tiles_in, tiles_out, out_shift=0, device_tables=True):
        self.g, self.p0, self.width, self.q0, self.count, self.length = g, p0, width, q0, count, length
        self.pre_diag, self.post_diag = pre_diag, post_diag
        self.accumulate = accumulate
        self.tiles_in, self.tiles_out = tiles_in, tiles_out
        self.out_shift = out_shift
        self.device_tables = device_tables
        self._pre = self._post = self._khat = None

    @property
    def m_count(self) -> int:
        d = self.pre_diag
        return d.m_count if isinstance(d, Modulation) else np.atleast_2d(d).shape[0]

    @staticmethod
    def _diag(d) -> np.ndarray:
        return d.host() if isinstance(d, Modulation) else np.atleast_2d(d)

    @property
    def pre(self) -> np.ndarray:
        if self._pre is None:
            pidx = np.arange(self.p0, self.p0 + self.width, dtype=np.int64)
            self._pre = np.ascontiguousarray(self._diag(self.pre_diag) * chirp(pidx, self.g)[None, :],
                                             dtype=np.complex128)
        return self._pre

    @property
    def post(self) -> np.ndarray:
        if self._post is None:
            qidx = np.arange(self.q0, self.q0 + self.count, dtype=np.int64)
            self._post = np.ascontiguousarray(self._diag(self.post_diag) * chirp(qidx, self.g)[None, :],
                                              dtype=np.complex128)
        return self._post

    @property
    def kernel_hat(self) -> np.ndarray:
        """(n_out, n_in, length) complex spectra, 1/length folded in."""
        if self._khat is None:
            khat = np.empty((len(self.tiles_out), len(self.tiles_in), self.length), dtype=np.complex128)
            for j, (so, sc) in enumerate(self.tiles_out):
                for i, (to, tw) in enumerate(self.tiles_in):
                    khat[j, i] = _spectrum(self.g, self.p0 + int(to), int(tw), self.q0 + int(so), int(sc),
                                           self.length)
            self._khat = khat
        return self._khat


FUSED_MAX = 8192        # largest Bluestein length kept entirely in one CTA's shared memory


# Measured B200 costs (ps per point per term per vector; config-2 launch
# lists, profiles/): an on-chip tile costs a forward FFT per input tile (with
# the fused loads and the spectrum sum) plus an inverse FFT per output tile;
# tiles up to 4096 points run 2 CTAs/SM, 8192-point tiles one.  An untiled
# multi-pass Bluestein (HBM round trips) costs _MULTIPASS per point: 18.5 ps
# with register column passes (L <= 2^17), ~29 ps with shared-memory columns
# (config-4 launch lists).
_TILE_COST = {4096: (9.7, 6.5), 8192: (10.9, 7.1)}   # (forward, inverse)
_MULTIPASS_COST = (18.5, 29.0)                       # register / shared-memory column passes


def _cost_overrides():
    """$CJT_TILE_COST="f4096,i4096,f8192,i8192,mp_reg,mp_smem" (experiments)."""
    import os
    e = os.environ.get("CJT_TILE_COST")
    if not e:
        return _TILE_COST, _MULTIPASS_COST
    v = [float(x) for x in e.split(",")]
    return {4096: (v[0], v[1]), 8192: (v[2], v[3])}, (v[4], v[5])


def _cost(length: int, n_in: int, n_out: int) -> float:
    tile, mp = _cost_overrides()
    if length <= FUSED_MAX:
        fwd, inv = tile[max(4096, length)]
        return n_out * length * (fwd * n_in + inv)
    # multi-pass: half the per-point cost per FFT; tiled multi-pass runs one
    # forward FFT per input tile and one inverse FFT per output tile (input
    # spectra summed, or one forward spectrum shared by the output tiles)
    return length * (mp[0] if length <= 1 << 17 else mp[1]) * 0.5 * (n_in + n_out)


def _spectrum(g: int, p0: int, width: int, q0: int, count: int, length: int) -> np.ndarray:
    """FFT of the cyclic kernel conj(chirp(q - p)), d = (q0 - p0) + s - t, / length."""
    ker = np.zeros(length, dtype=np.complex128)
    off = q0 - p0
    ker[:count] = np.conj(chirp(off + np.arange(count, dtype=np.int64), g))
    if width > 1:
        ker[length - width + 1:] = np.conj(chirp(off - np.arange(width - 1, 0, -1, dtype=np.int64), g))
    return np.fft.fft(ker) / length


def _split(n: int, parts: int) -> np.ndarray:
    edges = (np.arange(parts + 1, dtype=np.int64) * n) // parts
    return np.stack([edges[:-1], edges[1:] - edges[:-1]], axis=1)


KHAT_MAX_POINTS = 1 << 24    # tile spectra stored per chirp-z (x 16 B)


@functools.lru_cache(maxsize=4096)
def tile_layout(width: int, count: int, fused_max: int = FUSED_MAX):
    """Choose (length, n_in, n_out) for a width x count chirp-z: one untiled
    power-of-two Bluestein, or a grid of on-chip tiles, by measured cost."""
    whole = _next_pow2(width + count - 1)
    best = (_cost(whole, 1, 1), whole, 1, 1)
    # tiled multi-pass: input tiles (n_out = 1) or output tiles (n_in = 1)
    lm = 2 * fused_max
    while lm < whole:
        for n_in, n_out in [(k, 1) for k in range(2, 9)] + [(1, k) for k in range(2, 9)]:
            if -(-width // n_in) + -(-count // n_out) - 1 > lm or n_in * n_out * lm > KHAT_MAX_POINTS:
                continue
            cost = _cost(lm, n_in, n_out)
            if cost < best[0]:
                best = (cost, lm, n_in, n_out)
        lm *= 2
    lc = 1024
    while lc <= fused_max:
        n_min = -(-width // (lc - 1))
        for n_in in range(n_min, 8 * n_min + 64):
            wc = -(-width // n_in)
            n_out = -(-count // (lc - wc + 1))
            if n_in * n_out * lc > KHAT_MAX_POINTS:
                continue
            # one forward FFT per input tile and one inverse FFT per output
            # tile (input tiles are summed in the frequency domain)
            cost = _cost(lc, n_in, n_out)
            if cost < best[0]:
                best = (cost, lc, n_in, n_out)
        lc *= 2
    return best[1:]


def device_planning() -> bool:
    """Chirp-z tables and spectra are built on the device unless $CJT_DEVICE_PLAN=0."""
    import os
    return os.environ.get("CJT_DEVICE_PLAN", "1") != "0"


def chirpz(g: int, p0: int, width: int, q0: int, count: int,
           pre_scale, post_scale, accumulate: bool,
           tiled: bool = True, out_shift: int = 0, device_tables: bool | None = None) -> ChirpZ:
    """Lay out sum_p x_p e^{i pi p q/G} over [p0, p0+width) x [q0, q0+count)
    as a (tiled) Bluestein product.  pre_scale/post_scale: (M, width)/(M,
    count) real or complex diagonals, or Modulation."""
    if tiled:
        length, n_in, n_out = tile_layout(width, count)
    else:
        length, n_in, n_out = _next_pow2(width + count - 1), 1, 1
    if device_tables is None:
        device_tables = device_planning()
    return ChirpZ(g, p0, width, q0, count, length, pre_scale, post_scale, accumulate,
                  _split(width, n_in), _split(count, n_out), out_shift, device_tables)


# ---------------------------------------------------------------------------
# Whole-plan host description


@dataclass
class HostPlan:
    direction: str
    p: JacobiParameters
    n: int
    m_terms: int
    eps: float
    grid_n: int
    thetas: np.ndarray
    regions: np.ndarray
    cuts: np.ndarray
    layout: Partition
    tables: RecurrenceTables
    rec_cuts: np.ndarray          # cuts capped to the degrees the transform keeps
    blocks: list = field(default_factory=list)   # list[ChirpZ]
    analysis: ChirpZ | None = None   # forward: Lobatto values -> Chebyshev coefficients
    synthesis: ChirpZ | None = None  # inverse: Chebyshev coefficients -> weighted values
    weights: np.ndarray | None = None
    scalings: np.ndarray | None = None
    # alpha = beta = 1/2 exact expansion (half_exact_enabled): k_n = P_n(1)/(n+1)
    half_k: np.ndarray | None = None
    half_gemm: bool = False               # inverse: exact conversion + tensor-core correction
    exec_cuts: np.ndarray | None = None   # recurrence rows the device runs (None: cuts / rec_cuts)

    @property
    def device_cuts(self) -> np.ndarray:
        if self.exec_cuts is not None:
            return self.exec_cuts
        return self.cuts if self.direction == "forward" else self.rec_cuts


def host_angles(thetas: np.ndarray, regions: np.ndarray):
    """x = cos(theta) and the half-angle x -+ 1 values with the host libm, as
    the reference kernel computes them per point (_kernels_cy.pyx:27, 58-64)."""
    from . import _native as nat
    th = np.ascontiguousarray(thetas, dtype=np.float64)
    reg = np.ascontiguousarray(regions, dtype=np.int8)
    x, xm = np.empty(len(th)), np.empty(len(th))
    nat.check(nat.lib().cjt_host_angles(th.ctypes.data, reg.ctypes.data, len(th), x.ctypes.data,
                                        xm.ctypes.data), "cjt_host_angles")
    return x, xm


def half_exact_enabled(p: JacobiParameters) -> bool:
    """alpha = beta = 1/2 runs the exact (terminating) Hahn expansion instead
    of the reference's all-recurrence layout ($CJT_HALF_EXACT=0 disables)."""
    import os
    return p.alpha == 0.5 and p.beta == 0.5 and os.environ.get("CJT_HALF_EXACT", "1") != "0"


def half_exact_k(n: int) -> np.ndarray:
    """k_m = P_m(1)/(m+1), m <= n, in binary128 (all the forward plan needs)."""
    from . import _native as nat
    k = np.empty(n + 1)
    nat.check(nat.lib().cjt_host_half_exact(None, None, None, 0, n, k.ctypes.data, None, None),
              "cjt_host_half_exact")
    return k


def half_exact_tables(thetas: np.ndarray, regions: np.ndarray, g: int, n: int):
    """(k, inv_sin, delta_over_sin): k_m = P_m(1)/(m+1) (m <= n), and per grid
    row p the angle phi_p of the point the reference's recurrence evaluates
    (libm x_p / half-angle xm_p) as 1/sin(phi_p) and (phi_p - pi p/G)/sin(phi_p),
    in binary128 (csrc/cjt_host.cpp)."""
    from . import _native as nat
    x, xm = host_angles(thetas, regions)
    reg = np.ascontiguousarray(regions, dtype=np.int8)
    k, inv_sin, dos = np.empty(n + 1), np.empty(g + 1), np.empty(g + 1)
    nat.check(nat.lib().cjt_host_half_exact(x.ctypes.data, xm.ctypes.data, reg.ctypes.data, g, n,
                                            k.ctypes.data, inv_sin.ctypes.data, dos.ctypes.data),
              "cjt_host_half_exact")
    return k, inv_sin, dos


HALF_GEMM_MAX_N1 = 16384   # largest N+1 of the tensor-core correction ((N+1)^2 bf16 matrix per plan)


def half_gemm_enabled(n: int) -> bool:
    """alpha = beta = 1/2 inverse as exact conversion + correction GEMM for
    N + 1 <= HALF_GEMM_MAX_N1 ($CJT_HALF_GEMM=0 keeps the one-chirp-z form)."""
    import os
    return n + 1 <= HALF_GEMM_MAX_N1 and os.environ.get("CJT_HALF_GEMM", "1") != "0"


def half_correction_inverse(g: int, n: int, k: np.ndarray, inv_sin: np.ndarray, dos: np.ndarray,
                            scalings: np.ndarray) -> ChirpZ:
    """The reference's inverse minus the exact conversion, to first order in
    the evaluation-point offsets delta_p (half_exact_tables):

      M t [m] = k_m / A_m sum_p wv_p delta_p d/dtheta[sin(q theta)/sin theta](pi p/G)
              = k_m / A_m [ q sum_p wv_p delta_p / sin theta_p cos(pi p q/G)
                            - sum_p wv_p delta_p cos theta_p / sin^2 theta_p sin(pi p q/G) ],

    q = m + 1, theta_p = pi p/G, wv = the weighted synthesis of t (edge);
    endpoint rows have delta = 0.  The library applies it to the identity once
    per plan to form the correction matrix (cjt_plan_desc.half_gemm)."""
    p_ = np.arange(g + 1, dtype=np.float64)
    th = np.pi * p_ / g
    with np.errstate(divide="ignore", invalid="ignore"):
        delta = np.where(inv_sin != 0.0, dos / inv_sin, 0.0)
        s_, c_ = np.sin(th), np.cos(th)
        pre = np.zeros((2, g + 1))
        pre[0, 1:-1] = delta[1:-1] / s_[1:-1]
        pre[1, 1:-1] = -delta[1:-1] * c_[1:-1] / (s_[1:-1] * s_[1:-1])
    q = np.arange(1, n + 2, dtype=np.float64)
    ks = k * scalings
    post = np.empty((2, n + 1), dtype=np.complex128)
    post[0] = ks * q
    post[1] = -1j * ks
    return chirpz(g, 0, g + 1, 1, n + 1, pre, post, accumulate=False, out_shift=1)


def half_exact_inverse(g: int, n: int, k: np.ndarray, inv_sin: np.ndarray, dos: np.ndarray,
                       scalings: np.ndarray) -> ChirpZ:
    """The inverse's whole contraction for alpha = beta = 1/2 as ONE chirp-z
    product over the weighted grid values wv (engine.py:220-227 with
    P_m(cos phi) = k_m sin((m+1) phi)/sin phi evaluated at the reference's
    points phi_p = pi p/G + delta_p, to first order in (m+1) delta_p):

      out[m] = k_m / A_m [ sum_p wv_p / sin(phi_p) sin(pi p q/G)
                           + q sum_p wv_p delta_p / sin(phi_p) cos(pi p q/G) ],  q = m + 1

    plus the endpoint rows' exact limits P_m(+-1) = k_m (m+1) (+-1)^m.  Term 0
    (cosine, Re z) carries delta/sin and the endpoints, term 1 (sine, Im z)
    1/sin; outputs q = 1..N+1 land at out[q - 1]."""
    pre = np.zeros((2, g + 1))
    pre[0] = dos
    pre[0, 0], pre[0, g] = 1.0, -1.0
    pre[1] = inv_sin
    q = np.arange(1, n + 2, dtype=np.float64)
    ks = k * scalings
    post = np.empty((2, n + 1), dtype=np.complex128)
    post[0] = ks * q
    post[1] = -1j * ks
    return chirpz(g, 0, g + 1, 1, n + 1, pre, post, accumulate=False, out_shift=1)


def _build_half_exact(hp: HostPlan) -> HostPlan:
    """alpha = beta = 1/2: the reference's layout (no blocks, every row in the
    recurrence region) is kept in hp.layout / hp.cuts for the SURVEY 8(d)
    accounting; the device runs the exact expansion instead (no recurrence
    rows): forward = U -> T conversion with k_n, inverse = synthesis + one
    chirp-z (half_exact_inverse)."""
    g, n = hp.grid_n, hp.n
    if hp.direction == "inverse":
        k, inv_sin, dos = half_exact_tables(hp.thetas, hp.regions, g, n)
    else:
        k = half_exact_k(n)     # the row tables (binary128, ~1 us per row) are the inverse's
    hp.half_k = k
    hp.exec_cuts = np.zeros(g + 1, dtype=np.int64)
    if hp.direction == "inverse":
        mu = moments(hp.p, g)
        w = cc_weights(hp.p, g, mu)
        hp.weights = w
        hp.synthesis = chirpz(g, 0, n + 1, 0, g + 1, np.ones((1, n + 1)), w[None, :], accumulate=False)
        hp.scalings = 1.0 / orthonormality(hp.p, n)
        if half_gemm_enabled(n):
            hp.half_gemm = True
            hp.blocks = [half_correction_inverse(g, n, k, inv_sin, dos, hp.scalings)]
        else:
            hp.blocks = [half_exact_inverse(g, n, k, inv_sin, dos, hp.scalings)]
    return hp


def build(direction: str, p: JacobiParameters, n: int,
          m_terms: int = DEFAULT_M, eps: float = DEFAULT_EPS) -> HostPlan:
    """Plan one direction (engine.py:96-130) and lay out its device work."""
    if direction not in ("forward", "inverse"):
        raise ValueError("direction must be 'forward' or 'inverse'")
    p.require_core(f"the {direction} transform plan")
    if n < 1:
        raise ValueError("N must be >= 1")
    if m_terms < 2:
        raise ValueError("M >= 2 required")
    g = n if direction == "forward" else 2 * n
    th = angle_grid(g)
    layout = partition(p, g, m_terms, eps, th)
    tables = recurrence_tables(p, g + 1)
    cuts = layout.row_cuts()
    regions = region_codes(th)
    cuts.flags.writeable = False
    regions.flags.writeable = False
    hp = HostPlan(direction, p, n, m_terms, eps, g, th, regions, cuts, layout, tables,
                  np.minimum(cuts, n + 1))
    if half_exact_enabled(p) and not layout.blocks:
        return _build_half_exact(hp)

    if layout.blocks:
        # engine.py:133-141: u - i v over each block's rows (Modulation; built
        # on the device), C_{n,m} columns of its strip
        # only degrees <= N are used (inverse strips are clipped to N); the
        # table's values do not depend on its length once it reaches the
        # Stirling switch degree
        ccols = cnm_table(p, min(g, max(n, _cnm_switch(p.alpha, p.beta))), m_terms)
        jobs = []
        for (lo, hi), blk in zip(layout.column_strips(), layout.blocks):
            nrow = blk.i2 - blk.i1 + 1
            w_uv = Modulation(p, m_terms, th, blk.i1, nrow)
            if direction == "forward":
                # values[rows] += u_m DCT(C_m c)[rows] + v_m DST(C_m c)[rows]
                jobs.append((g, lo, hi - lo + 1, blk.i1, nrow,
                             np.ascontiguousarray(ccols[lo:hi + 1, :].T), w_uv, True))
            else:
                # out[strip] += C_m (DCT(u_m wv) + DST(v_m wv)); degrees > N dropped
                top = min(hi, n)
                if lo > top:
                    continue
                jobs.append((g, blk.i1, nrow, lo, top - lo + 1,
                             w_uv, np.ascontiguousarray(ccols[lo:top + 1, :].T), True))
        hp.blocks = [chirpz(*a) for a in jobs]

    if direction == "forward":
        # chebyshev_analysis (trig.py:53-63): scipy DCT-I of 0.5 v, i.e. the
        # plain cosine sum with the two end samples halved, then 2/G with the
        # two end coefficients halved
        pre = np.ones(g + 1)
        pre[0] = pre[-1] = 0.5
        post = np.full(g + 1, 2.0 / g)
        post[0] *= 0.5
        post[-1] *= 0.5
        hp.analysis = chirpz(g, 0, g + 1, 0, g + 1, pre[None, :],
                             post[None, :], accumulate=False)
    else:
        mu = moments(p, g)
        w = cc_weights(p, g, mu)
        hp.weights = w
        # wv = w * dct1([c, 0...]) (engine.py:201-203)
        hp.synthesis = chirpz(g, 0, n + 1, 0, g + 1, np.ones((1, n + 1)),
                              w[None, :], accumulate=False)
        hp.scalings = 1.0 / orthonormality(p, n)
    return hp
