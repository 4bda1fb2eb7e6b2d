"""Host planner vs the reference: partitions, tables and the chirp-z layout.

Golden data: tests/golden/layouts.json and *.npz were produced by the
reference itself (tests/golden/make_golden.py); the frozen values below are
the reference's own known answers (test_asymptotics.py:146-147, 186-192;
test_kernels.py:175-273).
"""
import hashlib
import json
import math

import mpmath as mp
import numpy as np
import pytest

from conftest import GOLDEN
from paper_1602_02618_b200 import planner as P

EPS = float(np.finfo(float).eps)
LAYOUTS = json.loads((GOLDEN / "layouts.json").read_text())
CASES = {
    "cfg1": (0.0, 0.0, 1023), "cfg2_small": (-0.25, 0.4, 2047), "cfg2_full": (-0.25, 0.4, 16383),
    "cfg3_full": (0.5, 0.5, 4095), "cfg4_small": (0.3, -0.45, 8191), "cfg5_a": (-0.45, 0.25, 255),
    "cfg5_b": (0.5, -0.2, 511), "cfg5_c": (0.0, 0.5, 2047), "cfg5_d": (0.25, 0.25, 4095),
    "cfg5_e": (0.5, 0.5, 1023), "tiny": (-0.25, 0.4, 3), "edge_n1": (0.125, -0.375, 1),
}


def digest(hp):
    h = hashlib.sha256()
    t = hp.tables
    for name in ("A", "B", "C", "rf_plus", "rf_minus", "rf_plus_inv", "rf_minus_inv"):
        h.update(np.ascontiguousarray(getattr(t, name)).tobytes())
    h.update(hp.cuts.tobytes())
    h.update(hp.regions.tobytes())
    h.update(hp.thetas.tobytes())
    if hp.weights is not None:
        h.update(hp.weights.tobytes())
        h.update(hp.scalings.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("direction", ["forward", "inverse"])
def test_plan_bitwise_vs_reference(name, direction):
    a, b, n = CASES[name]
    hp = P.build(direction, P.JacobiParameters(a, b), n)
    ref = LAYOUTS[name][direction]
    assert [[blk.j, blk.i1, blk.i2] for blk in hp.layout.blocks] == ref["blocks"]
    assert hp.layout.n_m == ref["n_m"] and hp.layout.theta_bar_index == ref["tbar"]
    assert digest(hp) == ref["digest"]


@pytest.mark.parametrize("name,params", [("cfg4_full", (0.3, -0.45, 2**20 - 1)),
                                         ("cfg5_max", (0.5, -0.45, 65535)),
                                         ("frozen_2_14", (0.125, 0.375, 2**14))])
def test_full_size_partitions(name, params):
    a, b, n = params
    for direction in ("forward", "inverse"):
        g = n if direction == "forward" else 2 * n
        lay = P.partition(P.JacobiParameters(a, b), g, 7, EPS)
        ref = LAYOUTS[name][direction]
        assert [[blk.j, blk.i1, blk.i2] for blk in lay.blocks] == ref["blocks"]
        assert lay.n_m == ref["n_m"] and lay.theta_bar_index == ref["tbar"]


def test_frozen_reference_values():
    assert P.n_m(P.JacobiParameters(0.0, 0.0), 7, EPS) == 111
    assert P.n_m(P.JacobiParameters(0.0, 0.0), 7, 1e6) == 0
    lay = P.partition(P.JacobiParameters(0.125, 0.375), 2**14, 7, EPS)
    assert lay.n_m == 107 and lay.k == 3
    assert [blk.j for blk in lay.blocks] == [3256, 647, 128]
    assert [(blk.i1, blk.i2) for blk in lay.blocks] == [(237, 16145), (1157, 15272), (6069, 10921)]


def test_half_half_has_no_blocks():
    # alpha = beta = 1/2: g_M == 0, tbar = 0 -> no certified block (pure recurrence)
    lay = P.partition(P.JacobiParameters(0.5, 0.5), 4095, 7, EPS)
    assert lay.k == 0 and lay.blocks == ()


def mp_cnm(a, b, n, m):
    with mp.workdps(40):
        a, b = mp.mpf(a), mp.mpf(b)
        return float(2 ** (2 * n - m + a + b + 1) * mp.beta(n + a + 1, n + b + 1)
                     / (mp.pi * mp.rf(2 * n + a + b + 2, m)))


def mp_anab(a, b, n):
    with mp.workdps(40):
        a, b = mp.mpf(a), mp.mpf(b)
        return float(2 ** (a + b + 1) * mp.gamma(n + a + 1) * mp.gamma(n + b + 1)
                     / ((2 * n + a + b + 1) * mp.gamma(n + a + b + 1) * mp.factorial(n)))


@pytest.mark.parametrize("a,b", [(0.0, 0.0), (0.125, 0.375), (-0.49, 0.5), (0.5, 0.5)])
def test_cnm_against_mpmath(a, b):
    p = P.JacobiParameters(a, b)
    table = P.cnm_table(p, 1000, 14)
    for n in (0, 1, 2, 5, 8, 9, 12, 20, 64, 1000):
        for m in (0, 1, 2, 7, 13):
            ref = mp_cnm(a, b, n, m)
            assert abs(P.cnm_scalar(p, n, m) / ref - 1.0) < 1e-13
            assert abs(table[n, m] / ref - 1.0) < 1e-13


@pytest.mark.parametrize("a,b", [(0.125, 0.375), (-0.49, 0.5), (0.5, 0.5)])
def test_orthonormality_against_mpmath(a, b):
    p = P.JacobiParameters(a, b)
    tab = P.orthonormality(p, 10**5)
    for n in (0, 1, 5, 8, 9, 15, 100, 10**5):
        assert abs(tab[n] / mp_anab(a, b, n) - 1.0) < 1e-13


def test_stirling_matches_gamma():
    # S(z) = Gamma(z) e^z z^(1/2-z) / sqrt(2 pi) to relative eps/20 for z >= 9
    for z in (9.0, 10.0, 26.0, 100.0, 591.0, 4000.0):
        with mp.workdps(40):
            zz = mp.mpf(z)
            ref = float(mp.gamma(zz) * mp.e ** zz * zz ** (mp.mpf(0.5) - zz) / mp.sqrt(2 * mp.pi))
        assert abs(float(P.stirling_series(z)) / ref - 1.0) < 4e-16
    with pytest.raises(ValueError):
        P.stirling_series(8.999)


def test_recurrence_tables_immutable_and_conventions():
    t = P.recurrence_tables(P.JacobiParameters(0.25, -0.25), 10)
    assert t.B[0] == 0.25 and t.C[0] == 0.0 and np.isnan(t.rb_plus[0])
    with pytest.raises(ValueError):
        t.A[0] = 1.0


def test_parameter_errors():
    with pytest.raises(P.ParameterRangeError):
        P.JacobiParameters(-1.0, 0.0)
    with pytest.raises(P.ParameterRangeError):
        P.build("forward", P.JacobiParameters(0.7, 0.0), 16)
    with pytest.raises(ValueError):
        P.build("sideways", P.JacobiParameters(0.0, 0.0), 16)
    with pytest.raises(ValueError):
        P.build("forward", P.JacobiParameters(0.0, 0.0), 0)
    with pytest.raises(ValueError):
        P.build("forward", P.JacobiParameters(0.0, 0.0), 16, m_terms=1)


# -- the chirp-z layout the device executes, emulated with NumPy FFTs ----------

def run_chirpz(cz, x, out):
    """Host emulation of one (tiled) chirp-z product exactly as the kernels lay it out."""
    acc = np.zeros(cz.count)
    for m in range(cz.m_count):
        for j, (so, sc) in enumerate(cz.tiles_out):
            for i, (to, tn) in enumerate(cz.tiles_in):
                a = np.zeros(cz.length, complex)
                a[:tn] = x[cz.p0 + to: cz.p0 + to + tn] * cz.pre[m, to:to + tn]
                y = np.fft.ifft(np.fft.fft(a) * cz.kernel_hat[j, i]) * cz.length
                acc[so:so + sc] += (cz.post[m, so:so + sc] * y[:sc]).real
    q = cz.q0 - cz.out_shift
    if cz.accumulate:
        out[q:q + cz.count] += acc
    else:
        out[q:q + cz.count] = acc


@pytest.mark.parametrize("tiled", [False, True])
def test_chirpz_equals_direct_sum(tiled):
    g = 1023
    rng = np.random.default_rng(7)
    p0, w, q0, r = 37, 300, 101, 700
    pre = rng.standard_normal((2, w))
    post = rng.standard_normal((2, r))
    x = rng.standard_normal(p0 + w)
    cz = P.chirpz(g, p0, w, q0, r, pre, post, accumulate=False, tiled=tiled)
    got = np.zeros(q0 + r)
    run_chirpz(cz, x, got)
    pp = np.arange(p0, p0 + w)
    qq = np.arange(q0, q0 + r)
    ang = np.pi * (np.outer(qq, pp) % (2 * g)) / g
    ref = sum((post[m] * ((np.cos(ang) + 1j * np.sin(ang)) @ (pre[m] * x[p0:]))).real for m in range(2))
    assert np.max(np.abs(got[q0:] - ref)) < 1e-12 * np.max(np.abs(ref))


def test_tile_layout_properties():
    for w, r in [(13159, 15956), (2590, 14259), (510, 5206), (30009, 4693), (16772, 813), (1, 1)]:
        length, n_in, n_out = P.tile_layout(w, r)
        assert length & (length - 1) == 0
        assert -(-w // n_in) + -(-r // n_out) - 1 <= length


def _gen_p(hp, nmax):
    t, th = hp.tables, hp.thetas
    x = np.array([math.cos(v) for v in th])
    out = np.zeros((nmax, hp.grid_n + 1))
    for i in range(hp.grid_n + 1):
        reg = hp.regions[i]
        out[0, i] = 1.0
        if reg == 0:
            pp, pc = 0.0, 1.0
            for n in range(1, nmax):
                pp, pc = pc, (t.A[n - 1] * x[i] + t.B[n - 1]) * pc - t.C[n - 1] * pp
                out[n, i] = pc
        else:
            h = math.sin(0.5 * th[i]) if reg == 1 else math.cos(0.5 * th[i])
            xm = -2.0 * h * h if reg == 1 else 2.0 * h * h
            rf, rfi = (t.rf_plus, t.rf_plus_inv) if reg == 1 else (t.rf_minus, t.rf_minus_inv)
            pc, d = 1.0, 0.0
            for n in range(nmax - 1):
                d = (t.A[n] * xm * pc + t.C[n] * d) * rfi[n]
                pc = (pc + d) * rf[n]
                out[n + 1, i] = pc
    return out


def half_forward_host(k, c):
    """Host emulation of k_half_forward: cheb_j = e_j sum_{n >= j, n = j mod 2} k_n c_n."""
    u = np.asarray(k, dtype=np.longdouble) * np.asarray(c, dtype=np.longdouble)
    out = np.zeros(len(c), dtype=np.longdouble)
    for par in (0, 1):
        out[par::2] = np.cumsum(u[par::2][::-1])[::-1]
    out[1:] *= 2
    return out.astype(float)


@pytest.mark.parametrize("name", ["cfg1", "cfg2_small", "cfg5_a", "cfg5_e", "cfg3_full"])
def test_device_decomposition_matches_reference(name, monkeypatch):
    """The exact decomposition the kernels execute (generated-P contraction over
    the recurrence region + tiled chirp-z blocks + chirp-z analysis/synthesis;
    for alpha = beta = 1/2 the exact-expansion path), emulated on the host,
    reproduces the reference's outputs."""
    from conftest import load_golden
    import cjt_oracle as O
    g = load_golden(name)
    a, b, n = float(g["alpha"]), float(g["beta"]), int(g["n"])
    p = P.JacobiParameters(a, b)
    c, ref_f, ref_i = g["c"][0], g["fwd"][0], g["inv"][0]
    if P.half_exact_enabled(p):
        hf, hi = P.build("forward", p, n), P.build("inverse", p, n)
        assert hf.half_k is not None and not hf.blocks and hf.analysis is None
        assert O.parity(half_forward_host(hf.half_k, c), ref_f, c) <= 1e-15
        wv = np.zeros(hi.grid_n + 1)
        run_chirpz(hi.synthesis, ref_f, wv)
        got_i = np.zeros(n + 1)
        (cz,) = hi.blocks
        run_chirpz(cz, wv, got_i)
        if hi.half_gemm:
            # blocks[0] is the correction only: add the exact T -> U conversion
            t = ref_f
            u = np.zeros(n + 1)
            u[0] = t[0]
            u[1:] += 0.5 * t[1:]
            u[:-2] -= 0.5 * t[2:]
            got_i += u / hi.half_k
        assert O.parity(got_i, ref_i, ref_f) <= 1e-13
        if name != "cfg5_e":
            return
        monkeypatch.setenv("CJT_HALF_EXACT", "0")   # and the recurrence layout below
    hf = P.build("forward", p, n)
    pm = _gen_p(hf, n + 1)
    vals = ((pm * (np.arange(n + 1)[:, None] < hf.cuts[None, :])) * c[:, None]).sum(0)
    for cz in hf.blocks:
        run_chirpz(cz, c, vals)
    got_f = np.zeros(n + 1)
    run_chirpz(hf.analysis, vals, got_f)
    assert O.parity(got_f, ref_f, c) <= 1e-13
    hi = P.build("inverse", p, n)
    wv = np.zeros(hi.grid_n + 1)
    run_chirpz(hi.synthesis, ref_f, wv)
    out = np.zeros(n + 1)
    for cz in hi.blocks:
        run_chirpz(cz, wv, out)
    pm = _gen_p(hi, n + 1)
    out += (pm * (np.arange(n + 1)[:, None] < hi.rec_cuts[None, :])) @ wv
    got_i = out * hi.scalings
    assert O.parity(got_i, ref_i, ref_f) <= 1e-13


def test_prefix_cached_tables_equal_direct():
    """The per-(alpha, beta) prefix caches return exactly the directly built
    tables (every entry depends on its degree alone), in any request order."""
    for a, b in ((-0.45, 0.25), (0.5, -0.2), (0.0, 0.0)):
        p = P.JacobiParameters(a, b)
        for n in (70, 4095, 300, 65535, 1000):
            assert np.array_equal(P.cnm_table(p, n, 7), P._cnm_table(p, n, 7))
            assert np.array_equal(P.orthonormality(p, n), P._orthonormality(p, n))
            r, d = P.recurrence_tables(p, n), P._recurrence_tables(p, n)
            for f in ("A", "B", "C", "rf_plus", "rf_minus", "rb_plus", "rb_minus", "rf_plus_inv", "rf_minus_inv"):
                assert np.array_equal(getattr(r, f), getattr(d, f), equal_nan=True)
