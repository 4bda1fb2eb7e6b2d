"""The oracle (oracle/cjt_oracle.py + oracle/recur.c) pinned against the
reference's outputs (tests/golden/*.npz) and the reference's known answers."""
import numpy as np
import pytest

import cjt_oracle as O
from conftest import load_golden
from paper_1602_02618_b200 import planner as P

NAMES = ["cfg1", "cfg2_small", "cfg2_full", "cfg3_full", "cfg4_small", "cfg5_a", "cfg5_b", "cfg5_c",
         "cfg5_d", "cfg5_e", "tiny", "edge_n1"]


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_reference(name):
    g = load_golden(name)
    a, b = float(g["alpha"]), float(g["beta"])
    for v in range(g["c"].shape[0]):
        f = O.oracle_forward(a, b, g["c"][v])
        i = O.oracle_inverse(a, b, g["fwd"][v])
        # same algorithm, same libm, same scipy, same operation order: bit-exact here;
        # a different host libm/SIMD may move the last bits, so allow 1e-15 relative
        assert O.parity(f, g["fwd"][v], g["c"][v]) <= 1e-15
        assert O.parity(i, g["inv"][v], g["fwd"][v]) <= 1e-15


def test_oracle_vs_double_double_dense():
    # reference's dense double-double oracle_forward (oracle.py:195-222), stored by make_golden
    g = load_golden("cfg1")
    f = O.oracle_forward(0.0, 0.0, g["c"][0])
    assert O.parity(f, g["dense"], g["c"][0]) <= 1e-15


def test_known_answers_legendre():
    # test_oracle.py:76-87: e0 -> e0, e2 -> [1/4, 0, 3/4] (P2 = (3 T2 + T0)/4)
    n = 16
    e0 = np.zeros(n + 1); e0[0] = 1.0
    e2 = np.zeros(n + 1); e2[2] = 1.0
    assert np.max(np.abs(O.oracle_forward(0.0, 0.0, e0) - e0)) < 1e-15
    ref = np.zeros(n + 1); ref[0] = 0.25; ref[2] = 0.75
    assert np.max(np.abs(O.oracle_forward(0.0, 0.0, e2) - ref)) < 1e-15


def test_c_kernels_match_reference_numpy_backend():
    # the reference's NumPy backend equals the Cython kernel bit for bit on the
    # forward; restated here from _kernels_np.py:22-57
    p = P.JacobiParameters(-0.2, 0.45)
    n = 300
    t = P.recurrence_tables(p, n + 1)
    th = P.angle_grid(n)
    cuts = np.full(n + 1, n + 1, dtype=np.int64)
    cuts[40:200] = 57
    reg = P.region_codes(th)
    c = np.random.default_rng(3).standard_normal(n + 1)
    out = np.empty(n + 1)
    O.clenshaw_points(t.A, t.B, t.C, t.rb_plus, t.rb_minus, t.rb_plus_inv, t.rb_minus_inv,
                      c, th, cuts, reg, out)
    ref = np.zeros(n + 1)
    for i in range(n + 1):
        nc = cuts[i]
        if reg[i] == 0:
            x = np.cos(th[i])
            u1 = u2 = 0.0
            for k in range(nc - 1, -1, -1):
                u1, u2 = (t.A[k] * x + t.B[k]) * u1 - t.C[k + 1] * u2 + c[k], u1
            ref[i] = u1
        else:
            h = np.sin(0.5 * th[i]) if reg[i] == 1 else np.cos(0.5 * th[i])
            xm = -2.0 * h * h if reg[i] == 1 else 2.0 * h * h
            rb, rbi = (t.rb_plus, t.rb_plus_inv) if reg[i] == 1 else (t.rb_minus, t.rb_minus_inv)
            u = d = 0.0
            for k in range(nc - 1, 0, -1):
                d = (t.A[k] * xm * u + t.C[k + 1] * d + c[k]) * rb[k]
                u = (u + d) * rbi[k]
            ref[i] = t.A[0] * xm * u + t.C[1] * d + c[0]
    assert np.max(np.abs(out - ref)) <= 1e-13 * np.abs(c).sum()


def test_seeded_inputs():
    c = O.seeded_vector(2, 5, 100)
    z = np.random.default_rng(2005).standard_normal(101)
    assert np.array_equal(c, z * (np.arange(101) + 1.0) ** -1.5)
    draws = O.config5_draws(32)
    assert len(draws) == 32 and all(n in {(1 << k) - 1 for k in range(8, 17)} for _, _, n in draws)


def test_oracle_plans_come_from_the_reference():
    """With oracle/_ref present the oracle takes every plan table from the
    reference's own planner (engine.plan + _block_diagonals), so it shares no
    code with the product; the product-planner fallback must agree bit for bit."""
    if O.reference_package() is None:
        pytest.skip("oracle/_ref (the built reference) is not present")
    assert O.plan_source() == "reference"
    g = load_golden("cfg2_small")
    a, b = float(g["alpha"]), float(g["beta"])
    O._plan.cache_clear()
    f_ref, i_ref = O.oracle_forward(a, b, g["c"][0]), O.oracle_inverse(a, b, g["fwd"][0])
    assert O._plan("forward", a, b, int(g["n"]), 7, O.DEFAULT_EPS).source == "reference"
    real = O.reference_package
    try:
        O.reference_package = lambda: None
        O._plan.cache_clear()
        assert O.plan_source() == "product-planner"
        f_pl, i_pl = O.oracle_forward(a, b, g["c"][0]), O.oracle_inverse(a, b, g["fwd"][0])
        assert O._plan("forward", a, b, int(g["n"]), 7, O.DEFAULT_EPS).source == "product-planner"
    finally:
        O.reference_package = real
        O._plan.cache_clear()
    assert np.array_equal(f_ref, f_pl) and np.array_equal(i_ref, i_pl)
