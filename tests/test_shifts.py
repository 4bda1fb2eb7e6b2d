"""Parameter shifts and jacobi_to_jacobi (engine.py:232-354): the oracle
restatement against golden vectors from the reference itself
(tests/golden/make_golden_shifts.py), the product's argument checks (no GPU
needed), and the C ABI's argument validation."""
import numpy as np
import pytest

import cjt_oracle as O
import paper_1602_02618_b200 as cj
from conftest import ROOT
from paper_1602_02618_b200 import _native as nat

G = np.load(ROOT / "tests" / "golden" / "shifts.npz")
OPS = ("increment_beta", "decrement_beta", "increment_alpha", "decrement_alpha")
ORACLE = {"increment_beta": O.oracle_increment_beta, "decrement_beta": O.oracle_decrement_beta,
          "increment_alpha": O.oracle_increment_alpha, "decrement_alpha": O.oracle_decrement_alpha}
SHIFT_IDS = sorted({k.split("_")[0] for k in G.files if k.startswith("shift")})
J2J_IDS = sorted({k.split("_")[0] for k in G.files if k.startswith("j2j")})


@pytest.mark.parametrize("case", SHIFT_IDS)
def test_oracle_shifts_bitwise_vs_reference(case):
    a, b = G[f"{case}_ab"]
    c = G[f"{case}_c"]
    seen = 0
    for op in OPS:
        key = f"{case}_{op}"
        if key not in G.files:
            continue
        seen += 1
        got = ORACLE[op](float(a), float(b), c)
        assert np.array_equal(got, G[key]), op
    assert seen >= 2


@pytest.mark.parametrize("case", J2J_IDS)
def test_oracle_to_core_and_jacobi_to_jacobi_vs_reference(case):
    a, b, ta, tb = (float(v) for v in G[f"{case}_case"])
    c = G[f"{case}_c"]
    ca, cb, core = O.oracle_to_core(a, b, c)
    assert (ca, cb) == tuple(G[f"{case}_core_ab"])
    assert np.array_equal(core, G[f"{case}_core"])
    got = O.oracle_jacobi_to_jacobi(a, b, c, ta, tb)
    ref = G[f"{case}_out"]
    assert np.max(np.abs(got - ref)) <= 1e-15 * np.sum(np.abs(c)) * max(1.0, np.max(np.abs(ref)))


def test_spec_examples_in_oracle():
    # SPEC: (0,0) e_1 -> [1/3, 2/3] in (0,1); alpha: e_1 -> [-1/3, 2/3] in (1,0)
    assert np.allclose(O.oracle_increment_beta(0.0, 0.0, [0.0, 1.0]), [1 / 3, 2 / 3], rtol=0, atol=1e-16)
    assert np.allclose(O.oracle_increment_alpha(0.0, 0.0, [0.0, 1.0]), [-1 / 3, 2 / 3], rtol=0, atol=1e-16)
    assert np.allclose(O.oracle_decrement_beta(0.0, 1.0, [1 / 3, 2 / 3]), [0.0, 1.0], rtol=0, atol=1e-15)


def test_product_argument_errors_without_gpu():
    c = cj.jacobi(cj.JacobiParameters(0.0, -0.5), np.ones(4))
    with pytest.raises(cj.ParameterRangeError, match="inadmissible shift target"):
        cj.decrement_beta(c)
    with pytest.raises(ValueError, match="require Jacobi coefficients"):
        cj.increment_beta(cj.chebyshev(np.ones(4)))
    with pytest.raises(ValueError, match="unknown shift"):
        cj.shift_batched("increment_gamma", cj.JacobiParameters(0.0, 0.0), None)


def test_abi_shift_validation():
    lib = nat.lib()
    buf = np.zeros(8)
    # inadmissible target, aliasing, bad sizes: rejected before any device work
    assert lib.cjt_jacobi_shift(nat.SHIFT_DEC_BETA, 0.0, -0.25, buf.ctypes.data, buf[4:].ctypes.data,
                                3, 1, None) == nat.CJT_EINVAL
    assert lib.cjt_jacobi_shift(nat.SHIFT_INC_BETA, 0.0, 0.0, buf.ctypes.data, buf.ctypes.data,
                                3, 1, None) == nat.CJT_EINVAL
    assert lib.cjt_jacobi_shift(7, 0.0, 0.0, buf.ctypes.data, buf[4:].ctypes.data,
                                3, 1, None) != nat.CJT_OK
    assert lib.cjt_jacobi_shift(nat.SHIFT_INC_BETA, 0.0, 0.0, buf.ctypes.data, buf[4:].ctypes.data,
                                -1, 1, None) == nat.CJT_EINVAL
