"""Expansion-evaluation API (recurrences.py:74-171 of the reference):
jacobi_forward[_reinsch], clenshaw_smith[_reinsch], evaluate_expansion and
the batched device variant, against golden vectors produced by the reference
itself (tests/golden/make_golden_recur.py).  Same operation order as the
reference, so the GPU results are compared BITWISE."""
import math

import numpy as np
import pytest

import paper_1602_02618_b200 as cj
from conftest import ROOT

G = np.load(ROOT / "tests" / "golden" / "recur.npz")
PT = sorted({k.split("_")[0] for k in G.files if k.startswith("pt")})
EV = sorted({k.split("_")[0] for k in G.files if k.startswith("ev")})
THETAS = G["thetas"]


# ---------------------------------------------------------------- host side

def test_angle_grid_matches_reference_expression():
    g = cj.AngleGrid(7)
    assert len(g) == 8
    assert np.array_equal(g.angles, np.pi * np.arange(8) / 7)
    assert not g.angles.flags.writeable
    with pytest.raises(ValueError):
        cj.AngleGrid(0)


def test_classify_region_breakpoints():
    from paper_1602_02618_b200 import recurrences as R
    assert R.classify_region(0.0) == 1 and R.classify_region(math.pi) == -1
    assert R.classify_region(0.25 * math.pi) == 0 and R.classify_region(0.75 * math.pi) == 0
    th = np.array([0.0, 0.25 * math.pi, 0.5, math.pi])
    assert list(R.classify_regions(th)) == [1, 0, 1, -1]


@pytest.mark.parametrize("bad", [-1e-9, math.pi + 1e-9])
def test_theta_range_checked_before_any_device_call(bad):
    p = cj.JacobiParameters(0.0, 0.0)
    for fn in (lambda: cj.jacobi_forward(p, 3, bad), lambda: cj.jacobi_forward_reinsch(p, 3, bad, 1),
               lambda: cj.clenshaw_smith(p, [1.0], bad), lambda: cj.clenshaw_smith_reinsch(p, [1.0], bad, 1)):
        with pytest.raises(ValueError):
            fn()


def test_reinsch_end_checked():
    p = cj.JacobiParameters(0.0, 0.0)
    with pytest.raises(ValueError):
        cj.jacobi_forward_reinsch(p, 3, 0.5, 0)
    with pytest.raises(ValueError):
        cj.clenshaw_smith_reinsch(p, [1.0], 0.5, 2)


def test_empty_clenshaw_returns_zero_like_reference():
    assert cj.clenshaw_smith(cj.JacobiParameters(0.0, 0.0), [], 0.3) == 0.0


# ---------------------------------------------------------------- GPU parity

@pytest.mark.gpu
@pytest.mark.parametrize("case", PT)
def test_forward_recurrences_bitwise(cuda, case):
    a, b = (float(v) for v in G[f"{case}_ab"])
    p = cj.JacobiParameters(a, b)
    n_max = G[f"{case}_fwd"].shape[1] - 1
    for k, th in enumerate(THETAS):
        assert np.array_equal(cj.jacobi_forward(p, n_max, float(th)), G[f"{case}_fwd"][k]), th
        assert np.array_equal(cj.jacobi_forward_reinsch(p, n_max, float(th), 1), G[f"{case}_rfp"][k]), th
        assert np.array_equal(cj.jacobi_forward_reinsch(p, n_max, float(th), -1), G[f"{case}_rfm"][k]), th


@pytest.mark.gpu
@pytest.mark.parametrize("case", PT)
def test_clenshaw_smith_bitwise(cuda, case):
    a, b = (float(v) for v in G[f"{case}_ab"])
    p = cj.JacobiParameters(a, b)
    c = G[f"{case}_c"]
    for k, th in enumerate(THETAS):
        assert cj.clenshaw_smith(p, c, float(th)) == G[f"{case}_cs"][k], th
        assert cj.clenshaw_smith_reinsch(p, c, float(th), 1) == G[f"{case}_crp"][k], th
        assert cj.clenshaw_smith_reinsch(p, c, float(th), -1) == G[f"{case}_crm"][k], th


@pytest.mark.gpu
@pytest.mark.parametrize("case", EV)
def test_evaluate_expansion_bitwise(cuda, case):
    a, b, n, g = G[f"{case}_abng"]
    p = cj.JacobiParameters(float(a), float(b))
    grid = cj.AngleGrid(int(g))
    c = G[f"{case}_c"]
    ref = G[f"{case}_vals"]
    for v in range(len(c)):
        assert np.array_equal(cj.evaluate_expansion(p, c[v], grid), ref[v])
    # batched device path: every row bit-identical to the single-vector call
    import torch
    out = cj.evaluate_expansion_batched(p, torch.from_numpy(c).to(cuda), grid)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)
    assert np.array_equal(cj.evaluate_expansion_batched(p, c, grid), ref)   # host arrays in/out


@pytest.mark.gpu
def test_evaluate_expansion_batched_large_and_linear(cuda):
    import torch
    p = cj.JacobiParameters(-0.25, 0.4)
    n, g, B = 4095, 8191, 96
    rng = np.random.default_rng(7)
    c = torch.from_numpy(rng.standard_normal((B, n + 1)) / np.arange(1, n + 2)).to(cuda)
    grid = cj.AngleGrid(g)
    v = cj.evaluate_expansion_batched(p, c, grid)
    v2 = cj.evaluate_expansion_batched(p, 2.0 * c[:2] - 0.5 * c[2:4], grid)
    torch.cuda.synchronize()
    lin = 2.0 * v[:2] - 0.5 * v[2:4]
    scale = float(c[:4].abs().sum(dim=1).max())
    assert float((v2 - lin).abs().max()) <= 1e-13 * scale
    # spot rows against the plugin path (bitwise)
    for r in (0, B - 1):
        assert np.array_equal(v[r].cpu().numpy(), cj.evaluate_expansion(p, c[r].cpu().numpy(), grid))


@pytest.mark.gpu
def test_legendre_known_values(cuda):
    # P_2^{(0,0)}(0) = -1/2; sum of P_n(1) = number of terms
    p = cj.JacobiParameters(0.0, 0.0)
    assert cj.jacobi_forward(p, 2, math.pi / 2)[2] == pytest.approx(-0.5, abs=1e-16)
    assert cj.clenshaw_smith_reinsch(p, np.ones(9), 0.0, 1) == pytest.approx(9.0, abs=1e-13)
