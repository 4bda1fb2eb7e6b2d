"""GPU parity: the CUDA path vs the oracle and the reference's golden outputs.

Tolerance (north_star): max|dc| <= 1e-12 * ||c||_1 per vector, float64,
for the forward and for the inverse applied to the reference's forward output.
"""
import numpy as np
import pytest

import cjt_oracle as O
import paper_1602_02618_b200 as cj
from conftest import load_golden

pytestmark = pytest.mark.gpu
TOL = 1e-12

GOLDEN_CASES = ["cfg1", "cfg2_small", "cfg2_full", "cfg3_full", "cfg4_small", "cfg5_a", "cfg5_b",
                "cfg5_c", "cfg5_d", "cfg5_e", "tiny", "edge_n1"]


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_golden_batched(cuda, name):
    import torch
    g = load_golden(name)
    a, b, n = float(g["alpha"]), float(g["beta"]), int(g["n"])
    p = cj.JacobiParameters(a, b)
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    got_f = cj.forward_batched(fp, torch.from_numpy(g["c"]).to(cuda)).cpu().numpy()
    got_i = cj.inverse_batched(ip, torch.from_numpy(g["fwd"]).to(cuda)).cpu().numpy()
    for v in range(g["c"].shape[0]):
        ef = O.parity(got_f[v], g["fwd"][v], g["c"][v])
        ei = O.parity(got_i[v], g["inv"][v], g["fwd"][v])
        assert ef <= TOL, (name, v, "forward", ef)
        assert ei <= TOL, (name, v, "inverse", ei)


@pytest.mark.parametrize("name", ["cfg1", "cfg2_small", "tiny", "edge_n1"])
def test_golden_single_vector_api(cuda, name):
    g = load_golden(name)
    a, b, n = float(g["alpha"]), float(g["beta"]), int(g["n"])
    p = cj.JacobiParameters(a, b)
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    f = cj.forward(fp, cj.jacobi(p, g["c"][0]))
    i = cj.inverse(ip, cj.chebyshev(g["fwd"][0]))
    assert f.basis == cj.CHEBYSHEV and i.basis == cj.JACOBI and i.params == p
    assert O.parity(f.data, g["fwd"][0], g["c"][0]) <= TOL
    assert O.parity(i.data, g["inv"][0], g["fwd"][0]) <= TOL


@pytest.mark.parametrize("batch", [1, 17, 24, 30, 40, 70, 129, 300])
def test_batch_tiles_vs_oracle(cuda, batch):
    """Every vector-tile width (16/24/32/64/128) and ragged batch tails."""
    import torch
    a, b, n = 0.25, -0.2, 1023
    p = cj.JacobiParameters(a, b)
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    c = np.stack([O.seeded_vector(5, v, n) for v in range(batch)])
    f = cj.forward_batched(fp, torch.from_numpy(c).to(cuda)).cpu().numpy()
    i = cj.inverse_batched(ip, torch.from_numpy(f).to(cuda)).cpu().numpy()
    for v in sorted({0, batch // 2, batch - 1}):
        rf = O.oracle_forward(a, b, c[v])
        ri = O.oracle_inverse(a, b, f[v])
        assert O.parity(f[v], rf, c[v]) <= TOL
        assert O.parity(i[v], ri, f[v]) <= TOL


@pytest.mark.parametrize("batch", [20, 28])
def test_vector_tile_width_invariance(cuda, batch):
    """A vector's result does not depend on the tile width it ran in (24 / 32
    vs 16): the contraction order per output element is the same."""
    import torch
    a, b, n = 0.5, 0.5, 1023      # pure recurrence: K = 0
    p = cj.JacobiParameters(a, b)
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    c = torch.from_numpy(np.stack([O.seeded_vector(3, v, n) for v in range(batch)])).to(cuda)
    f = cj.forward_batched(fp, c)
    i = cj.inverse_batched(ip, f)
    f1 = cj.forward_batched(fp, c[:8].contiguous())
    i1 = cj.inverse_batched(ip, f[:8].contiguous())
    torch.cuda.synchronize()
    scale = float(c[:8].abs().sum(dim=1).max())
    assert float((f[:8] - f1).abs().max()) <= 1e-15 * scale
    assert float((i[:8] - i1).abs().max()) <= 1e-15 * scale


@pytest.mark.parametrize("ab,n", [((0.0, 0.0), 1023), ((0.5, 0.5), 4095), ((-0.45, -0.45), 2047),
                                  ((0.25, 0.25), 8191), ((0.0, 0.0), 1), ((0.5, 0.5), 2),
                                  ((-0.2, -0.2), 3)])
def test_parity_folding_alpha_eq_beta(cuda, monkeypatch, ab, n):
    """alpha = beta: the forward recurrence runs parity-folded (rows i and G-i
    from one generated row, even / odd degrees contracted separately); it
    agrees with the unfolded contraction and the oracle.  The opt-in folded
    inverse ($CJT_FOLD_INVERSE=1) stays within the transform tolerance."""
    import torch
    a, b = ab
    p = cj.JacobiParameters(a, b)
    c = np.stack([O.seeded_vector(3, v, n) for v in range(20)])
    x = torch.from_numpy(c).to(cuda)
    scale = np.abs(c).sum(axis=1)

    def run(direction, inp, env):
        for k in ("CJT_FOLD", "CJT_FOLD_INVERSE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        tp = cj.plan(direction, p, n)
        f = cj.forward_batched if direction == "forward" else cj.inverse_batched
        out = f(tp, inp)
        torch.cuda.synchronize()
        return out

    f_fold = run("forward", x, {})
    f_flat = run("forward", x, {"CJT_FOLD": "0"})
    d = (f_fold - f_flat).abs().max(dim=1).values.cpu().numpy()
    assert np.all(d <= 1e-14 * scale)
    for v in (0, 19):
        assert O.parity(f_fold[v].cpu().numpy(), O.oracle_forward(a, b, c[v]), c[v]) <= TOL
    i_fold = run("inverse", f_flat, {"CJT_FOLD_INVERSE": "1"})
    fh = f_flat.cpu().numpy()
    for v in (0, 19):
        assert O.parity(i_fold[v].cpu().numpy(), O.oracle_inverse(a, b, fh[v]), fh[v]) <= TOL


def test_parity_folding_full_size_forward(cuda, monkeypatch):
    """Folded forward at the largest ragged-config size, alpha = beta = 1/2,
    N = 65535 (pure recurrence): equal to the unfolded contraction to 1e-14."""
    import torch
    p = cj.JacobiParameters(0.5, 0.5)
    n = 65535
    c = torch.from_numpy(np.stack([O.seeded_vector(5, v, n) for v in range(4)])).to(cuda)
    monkeypatch.delenv("CJT_FOLD", raising=False)
    f_fold = cj.forward_batched(cj.plan("forward", p, n), c)
    monkeypatch.setenv("CJT_FOLD", "0")
    f_flat = cj.forward_batched(cj.plan("forward", p, n), c)
    torch.cuda.synchronize()
    d = (f_fold - f_flat).abs().max(dim=1).values / c.abs().sum(dim=1)
    assert float(d.max()) <= 1e-14


def test_cluster_chirpz_path_golden():
    """$CJT_CLUSTER=1 (opt-in): untiled Bluestein products of 2^14..2^17 points
    run in thread-block clusters over distributed shared memory; tiled products
    keep the multi-pass kernels.  Checked in a child process (the switch is read
    once per process) against the reference's golden outputs of config 2."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path[:0] = [%r, %r, %r]\n"
        "import numpy as np, torch\n"
        "import cjt_oracle as O, paper_1602_02618_b200 as cj\n"
        "from conftest import load_golden\n"
        "worst = 0.0\n"
        "for name in ('cfg2_full', 'cfg5_d'):\n"
        "    g = load_golden(name)\n"
        "    p = cj.JacobiParameters(float(g['alpha']), float(g['beta'])); n = int(g['n'])\n"
        "    fp, ip = cj.plan('forward', p, n), cj.plan('inverse', p, n)\n"
        "    f = cj.forward_batched(fp, torch.from_numpy(g['c']).cuda()).cpu().numpy()\n"
        "    i = cj.inverse_batched(ip, torch.from_numpy(g['fwd']).cuda()).cpu().numpy()\n"
        "    for v in range(g['c'].shape[0]):\n"
        "        worst = max(worst, O.parity(f[v], g['fwd'][v], g['c'][v]), O.parity(i[v], g['inv'][v], g['c'][v]))\n"
        "print('WORST', worst)\n"
    ) % (root, os.path.join(root, "oracle"), os.path.join(root, "tests"))
    env = dict(os.environ, CJT_CLUSTER="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    worst = float(out.stdout.strip().split("WORST")[-1])
    assert worst <= TOL, worst
