"""GPU: the alpha = beta = 1/2 exact-expansion path (planner.half_exact_*,
csrc/cjt_half.cu, csrc/cjt_host.cpp) against the reference's outputs and
against the recurrence layout the reference itself runs ($CJT_HALF_EXACT=0).

Tolerance (north_star): 1e-12 * ||c||_1 per vector; the measured margin is
reported by the full-size tests (tests/test_gpu_fullsize.py)."""
import numpy as np
import pytest

import cjt_oracle as O
import paper_1602_02618_b200 as cj
from conftest import load_golden

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _run(p, n, c, monkeypatch, exact: bool):
    import torch
    monkeypatch.setenv("CJT_HALF_EXACT", "1" if exact else "0")
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    assert (fp.host.half_k is not None) == exact
    x = torch.from_numpy(c).cuda()
    f = cj.forward_batched(fp, x)
    i = cj.inverse_batched(ip, f)
    return f.cpu().numpy(), i.cpu().numpy()


@pytest.mark.parametrize("name", ["cfg3_full", "cfg5_e"])
def test_half_exact_vs_reference_goldens(cuda, name, monkeypatch):
    import torch
    g = load_golden(name)
    n = int(g["n"])
    p = cj.JacobiParameters(0.5, 0.5)
    monkeypatch.setenv("CJT_HALF_EXACT", "1")
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    f = cj.forward_batched(fp, torch.from_numpy(g["c"]).to(cuda)).cpu().numpy()
    i = cj.inverse_batched(ip, torch.from_numpy(g["fwd"]).to(cuda)).cpu().numpy()
    for v in range(g["c"].shape[0]):
        assert O.parity(f[v], g["fwd"][v], g["c"][v]) <= 1e-15
        assert O.parity(i[v], g["inv"][v], g["fwd"][v]) <= 1e-13


@pytest.mark.parametrize("n", [1, 2, 3, 4, 17, 255, 1000, 2047, 4095, 4096, 8191, 12288, 16383])
def test_half_exact_vs_recurrence_layout(cuda, n, monkeypatch):
    """Same inputs through both device paths (the recurrence layout is the
    reference's own algorithm, parity-pinned elsewhere), and the oracle."""
    p = cj.JacobiParameters(0.5, 0.5)
    batch = 3 if n < 4000 else 2
    c = np.stack([O.seeded_vector(5, v, n) for v in range(batch)])
    f1, i1 = _run(p, n, c, monkeypatch, exact=True)
    f0, i0 = _run(p, n, c, monkeypatch, exact=False)
    l1c = np.abs(c).sum(axis=1)
    l1f = np.abs(f0).sum(axis=1)
    assert np.all(np.max(np.abs(f1 - f0), axis=1) <= 1e-14 * l1c)
    assert np.all(np.max(np.abs(i1 - i0), axis=1) <= TOL * l1f)
    for v in (0, batch - 1):
        rf = O.oracle_forward(0.5, 0.5, c[v])
        assert O.parity(f1[v], rf, c[v]) <= 1e-14
        assert O.parity(i1[v], O.oracle_inverse(0.5, 0.5, f1[v]), f1[v]) <= TOL


def test_half_exact_large_batch_and_host_api(cuda, monkeypatch):
    """Many vectors (multi-tile scan, stream-K chirp-z) and the single-vector
    host API (engine.forward / inverse) on the exact path."""
    import torch
    monkeypatch.setenv("CJT_HALF_EXACT", "1")
    p = cj.JacobiParameters(0.5, 0.5)
    n = 4095
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    c = np.stack([O.seeded_vector(3, v, n) for v in range(300)])
    f = cj.forward_batched(fp, torch.from_numpy(c).to(cuda))
    i = cj.inverse_batched(ip, f).cpu().numpy()
    f = f.cpu().numpy()
    for v in (0, 137, 299):
        assert O.parity(f[v], O.oracle_forward(0.5, 0.5, c[v]), c[v]) <= 1e-14
        assert O.parity(i[v], c[v], c[v]) <= 1e-12                 # round trip
    one = cj.forward(fp, cj.jacobi(p, c[137]))
    assert np.array_equal(one.data, f[137])
    back = cj.inverse(ip, cj.chebyshev(f[137]))
    assert np.max(np.abs(back.data - i[137])) <= 1e-15 * np.abs(f[137]).sum()


@pytest.mark.parametrize("n,batch", [(7, 3), (15, 2), (63, 9), (255, 5), (1023, 300), (4095, 257), (8191, 40)])
def test_tcgen05_inverse_matches_cublas_path(cuda, n, batch, monkeypatch):
    """The tcgen05 correction GEMM with its fused fp64 epilogue (cjt_umma.cu)
    against the cuBLAS GEMM + separate finish on the same plan: the two differ
    only in the fp32 accumulation order of a ~1e-12 ||t||_1 correction."""
    import torch
    p = cj.JacobiParameters(0.5, 0.5)
    ip = cj.plan("inverse", p, n)
    assert ip.host.half_gemm
    t = torch.from_numpy(np.stack([O.seeded_vector(3, v, n) for v in range(batch)])).to(cuda)
    monkeypatch.delenv("CJT_HALF_CUBLAS", raising=False)
    a = cj.inverse_batched(ip, t).cpu().numpy()
    monkeypatch.setenv("CJT_HALF_CUBLAS", "1")
    b = cj.inverse_batched(ip, t).cpu().numpy()
    l1 = np.abs(t.cpu().numpy()).sum(axis=1)
    assert np.all(np.max(np.abs(a - b), axis=1) <= 1e-16 * l1)


@pytest.mark.parametrize("n", [255, 4095, 8191, 16383])
def test_half_forward_independent_of_batch(cuda, n):
    """The exact forward picks its kernel by layout only and gives each vector
    one warp (or one chunk chain) whatever the batch: a vector's result is
    bit-identical in batches of 1, 5, 150 and 2000."""
    import torch
    p = cj.JacobiParameters(0.5, 0.5)
    fp = cj.plan("forward", p, n)
    c = torch.from_numpy(np.stack([O.seeded_vector(3, v, n) for v in range(2000)])).to(cuda)
    full = cj.forward_batched(fp, c)
    for b in (1, 5, 150):
        part = cj.forward_batched(fp, c[:b].contiguous())
        assert torch.equal(part, full[:b])


def test_tcgen05_inverse_tile_width_invariance(cuda, monkeypatch):
    """Small batches run the tcgen05 GEMM with 128-vector tiles (more CTA
    pairs busy), large ones with 256: same K order and epilogue, so the
    results are bit-identical."""
    import torch
    p = cj.JacobiParameters(0.5, 0.5)
    ip = cj.plan("inverse", p, 4095)
    t = torch.from_numpy(np.stack([O.seeded_vector(3, v, 4095) for v in range(300)])).to(cuda)
    monkeypatch.delenv("CJT_UMMA_BN256", raising=False)
    a = cj.inverse_batched(ip, t)
    monkeypatch.setenv("CJT_UMMA_BN256", "1")
    b = cj.inverse_batched(ip, t)
    assert torch.equal(a, b)


@pytest.mark.parametrize("n,batch", [(1023, 37), (4095, 300), (4095, 1100)])
def test_tcgen05_inverse_overlapped_conversion(cuda, n, batch, monkeypatch):
    """$CJT_HALF_OVERLAP=1: the fp64 -> bf16 conversion runs concurrently with
    the tcgen05 GEMM (programmatic dependent launch; the GEMM's TMA producers
    wait on per-128-vector progress counters).  Same arithmetic, so the
    results are bit-identical to the convert-then-multiply default, also on
    repeated executions (the counters are reset per execution)."""
    import torch
    p = cj.JacobiParameters(0.5, 0.5)
    ip = cj.plan("inverse", p, n)
    t = torch.from_numpy(np.stack([O.seeded_vector(3, v, n) for v in range(batch)])).to(cuda)
    monkeypatch.delenv("CJT_HALF_OVERLAP", raising=False)
    a = cj.inverse_batched(ip, t)
    monkeypatch.setenv("CJT_HALF_OVERLAP", "1")
    for _ in range(3):
        b = cj.inverse_batched(ip, t)
        assert torch.equal(a, b)
