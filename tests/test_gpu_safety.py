"""GPU: shared plans under concurrency (SPEC.md:571 -- plans are immutable and
shareable across threads), CUDA-graph safety of plan growth, batches beyond
the 65535 per-launch grid limit, and side-stream allocation."""
import threading

import numpy as np
import pytest

import cjt_oracle as O
import paper_1602_02618_b200 as cj

pytestmark = pytest.mark.gpu


def test_one_plan_two_host_threads_different_batches(cuda):
    """Two host threads execute ONE plan pair concurrently, each on its own
    stream and with its own (different, growing) batch sizes; every result
    equals the single-threaded execution of the same batch."""
    import torch
    a, b, n = -0.25, 0.4, 1023
    p = cj.JacobiParameters(a, b)
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    c = torch.from_numpy(np.stack([O.seeded_vector(2, v, n) for v in range(40)])).to(cuda)
    sizes = {0: [3, 17, 40, 9], 1: [40, 1, 24, 33]}
    want = {}
    for bs in {s for v in sizes.values() for s in v}:
        x = c[:bs].contiguous()
        want[bs] = cj.inverse_batched(ip, cj.forward_batched(fp, x)).clone()
    torch.cuda.synchronize()
    got, errors = {}, []

    def worker(t):
        try:
            s = torch.cuda.Stream(cuda)
            with torch.cuda.stream(s):
                for rep in range(3):
                    for bs in sizes[t]:
                        x = c[:bs].contiguous()
                        y = cj.inverse_batched(ip, cj.forward_batched(fp, x))
                        s.synchronize()
                        got[(t, rep, bs)] = y.clone()
        except Exception as e:   # surfaced below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(t,)) for t in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errors, errors
    torch.cuda.synchronize()
    for (t, rep, bs), y in got.items():
        scale = c[:bs].abs().sum(dim=1)
        d = ((y - want[bs]).abs().max(dim=1).values / scale).max()
        # a batch's schedule can depend on the reserved size: rounding only
        assert float(d) <= 1e-14, (t, rep, bs, float(d))


def test_growth_after_graph_capture_is_an_error(cuda):
    """A plan recorded into a CUDA graph keeps its buffers: executing it with
    a larger batch afterwards fails loudly instead of freeing memory the graph
    still uses; batches up to the captured size keep working."""
    import torch
    p = cj.JacobiParameters(0.0, 0.25)
    n = 255
    fp = cj.plan("forward", p, n)
    x = torch.from_numpy(np.stack([O.seeded_vector(5, v, n) for v in range(8)])).to(cuda)
    y = torch.empty_like(x)
    s = torch.cuda.Stream(cuda)
    with torch.cuda.stream(s):
        cj.forward_batched(fp, x, out=y)
    s.synchronize()
    ref = y.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        cj.forward_batched(fp, x, out=y, check_finite=False)   # no host sync while capturing
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
    big = torch.from_numpy(np.stack([O.seeded_vector(5, v, n) for v in range(64)])).to(cuda)
    with pytest.raises(ValueError, match="captured CUDA graph"):
        cj.forward_batched(fp, big)
    small = cj.forward_batched(fp, x[:4].contiguous())
    torch.cuda.synchronize()
    assert float((small - ref[:4]).abs().max()) <= 1e-15 * float(x[:4].abs().sum(dim=1).max())
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, ref)


def test_batch_beyond_grid_limit(cuda):
    """B > 65535 vectors in one call (per-vector grid dimensions are capped at
    65535: the library executes in chunks)."""
    import torch
    a, b, n = 0.25, -0.2, 15
    p = cj.JacobiParameters(a, b)
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    B = 70001
    rng = np.random.default_rng(7)
    c = rng.standard_normal((B, n + 1))
    x = torch.from_numpy(c).to(cuda)
    f = cj.forward_batched(fp, x)
    i = cj.inverse_batched(ip, f).cpu().numpy()
    f = f.cpu().numpy()
    for v in (0, 65534, 65535, 65536, B - 1):
        rf = O.oracle_forward(a, b, c[v])
        assert O.parity(f[v], rf, c[v]) <= 1e-13
        assert O.parity(i[v], O.oracle_inverse(a, b, f[v]), f[v]) <= 1e-13
    # host path (cjt_execute_host) chunks the same way
    fh = cj.forward_batched(fp, c)
    assert np.max(np.abs(fh - f)) <= 1e-15 * np.abs(c).sum(axis=1).max()


def test_side_stream_outputs_and_shift_temporaries(cuda):
    """Outputs / temporaries allocated for kernels on a non-current stream are
    recorded on that stream (no allocator reuse while they are in flight)."""
    import torch
    a, b, n = 1.3, -0.6, 511      # outside the core: shifts in and out
    p = cj.JacobiParameters(a, b)
    c = torch.from_numpy(np.stack([O.seeded_vector(5, v, n) for v in range(4)])).to(cuda)
    s = torch.cuda.Stream(cuda)
    s.wait_stream(torch.cuda.current_stream(cuda))
    target = cj.JacobiParameters(-0.3, 0.2)
    ys = []
    for _ in range(3):
        ys.append(cj.jacobi_to_jacobi_batched(p, c, target, stream=s))
        # churn the allocator on the current stream while s is busy
        _ = [torch.empty(1 << 16, dtype=torch.float64, device=cuda).fill_(1.0) for _ in range(8)]
    s.synchronize()
    ref = cj.jacobi_to_jacobi_batched(p, c, target)
    torch.cuda.synchronize()
    for y in ys:
        assert torch.equal(y, ref)
