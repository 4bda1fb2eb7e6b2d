"""Multi-GPU batch sharding: pure host logic, plus world_size-2 gloo runs of
the collective helpers and of bench.py's per-rank path (contiguous slice of the
fixed seeded batch, local forward+inverse with the CPU oracle standing in for
the device, in-order reassembly, max-reduced timing)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_1602_02618_b200 import sharding


def test_contiguous_slices_partition():
    for n in (1, 7, 64, 8192):
        for world in (1, 2, 3, 8):
            spans = [sharding.contiguous_slice(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_lpt_balances_ragged_costs():
    rng = np.random.default_rng(0)
    costs = rng.choice([1e6, 1e8, 4.7e10], size=200, p=[0.6, 0.35, 0.05])
    bins = sharding.lpt_assign(costs, 8)
    assert sorted(i for b in bins for i in b) == list(range(200))
    loads = [costs[b].sum() for b in bins]
    assert max(loads) <= max(costs.max(), 1.2 * costs.sum() / 8)


def test_lpt_keeps_groups_together():
    costs = np.ones(12)
    groups = [[0, 1, 2], [3, 4], [5], [6, 7, 8, 9], [10, 11]]
    bins = sharding.lpt_assign(costs, 2, groups)
    for g in groups:
        assert sum(all(i in b for i in g) for b in bins) == 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench_rank(rank, world, port, q):
    """bench.py's per-rank data path with the CPU oracle standing in for the
    device: contiguous slice of the fixed seeded batch, local forward+inverse,
    reassembly in global vector order (sharding.gather_rows), max-reduced time."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    import bench
    import cjt_oracle as O
    config, n, total = 3, 63, 7
    lo, hi, c = bench.shard_batch(config, n, total, world, rank)
    a = b = 0.5
    cheb = np.stack([O.oracle_forward(a, b, v) for v in c])
    back = np.stack([O.oracle_inverse(a, b, v) for v in cheb])
    ct, bt = torch.from_numpy(c), torch.from_numpy(back)
    full_c = sharding.gather_rows(ct, total, world, rank)
    full_cheb = sharding.gather_rows(torch.from_numpy(cheb), total, world, rank)
    stats = sharding.gather_rows(bench.roundtrip_stats(ct, bt), total, world, rank)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((lo, hi, full_c.numpy(), full_cheb.numpy(), stats.numpy(), t.item()))
    dist.destroy_process_group()


def test_two_rank_gloo_bench_rank_logic():
    import cjt_oracle as O
    ctx = tmp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    lo, hi, full_c, full_cheb, stats, tmax = q.get()
    assert (lo, hi) == (0, 4)          # rank 0 owns the first ceil(7/2) vectors
    # disjoint, complete coverage of the seeded stream, reassembled in order
    want = np.stack([O.seeded_vector(3, v, 63) for v in range(7)])
    assert np.array_equal(full_c, want)
    assert np.array_equal(full_cheb, np.stack([O.oracle_forward(0.5, 0.5, v) for v in want]))
    assert stats.shape == (7, 1) and float(stats.max()) < 1e-12
    assert tmax == 2.0


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    n = 64
    lo, hi = sharding.contiguous_slice(n, world, rank)
    mine = torch.arange(lo, hi, dtype=torch.float64)
    # each rank owns a disjoint slice; gather proves full coverage, no overlap
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([hi - lo]))
    buf = [torch.zeros(int(s.item()), dtype=torch.float64) for s in sizes]
    dist.all_gather(buf, mine)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((torch.cat(buf).tolist(), t.item()))
    dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    ctx = tmp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    values, tmax = q.get()
    assert values == list(range(64)) and tmax == 2.0
