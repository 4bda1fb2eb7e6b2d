"""GPU parity at the BASELINE configurations' FULL sizes against the real
reference, run at test time.

The checker is the unmodified reference package (chebjac, Cython backend)
built into oracle/_ref by oracle/build_ref.sh; it travels to the GPU box with
the repository and runs here on the host cores (a process pool, one reference
process per core).  Protocol: forward on the seeded Jacobi
vector; inverse on the REFERENCE's forward output, so each direction is
checked on its own.  Tolerance (north_star): max|dc| <= 1e-12 * ||c||_1 per
vector, float64.

  * config 2: all 64 vectors, N = 2^14 - 1, (alpha, beta) = (-0.25, 0.4)
  * config 3: every 8th of the 8192 vectors (1024), N = 4095, alpha = beta = 1/2
  * config 4: vectors 0 and 15, N = 2^20 - 1, (0.3, -0.45)
  * config 5: one vector of each of the 25 parameter classes at the largest
    degree N = 65535, plus alpha = beta = 1/2 at N = 16383 and 32767 (the
    conditioning-limited classes)
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np
import pytest

import cjt_oracle as O
import paper_1602_02618_b200 as cj

pytestmark = pytest.mark.gpu
TOL = 1e-12

_REF = {}


def _ref_init():
    ch = O.reference_package()
    from chebjac import engine
    _REF["ch"], _REF["engine"], _REF["plans"] = ch, engine, {}


def _ref_pair(task):
    """Reference forward of the seeded vector and inverse of that forward."""
    config, idx, a, b, n = task
    ch, engine, plans = _REF["ch"], _REF["engine"], _REF["plans"]
    key = (a, b, n)
    if key not in plans:
        if len(plans) >= 2:
            plans.clear()
        p = ch.JacobiParameters(a, b)
        plans[key] = (p, engine.plan("forward", p, n), engine.plan("inverse", p, n))
    p, fp, ip = plans[key]
    c = O.seeded_vector(config, idx, n)
    f = engine.forward(fp, ch.jacobi(p, c)).data
    i = engine.inverse(ip, ch.chebyshev(f)).data
    return task, f, i


@pytest.fixture(scope="module")
def refpool():
    if O.reference_package() is None:
        pytest.skip("oracle/_ref (the reference built by oracle/build_ref.sh) is not present")
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    pool = mp.get_context("spawn").Pool(max(1, cores), initializer=_ref_init)
    yield pool
    pool.terminate()


def _check(cuda, refpool, tasks, label, chunksize=1):
    """Run the reference on `tasks` (grouped by parameters) and the CUDA path on
    the same seeded vectors; return the worst forward / inverse deviations."""
    import torch
    t0 = time.perf_counter()
    res = refpool.map(_ref_pair, tasks, chunksize=chunksize)
    t_ref = time.perf_counter() - t0
    groups = {}
    for task, f, i in res:
        groups.setdefault(task[2:], []).append((task, f, i))
    worst_f = worst_i = 0.0
    for (a, b, n), items in groups.items():
        p = cj.JacobiParameters(a, b)
        fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
        c = np.stack([O.seeded_vector(t[0], t[1], n) for t, _, _ in items])
        rf = np.stack([f for _, f, _ in items])
        ri = np.stack([i for _, _, i in items])
        got_f = cj.forward_batched(fp, torch.from_numpy(c).to(cuda)).cpu().numpy()
        got_i = cj.inverse_batched(ip, torch.from_numpy(rf).to(cuda)).cpu().numpy()
        ef = np.max(np.abs(got_f - rf), axis=1) / np.abs(c).sum(axis=1)
        ei = np.max(np.abs(got_i - ri), axis=1) / np.abs(rf).sum(axis=1)
        worst_f, worst_i = max(worst_f, float(ef.max())), max(worst_i, float(ei.max()))
        bad = [(items[k][0], float(ef[k]), float(ei[k])) for k in range(len(items))
               if not (ef[k] <= TOL and ei[k] <= TOL)]
        assert not bad, (label, bad[:5])
    print(f"{label}: {len(tasks)} vectors, worst forward {worst_f:.3e}, inverse {worst_i:.3e} "
          f"(x ||c||_1; reference {t_ref:.1f} s on the host pool)")
    return worst_f, worst_i


def test_config2_all_64_vectors(cuda, refpool):
    tasks = [(2, v, -0.25, 0.4, 2**14 - 1) for v in range(64)]
    _check(cuda, refpool, tasks, "config2")


def test_config3_every_8th_vector(cuda, refpool):
    tasks = [(3, v, 0.5, 0.5, 4095) for v in range(0, 8192, 8)]
    _check(cuda, refpool, tasks, "config3", chunksize=8)


def test_config4_full_degree(cuda, refpool):
    tasks = [(4, v, 0.3, -0.45, 2**20 - 1) for v in (0, 15)]
    _check(cuda, refpool, tasks, "config4")


def _config5_tasks():
    draws = O.config5_draws(4096)
    first = {}
    for i, d in enumerate(draws):
        first.setdefault(d, i)
    tasks = []
    for a in O.CONFIG5_PARAMS:
        for b in O.CONFIG5_PARAMS:
            key = (a, b, 65535)
            # the seeded stream's own vector of this class when config 5 draws
            # one, else a vector index past the 4096 drawn
            tasks.append((5, first.get(key, 4096 + len(tasks)), a, b, 65535))
    for n in (16383, 32767):
        tasks.append((5, first.get((0.5, 0.5, n), 5000 + n), 0.5, 0.5, n))
    # most expensive first (alpha = beta = 1/2 is a pure O(N^2) recurrence)
    tasks.sort(key=lambda t: -(t[4] * (50 if t[2] == t[3] == 0.5 else 1)))
    return tasks


def test_config5_largest_degree_every_class(cuda, refpool):
    _check(cuda, refpool, _config5_tasks(), "config5 N=65535 x 25 classes + (1/2,1/2) ladder")
