"""Ragged batches: many (alpha, beta, N) plans in one execution (configuration 5).

Vectors are grouped by (alpha, beta, N); each group runs the batched
forward / inverse of its own plan pair on a contiguous slice of one packed
device buffer (group-major order, each group a row-major (B_g, N_g + 1)
block).  Groups are spread over several CUDA streams by longest-processing-time
on their modelled cost, and a whole execution can be captured into one CUDA
graph (hundreds of small plans would otherwise be launch bound).  Across GPUs
the same LPT assignment shards whole groups (sharding.lpt_assign), so no plan
is built or generated twice.
"""

from __future__ import annotations

import collections
import concurrent.futures as cf

import numpy as np

from . import engine
from . import sharding
from . import planner
from .planner import DEFAULT_EPS, DEFAULT_M, JacobiParameters


class RaggedPlan:
    """Plans and device layout for a ragged list of (alpha, beta, N), one per vector."""

    def __init__(self, params, m_terms: int = DEFAULT_M, eps: float = DEFAULT_EPS,
                 groups_subset=None, threads: int = 16, device: int | None = None, upload: bool = True):
        params = [(float(a), float(b), int(n)) for a, b, n in params]
        order = collections.OrderedDict()
        for i, key in enumerate(params):
            order.setdefault(key, []).append(i)
        keys = list(order)
        if groups_subset is not None:
            keys = [keys[k] for k in groups_subset]
        self.keys = keys
        self.members = [order[k] for k in keys]        # original vector indices per group
        self.sizes = [len(m) for m in self.members]

        device = engine._current_device() if device is None else device

        def build(key):
            # host plan and device upload in the same worker: the library's
            # plan builds run on per-thread streams and overlap
            a, b, n = key
            p = JacobiParameters(a, b)
            pair = (engine.plan("forward", p, n, m_terms, eps), engine.plan("inverse", p, n, m_terms, eps))
            if upload:
                for tp in pair:
                    tp.device_plan(device)
            return pair

        # per-(alpha, beta) tables at the largest degree first: every plan of
        # the pair then slices them (planner.prewarm)
        top = {}
        for a, b, n in keys:
            top[(a, b)] = max(top.get((a, b), 0), n)
        with cf.ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(lambda kv: planner.prewarm(JacobiParameters(*kv[0]), kv[1], m_terms), top.items()))
            # largest degrees first (their plans take longest: no long tail)
            by_cost = sorted(range(len(keys)), key=lambda i: -keys[i][2])
            built = list(ex.map(build, [keys[i] for i in by_cost]))
            self.plans = [None] * len(keys)
            for i, pair in zip(by_cost, built):
                self.plans[i] = pair
        # packed layout: group g occupies [offsets[g], offsets[g] + B_g (N_g + 1))
        lens = [b * (n + 1) for (a, bb, n), b in zip(keys, self.sizes)]
        self.offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        self.total = int(self.offsets[-1])
        self.coefficients = self.total

    def cost(self, g: int) -> float:
        """Relative cost of group g (recurrence steps and Bluestein points, per vector)."""
        fp, ip = self.plans[g]
        fs, is_ = fp.device_plan().stats(), ip.device_plan().stats()
        return self.sizes[g] * sharding.plan_cost_model(fs.rec_steps_executed, is_.rec_steps_executed,
                                                        fs.fft_points_per_vector,
                                                        is_.fft_points_per_vector)

    def pack(self, vectors) -> np.ndarray:
        """Concatenate per-vector arrays (original order) into the group-major layout."""
        out = np.empty(self.total)
        for g, mem in enumerate(self.members):
            n1 = self.keys[g][2] + 1
            blk = out[self.offsets[g]:self.offsets[g + 1]].reshape(len(mem), n1)
            for r, i in enumerate(mem):
                blk[r] = vectors[i]
        return out

    def group_view(self, buf, g: int):
        n1 = self.keys[g][2] + 1
        return buf[self.offsets[g]:self.offsets[g + 1]].view(self.sizes[g], n1)

    def reserve(self):
        for (fp, ip), b in zip(self.plans, self.sizes):
            fp.device_plan().reserve(b)
            ip.device_plan().reserve(b)

    def execute(self, direction: str, src, dst, streams=None, assignment=None):
        """forward ("forward") or inverse ("inverse") of every group: src/dst are
        packed float64 CUDA tensors.  streams: list of torch streams; assignment:
        per-stream lists of group indices (default: LPT over the streams)."""
        import torch
        cur = torch.cuda.current_stream()
        if streams is None:
            streams = [cur]
        if assignment is None:
            assignment = self.assign(len(streams))
        k = 0 if direction == "forward" else 1
        fn = engine.forward_batched if k == 0 else engine.inverse_batched
        for s in streams:
            if s is not cur:
                s.wait_stream(cur)
        for s, groups in zip(streams, assignment):
            with torch.cuda.stream(s):
                for g in groups:
                    fn(self.plans[g][k], self.group_view(src, g), out=self.group_view(dst, g),
                       check_finite=False)
        for s in streams:
            if s is not cur:
                cur.wait_stream(s)

    def assign(self, nbins: int):
        costs = np.array([self.cost(g) for g in range(len(self.keys))])
        return sharding.lpt_assign(costs, nbins)

    def launches(self) -> int:
        n = 0
        for fp, ip in self.plans:
            n += fp.device_plan().stats().launches_per_execute + ip.device_plan().stats().launches_per_execute
        return n
