"""Benchmark: forward + inverse CJT throughput (coefficients/s, fp64) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = forward then inverse transform of one batch of seeded synthetic
coefficient vectors; value = coefficients pushed through
fwd+inv per second over all ranks.  Default workload: BASELINE.json configs[1]
(alpha=-0.25, beta=0.4, N=2^14-1, 64 vectors per GPU; weak scaling across
GPUs).  Inputs are resident in HBM for `value`; `e2e` goes through the public
batched API with pinned host arrays (H2D and D2H inside the timed region).
`--impl reference` times the unmodified reference (oracle/_ref, Cython
backend) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

METRIC = "CJT coeffs/s (fp64 fwd+inv)"
UNIT = "coeffs/s"
NOMINAL_FP64_TFLOPS = 37.2

WORKLOADS = {
    1: dict(alpha=0.0, beta=0.0, n=1023, batch=1, env="1/(n+1)"),
    2: dict(alpha=-0.25, beta=0.4, n=2**14 - 1, batch=64, env="(n+1)^-1.5"),
    3: dict(alpha=0.5, beta=0.5, n=4095, batch=8192, env="0.999^n"),
    4: dict(alpha=0.3, beta=-0.45, n=2**20 - 1, batch=16, env="1/(n+1)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None, help="vectors per GPU (default: the config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (1 warm-up + steps)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


# ---------------------------------------------------------------------------
# CPU side: the reference (oracle/_ref) or, failing that, the oracle port


_W = {}


def _worker_init(alpha, beta, n, config):
    import cjt_oracle as O
    ref = O.reference_package()
    _W["O"] = O
    _W["config"] = config
    if ref is not None:
        from chebjac import engine
        p = ref.JacobiParameters(alpha, beta)
        fp, ip = engine.plan("forward", p, n), engine.plan("inverse", p, n)
        _W["run"] = lambda c: engine.inverse(ip, engine.forward(fp, ref.jacobi(p, c))).data
        _W["kind"] = "reference"
    else:
        _W["run"] = lambda c: O.oracle_inverse(alpha, beta, O.oracle_forward(alpha, beta, c))
        _W["kind"] = "port"


def _worker_run(task):
    config, n, idx = task
    O = _W["O"]
    c = O.seeded_vector(config, idx, n)
    t = time.perf_counter()
    _W["run"](c)
    return time.perf_counter() - t, _W["kind"]


def _cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class CpuArm:
    """Process pool, one worker per host core, plans built once per worker."""

    def __init__(self, wl, config):
        self.cores = _cpu_cores()
        self.wl = wl
        self.config = config
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(self.cores, initializer=_worker_init,
                             initargs=(wl["alpha"], wl["beta"], wl["n"], config))
        # warm every worker (plans + first call), estimate per-vector seconds
        res = self.pool.map(_worker_run, [(config, wl["n"], i) for i in range(self.cores)], chunksize=1)
        self.kind = res[0][1]
        self.sec_per_vec = statistics.median(r[0] for r in res)

    def sample(self, nvec, offset=0):
        tasks = [(self.config, self.wl["n"], offset + i) for i in range(nvec)]
        t = time.perf_counter()
        self.pool.map(_worker_run, tasks, chunksize=1)
        return time.perf_counter() - t

    def close(self):
        self.pool.terminate()


def sample_size(arm, target_cpu_seconds):
    n = max(arm.cores, int(round(target_cpu_seconds / max(arm.sec_per_vec, 1e-6))))
    return int(math.ceil(n / arm.cores) * arm.cores)


def config_json(wl, config, batch, world, scaling):
    return {"workload": f"config{config}: fwd+inv CJT alpha={wl['alpha']} beta={wl['beta']} "
                        f"N={wl['n']} batch={batch}/GPU c_n=z_n*{wl['env']}",
            "alpha": wl["alpha"], "beta": wl["beta"], "N": wl["n"], "global_batch": batch * world,
            "batch_per_gpu": batch, "m_terms": 7, "parallelism": f"batch-sharded x{world}",
            "l2": "flushed between timed steps (256 MiB write)"}


def run_reference(args, wl):
    rank, _, world = dist_env()
    if rank != 0:
        return
    arm = CpuArm(wl, args.config)
    nvec = sample_size(arm, target_cpu_seconds=3.0 * arm.cores)
    for w in range(max(0, args.warmup - 1)):
        arm.sample(arm.cores, offset=10_000 + w * arm.cores)
    times = [arm.sample(nvec, offset=k * nvec) for k in range(args.steps)]
    arm.close()
    total = sum(times)
    value = nvec * (wl["n"] + 1) * args.steps / total
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md 8(d))",
        "config": config_json(wl, args.config, wl["batch"], 1, "weak"), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": arm.cores, "kind": arm.kind,
                         "sample": f"{nvec} vectors fwd+inv per step (bounded sample of config{args.config}), "
                                   f"multiprocessing over {arm.cores} host cores, plans untimed"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for k, nm in enumerate(names):
                    if r[3 + k].lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU arm


def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    import paper_1602_02618_b200 as cj
    from paper_1602_02618_b200 import _native as nat
    import cjt_oracle as O

    rank, local, world = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    batch = args.batch or wl["batch"]
    n1 = wl["n"] + 1
    p = cj.JacobiParameters(wl["alpha"], wl["beta"])
    fp = cj.plan("forward", p, wl["n"])
    ip = cj.plan("inverse", p, wl["n"])
    # weak scaling: rank r owns vectors [r*batch, (r+1)*batch) of the seeded stream
    c_host = np.stack([O.seeded_vector(args.config, rank * batch + v, wl["n"]) for v in range(batch)])
    c_dev = torch.from_numpy(c_host).to(dev)
    cheb = torch.empty_like(c_dev)
    back = torch.empty_like(c_dev)
    fdp, idp = fp.device_plan(local), ip.device_plan(local)
    fdp.reserve(batch)
    idp.reserve(batch)
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        cj.forward_batched(fp, c_dev, out=cheb, check_finite=False)
        cj.inverse_batched(ip, cheb, out=back, check_finite=False)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize(dev)
    launches = fdp.stats().launches_per_execute + idp.stats().launches_per_execute

    def timed(fn, k):
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for i in range(k):
            flush.zero_()
            starts[i].record(stream)
            fn()
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        return [s.elapsed_time(e) for s, e in zip(starts, ends)]

    with ClockSampler(local) as clk:
        step_ms = timed(step, args.steps)
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * batch * n1 / (ms_per_step * 1e-3)

    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_per_step}), flush=True)
        return

    # correctness spot check of the timed output against the oracle (not timed)
    chk = None
    if rank == 0:
        v = 0
        ref_f = O.oracle_forward(wl["alpha"], wl["beta"], c_host[v]) if wl["n"] < 70000 else None
        if ref_f is not None:
            ref_i = O.oracle_inverse(wl["alpha"], wl["beta"], ref_f)
            chk = {"fwd": O.parity(cheb[v].cpu().numpy(), ref_f, c_host[v]),
                   "inv": O.parity(back[v].cpu().numpy(), ref_i, c_host[v]),
                   "roundtrip": O.parity(back[v].cpu().numpy(), c_host[v], c_host[v])}

    # per-stage timing -> dominant kernel and its roofline
    L = nat.lib()
    st = stream.cuda_stream
    stages = {}
    for name, dp, src, dst in (("fwd", fdp, c_dev, cheb), ("inv", idp, cheb, back)):
        for sname, mask in (("rec", nat.STAGE_REC), ("blocks", nat.STAGE_BLOCKS), ("edge", nat.STAGE_EDGE)):
            def fn(dp=dp, src=src, dst=dst, mask=mask):
                nat.check(L.cjt_execute_stage(dp.handle, src.data_ptr(), dst.data_ptr(), batch, mask, st))
            fn()
            ms = timed(fn, max(3, min(args.steps, 10)))
            stages[f"{name}_{sname}"] = statistics.median(ms)
    # restore valid outputs
    step()
    torch.cuda.synchronize(dev)
    peak = ctypes_peak(L, st)
    fst, ist = fdp.stats(), idp.stats()
    rec_flops = {"fwd_rec": 2.0 * fst.rec_steps * batch + 5.0 * fst.rec_steps,
                 "inv_rec": 2.0 * ist.rec_steps * batch + 5.0 * ist.rec_steps}
    # nominal 5 L log2 L flop per complex FFT of length L (2 per Bluestein) per term per vector
    fft_flops = {"fwd": 2.5 * fst.fft_points_per_vector * batch, "inv": 2.5 * ist.fft_points_per_vector * batch}
    dom = max(stages, key=stages.get)
    if dom.endswith("rec"):
        flops = rec_flops[dom]
        kern = "k_rec_forward (K1)" if dom.startswith("fwd") else "k_rec_inverse (K2)"
        unit_note = "2 flop per (point, degree, vector) contraction + 5 flop per (point, degree) generation"
    else:
        d = dom.split("_")[0]
        share = stages[dom] / (stages[f"{d}_blocks"] + stages[f"{d}_edge"])
        flops = fft_flops[d] * share
        kern = "k_chirpz_* (Bluestein chirp-z)"
        unit_note = "5 L log2 L flop per complex FFT, 2 FFTs per chirp-z term"
    achieved = flops / (stages[dom] * 1e-3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(dom)
        except (ValueError, OSError):
            traffic = None
    roofline = {"bound": "fp64", "kernel": kern, "stage": dom, "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak if peak else None, "traffic": traffic,
                "peak_source": "measured on this GPU by cjt_probe_fp64_peak (DFMA chains)",
                "nominal_peak": NOMINAL_FP64_TFLOPS, "flops_model": unit_note,
                "stage_ms": {k: round(v, 4) for k, v in stages.items()},
                "stage_share": {k: round(v / sum(stages.values()), 4) for k, v in stages.items()}}

    # e2e through the public API with pinned host arrays
    e2e = None
    if not args.no_e2e:
        pin_in = torch.from_numpy(c_host).pin_memory()
        pin_mid = torch.empty_like(pin_in).pin_memory()
        pin_out = torch.empty_like(pin_in).pin_memory()
        a_in, a_mid, a_out = pin_in.numpy(), pin_mid.numpy(), pin_out.numpy()

        def e2e_step():
            a_mid[...] = cj.forward_batched(fp, a_in, check_finite=False)
            a_out[...] = cj.inverse_batched(ip, a_mid, check_finite=False)

        e2e_step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        e2e_s = (time.perf_counter() - t0) / args.steps
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        nbytes = batch * n1 * 8
        e2e = {"value": world * batch * n1 / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 2 * nbytes,
               "d2h_bytes_per_step": 2 * nbytes,
               "path": "forward_batched/inverse_batched on pinned NumPy arrays (cjt_execute_host: H2D, "
                       "execute, D2H per call), host wall clock per step, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        arm = CpuArm(wl, args.config)
        nvec = min(max(arm.cores, sample_size(arm, 20.0)), 4 * arm.cores * 8)
        wall = arm.sample(nvec)
        arm.close()
        cpu = {"value": nvec * n1 / wall, "unit": UNIT, "cores": arm.cores, "kind": arm.kind,
               "sample": f"{nvec} seeded config{args.config} vectors, fwd+inv each, over {arm.cores} "
                         f"host processes (~{arm.sec_per_vec:.3f} s per vector per core), plans untimed"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SURVEY.md 8(d))",
            "config": config_json(wl, args.config, batch, world, "weak"),
            "gpu_launches": int(launches), "clocks": clk.summary(), "roofline": roofline,
            "cpu_baseline": cpu, "e2e": e2e, "parity_check_vector0": chk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def ctypes_peak(L, st):
    import ctypes
    v = ctypes.c_double(0.0)
    rc = L.cjt_probe_fp64_peak(ctypes.byref(v), st)
    return v.value if rc == 0 else None


def main():
    args = parse()
    wl = WORKLOADS[args.config]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
