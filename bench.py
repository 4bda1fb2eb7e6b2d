"""Benchmark: forward + inverse CJT throughput (coefficients/s, fp64) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One step = forward then inverse transform of one batch of seeded synthetic
coefficient vectors; value = coefficients pushed through
fwd+inv per second over all ranks.  Default workload: the headline
configuration the "1/2/4/8 B200" metric is quoted on, BASELINE.json
configs[2] (alpha = beta = 1/2, N = 4095, a fixed batch of 8192 vectors split
into contiguous slices over the GPUs: strong scaling).
`--gpus N` outside torchrun re-launches itself as N ranks.  Inputs are
resident in HBM for `value`; `e2e` goes through the public batched API with
pinned host arrays (H2D and D2H inside the timed region).  `--impl reference`
times the unmodified reference (oracle/_ref, Cython backend) on the host
cores instead (rank 0 only).
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
BOUND_NOTE = ("fp64 pipe: the FFT stages run on DFMA/DADD, the contractions on DMMA (mma.sync f64; tcgen05 "
              "has no f64 kind), which shares that pipe on B200; every stage moves <= 2.3 TB/s of HBM "
              "(profiles/ncu_traffic.json), so neither 'hbm' nor the bf16 'tensor' peak applies")

WORKLOADS = {
    1: dict(alpha=0.0, beta=0.0, n=1023, batch=1, env="1/(n+1)"),
    2: dict(alpha=-0.25, beta=0.4, n=2**14 - 1, batch=64, env="(n+1)^-1.5"),
    3: dict(alpha=0.5, beta=0.5, n=4095, batch=8192, env="0.999^n"),
    4: dict(alpha=0.3, beta=-0.45, n=2**20 - 1, batch=16, env="1/(n+1)"),
    5: dict(alpha=None, beta=None, n=None, batch=4096, env="(n+1)^-1.2"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None,
                    help="global batch, split over the GPUs (default: the config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (1 warm-up + steps)")
    ap.add_argument("--profile-stage", default=None,
                    help="ncu --profile-from-start off: one execution of one stage (fwd_rec, fwd_blocks, "
                         "fwd_edge, inv_rec, inv_blocks, inv_edge) inside cudaProfilerStart/Stop")
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
    plans = {}
    if ref is not None:
        from chebjac import engine

        def run(c, a, b, nn):
            key = (a, b, nn)
            if key not in plans:
                p = ref.JacobiParameters(a, b)
                plans[key] = (p, engine.plan("forward", p, nn), engine.plan("inverse", p, nn))
            p, fp, ip = plans[key]
            t = time.perf_counter()
            engine.inverse(ip, engine.forward(fp, ref.jacobi(p, c)))
            return time.perf_counter() - t
        _W["kind"] = "reference"
    else:
        def run(c, a, b, nn):
            O.oracle_forward(a, b, c)   # warms the oracle's plan cache
            t = time.perf_counter()
            O.oracle_inverse(a, b, O.oracle_forward(a, b, c))
            return time.perf_counter() - t
        _W["kind"] = "port"
    _W["run"] = run
    _W["default"] = (alpha, beta, n)


def _worker_run(task):
    config, n, idx, a, b = task
    O = _W["O"]
    if a is None:
        a, b, n = _W["default"][0], _W["default"][1], n
    c = O.seeded_vector(config, idx, n)
    # plan construction is excluded (cached per worker); only fwd+inv is timed
    return _W["run"](c, a, b, n), _W["kind"]


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
        if config != 5:
            res = self.pool.map(_worker_run, [(config, wl["n"], i, None, None) for i in range(self.cores)],
                                chunksize=1)
            self.kind = res[0][1]
            self.sec_per_vec = statistics.median(r[0] for r in res)

    def sample(self, nvec, offset=0):
        tasks = [(self.config, self.wl["n"], offset + i, None, None) for i in range(nvec)]
        t = time.perf_counter()
        self.pool.map(_worker_run, tasks, chunksize=1)
        return time.perf_counter() - t

    def sample_tasks(self, tasks):
        """(config, n, idx, alpha, beta) tasks; returns summed per-vector fwd+inv
        seconds (plans built and cached untimed inside each worker) and the kind."""
        res = self.pool.map(_worker_run, tasks, chunksize=1)
        self.kind = res[0][1]
        return sum(r[0] for r in res)

    def close(self):
        self.pool.terminate()


def sample_size(arm, target_cpu_seconds):
    n = max(arm.cores, int(round(target_cpu_seconds / max(arm.sec_per_vec, 1e-6))))
    return int(math.ceil(n / arm.cores) * arm.cores)


def config_json(wl, config, total, world):
    """The workload identity, identical in both arms (ours and --impl reference)."""
    return {"workload": f"config{config}: fwd+inv CJT alpha={wl['alpha']} beta={wl['beta']} "
                        f"N={wl['n']} batch={total} c_n=z_n*{wl['env']}",
            "alpha": wl["alpha"], "beta": wl["beta"], "N": wl["n"], "global_batch": total,
            "m_terms": 7, "parallelism": f"contiguous batch slices x{world} (SURVEY.md 8(e))",
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
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md 8(d))",
        "config": config_json(wl, args.config, args.batch or wl["batch"], world), "impl": "reference",
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
            # nvidia-smi needs a moment to start: wait for its first sample so
            # that even a millisecond-long timed region is bracketed
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            # one more sample after the timed region (-lms 100)
            n0, t0 = len(self.rows), time.time()
            while len(self.rows) == n0 and time.time() - t0 < 1.0 and self.proc.poll() is None:
                time.sleep(0.01)
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


def stage_model(fhost, ihost, batch: int) -> dict:
    """SURVEY.md 8(d) algorithmic work per stage of one forward + inverse of
    `batch` vectors: flops with the reference's own per-step constants and
    layout (a build doing fewer real flops still uses these), and the
    compulsory HBM bytes of each stage (read its input vectors, write its
    output vectors, f64):
      fwd_rec    B (6 S_f^int + 8 S_f^end)                 bytes B 8 ((N+1) + (G_f+1))
      fwd_blocks B 2 M K_f 2.5 N log2 N                    bytes B 8 ((N+1) + 2 (G_f+1))
      fwd_edge   B 2.5 N log2 N                            bytes B 8 ((G_f+1) + (N+1))
      inv_edge   B 2.5 (2N) log2 (2N)                      bytes B 8 ((N+1) + (G_i+1))
      inv_blocks B 2 M K_i 2.5 (2N) log2 (2N)              bytes B 8 ((G_i+1) + (N+1))
      inv_rec    B 2 (S_i^int + S_i^end) + 5 S_i^int + 7 S_i^end
                                                           bytes B 8 ((G_i+1) + 2 (N+1))
    with S_f = sum of forward row cuts per region, S_i = sum of inverse row
    cuts capped at N+1 (degrees > N are discarded by the reference)."""
    n, m = fhost.n, fhost.m_terms
    fr, fc = fhost.regions, fhost.cuts.astype(np.float64)
    ir, ic = ihost.regions, np.minimum(ihost.cuts, n + 1).astype(np.float64)
    sf_int, sf_end = fc[fr == 0].sum(), fc[fr != 0].sum()
    si_int, si_end = ic[ir == 0].sum(), ic[ir != 0].sum()
    kf, ki = len(fhost.layout.blocks), len(ihost.layout.blocks)
    nlog = n * math.log2(n) if n > 1 else 0.0
    n2log = 2 * n * math.log2(2 * n)
    gf1, gi1, n1 = fhost.grid_n + 1, ihost.grid_n + 1, n + 1
    flops = {
        "fwd_rec": batch * (6 * sf_int + 8 * sf_end),
        "fwd_blocks": batch * 2 * m * kf * 2.5 * nlog,
        "fwd_edge": batch * 2.5 * nlog,
        "inv_edge": batch * 2.5 * n2log,
        "inv_blocks": batch * 2 * m * ki * 2.5 * n2log,
        "inv_rec": batch * 2 * (si_int + si_end) + 5 * si_int + 7 * si_end,
    }
    nbytes = {
        "fwd_rec": batch * 8.0 * (n1 + gf1),
        "fwd_blocks": batch * 8.0 * (n1 + 2 * gf1) if kf else 0.0,
        "fwd_edge": batch * 8.0 * (gf1 + n1),
        "inv_edge": batch * 8.0 * (n1 + gi1),
        "inv_blocks": batch * 8.0 * (gi1 + n1) if ki else 0.0,
        "inv_rec": batch * 8.0 * (gi1 + 2 * n1),
    }
    return {"flops": flops, "bytes": nbytes}


def remap_half_exact(model: dict, executed: dict, fhost, ihost, batch: int) -> None:
    """alpha = beta = 1/2 plans run the exact expansion: the forward's U -> T
    kernel (timed as fwd_rec) replaces the reference's recurrence AND its
    analysis DCT, the inverse's one chirp-z product (timed as inv_blocks)
    replaces its transposed recurrence.  The SURVEY 8(d) algorithmic work of
    the replaced reference stages is credited to the stages that now do it."""
    f, b = model["flops"], model["bytes"]
    n1 = fhost.n + 1
    model["half_exact"] = fhost.half_k is not None or ihost.half_k is not None
    if fhost.half_k is not None:
        f["fwd_rec"], f["fwd_edge"] = f["fwd_rec"] + f["fwd_edge"], 0.0
        b["fwd_rec"], b["fwd_edge"] = batch * 8.0 * 2 * n1, 0.0
        executed["fwd_rec"] = None
    if ihost.half_k is not None:
        f["inv_blocks"], f["inv_rec"] = f["inv_blocks"] + f["inv_rec"] + f["inv_edge"], 0.0
        b["inv_blocks"], b["inv_rec"] = batch * 8.0 * ((ihost.grid_n + 1) + n1), 0.0
        executed["inv_rec"] = None
        if getattr(ihost, "half_gemm", False):
            # exact conversion + bf16 tensor-core correction (no fp64 FFT work per
            # execution): it replaces the synthesis, blocks and recurrence
            f["inv_edge"] = 0.0
            b["inv_blocks"], b["inv_edge"] = batch * 16.0 * n1, 0.0
            executed["inv_blocks"] = None
        else:
            f["inv_blocks"] -= f["inv_edge"]
    # the kernels' own rooflines (what bounds the work they actually do): the
    # U -> T scan moves 16 B per coefficient (HBM); the correction GEMM does
    # 2 (N+1)^2 bf16 flop per vector on the tensor cores
    kinds = model.setdefault("kind", {})
    if fhost.half_k is not None:
        kinds["fwd_rec"] = ("hbm", batch * 16.0 * n1,
                            "k_half_fwd_warp (alpha = beta = 1/2 exact U -> T conversion, TMA-fed warp scans): "
                            "read c, write cheb")
    if ihost.half_k is not None and getattr(ihost, "half_gemm", False):
        kinds["inv_blocks"] = ("tensor", batch * 2.0 * n1 * n1,
                               "alpha = beta = 1/2 inverse: k_to_bf16 + k_half_inv_umma (tcgen05 bf16 GEMM of "
                               "the first-order correction to the reference's points, TMEM accumulators, fp64 "
                               "exact T -> U fused into the epilogue); achieved = the GEMM's 2 (N+1)^2 flop per "
                               "vector over the whole stage time (both kernels)")


def survey_flops(fhost, ihost, batch: int) -> float:
    """SURVEY.md 8(d) F of one forward + inverse step (sum over the stages;
    the diagonal scalings, < 2 %, are omitted)."""
    return float(sum(stage_model(fhost, ihost, batch)["flops"].values()))


def step_roofline(flop: float, peak_tflops: float, ms_per_step: float, coeffs: float) -> dict:
    t_ms = flop / (peak_tflops * 1e12) * 1e3
    t_hbm_ms = 32.0 * coeffs / 6.5546e12 * 1e3   # read c, write c per direction (SURVEY 8(d) bytes)
    t_roof = max(t_ms, t_hbm_ms)
    return {"model": "SURVEY.md 8(d) F: the reference's algorithmic fp64 flops per step",
            "flop_per_step": float(flop), "t_fp64_ms": float(t_ms), "t_hbm_ms": float(t_hbm_ms),
            "roofline_coeffs_per_s": float(coeffs / (t_roof * 1e-3)),
            # capped at 1: the DMMA contraction does fewer real
            # flops than the reference's per-vector Clenshaw chains
            "frac": float(min(1.0, t_roof / ms_per_step)), "frac_uncapped": float(t_roof / ms_per_step)}


def dominant_roofline(stages_ms: dict, model: dict, executed: dict, peak: float, config: int) -> dict:
    """roofline object of the dominant stage (longest CUDA-event time):
    achieved = its SURVEY 8(d) algorithmic flops / its time, frac = achieved /
    measured fp64 peak (capped at 1, uncapped kept); the executed-flop rate and
    pipe fraction are reported beside it, and ncu's DRAM bytes of one
    execution of the stage over its compulsory bytes."""
    dom = max(stages_ms, key=stages_ms.get)
    t = stages_ms[dom] * 1e-3
    alg = model["flops"][dom]
    achieved = alg / t / 1e12
    kern = {"fwd_rec": "k_rec_forward_ws / k_pgen_fwd + k_rec_gemm (K1)",
            "inv_rec": "k_rec_inverse_ws / k_pgen_inv + k_rec_gemm (K2)"}.get(
        dom, "k_chirpz_* (Bluestein chirp-z, K3/K4)")
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            t_ = json.loads(prof.read_text()).get(f"config{config}", {}).get(dom)
            traffic = None if t_ is None else float(t_["bytes"])
        except (ValueError, OSError, KeyError, TypeError):
            traffic = None
    ex = executed.get(dom)
    ab = model["bytes"][dom]
    stage_ms = {k: round(v, 4) for k, v in stages_ms.items()}
    stage_share = {k: round(v / sum(stages_ms.values()), 4) for k, v in stages_ms.items()}
    kind = model.get("kind", {}).get(dom)
    if kind is not None:
        bound, work, kname = kind
        peaks = measured_peaks()
        if bound == "hbm":
            achieved, pk, unit = work / t / 1e9, peaks["hbm_gbs"], "GB/s"
        else:
            achieved, pk, unit = work / t / 1e12, peaks["bf16_tflops"], "TFLOP/s"
        return {
            "bound": bound, "kernel": kname, "stage": dom, "achieved": achieved, "peak": pk, "unit": unit,
            "frac": achieved / pk, "traffic": traffic,
            "traffic_note": "ncu dram__bytes_read+write of one execution of this stage (profiles/ncu_traffic.json)",
            "algorithmic_bytes" if bound == "hbm" else "algorithmic_flop": work,
            "peak_source": peaks["source"] + (" (hbm_gbs)" if bound == "hbm" else " (bf16_tflops, burst: the stage "
                                                                                  "is timed alone)"),
            "fp64_peak_measured": peak,
            "stage_ms": stage_ms, "stage_share": stage_share,
        }
    return {
        "bound": "fp64", "bound_note": BOUND_NOTE, "kernel": kern, "stage": dom,
        "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": min(1.0, achieved / peak) if peak else None,
        "frac_uncapped": achieved / peak if peak else None,
        "traffic": traffic,
        "traffic_note": "ncu dram__bytes_read+write of one execution of this stage (profiles/ncu_traffic.json)",
        "algorithmic_flop": alg, "algorithmic_bytes": ab,
        "traffic_over_algorithmic_bytes": (traffic / ab) if (traffic and ab) else None,
        "flops_model": "SURVEY.md 8(d) per-stage algorithmic flops (bench.stage_model)",
        "executed": None if ex is None else {
            "flop": ex, "tflops": ex / t / 1e12, "pipe_frac": ex / t / 1e12 / peak if peak else None,
            "note": "flops the kernels actually execute (contraction 2 per row x degree x vector + "
                    "generation; FFT 5 L log2 L per complex FFT executed)"},
        "peak_source": "measured on this GPU by cjt_probe_fp64_peak (DFMA chains); nominal 37.2",
        "nominal_peak": NOMINAL_FP64_TFLOPS,
        "stage_ms": stage_ms, "stage_share": stage_share,
    }


def measured_peaks() -> dict:
    """HBM GB/s and bf16 TF/s from the driver-written MEASURED_PEAKS.json, else
    the profiling recipe's fallback (6650 GB/s, 1590 TF/s)."""
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "source": "of measured (MEASURED_PEAKS.json)"}
    except (OSError, ValueError, KeyError, TypeError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "of fallback (B200_PROFILING.md)"}


def shard_batch(config: int, n: int, total: int, world: int, rank: int) -> tuple[int, int, np.ndarray]:
    """This rank's contiguous slice [lo, hi) of the config's fixed seeded batch
     and its input vectors."""
    import cjt_oracle as O
    from paper_1602_02618_b200 import sharding
    lo, hi = sharding.contiguous_slice(total, world, rank)
    if hi <= lo:
        return lo, hi, np.zeros((0, n + 1))
    return lo, hi, np.stack([O.seeded_vector(config, v, n) for v in range(lo, hi)])


def roundtrip_stats(c, back):
    """Per-vector round-trip error max|inv(fwd(c)) - c| / ||c||_1 (a (rows, 1) tensor)."""
    return ((back - c).abs().amax(dim=1) / c.abs().sum(dim=1)).unsqueeze(1)


def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    import paper_1602_02618_b200 as cj
    from paper_1602_02618_b200 import _native as nat
    from paper_1602_02618_b200 import sharding
    import cjt_oracle as O

    rank, local, world = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    total = args.batch or wl["batch"]
    n1 = wl["n"] + 1
    p = cj.JacobiParameters(wl["alpha"], wl["beta"])
    fp = cj.plan("forward", p, wl["n"])
    ip = cj.plan("inverse", p, wl["n"])
    # strong scaling: the config's fixed batch, contiguous slices per rank
    lo, hi, c_host = shard_batch(args.config, wl["n"], total, world, rank)
    batch = hi - lo
    if batch < 1:
        raise SystemExit(f"rank {rank}: empty shard (batch {total} over {world} GPUs)")
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
    if args.profile_stage:
        d, sname = args.profile_stage.split("_")
        mask = {"rec": nat.STAGE_REC, "blocks": nat.STAGE_BLOCKS, "edge": nat.STAGE_EDGE}[sname]
        dp, src, dst = (fdp, c_dev, cheb) if d == "fwd" else (idp, cheb, back)
        L = nat.lib()
        nat.check(L.cjt_execute_stage(dp.handle, src.data_ptr(), dst.data_ptr(), batch, mask, stream.cuda_stream))
        torch.cuda.synchronize(dev)
        torch.cuda.profiler.start()
        nat.check(L.cjt_execute_stage(dp.handle, src.data_ptr(), dst.data_ptr(), batch, mask, stream.cuda_stream))
        torch.cuda.synchronize(dev)
        torch.cuda.profiler.stop()
        return

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

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # one step captured into a CUDA graph (stream-ordered, allocation-free
    # executes), replayed per timed step: launch overhead off the small configs
    graph = None
    if not os.environ.get("CJT_BENCH_NO_GRAPH"):
        try:
            # capture on a stream whose per-stream plan workspaces exist
            # (warmed up eagerly first; nothing is allocated while capturing)
            gs = torch.cuda.Stream(dev)
            gs.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(gs):
                step()
            gs.synchronize()
            g_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_, stream=gs):
                step()
            g_.replay()
            torch.cuda.synchronize(dev)
            graph = g_
        except RuntimeError:
            graph = None
            torch.cuda.synchronize(dev)
    run_step = graph.replay if graph is not None else step
    for _ in range(2):
        run_step()
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)

    with ClockSampler(local) as clk:
        step_ms = timed(run_step, args.steps)
    ms_per_step = max_over_ranks(sum(step_ms)) / args.steps
    value = total * n1 / (ms_per_step * 1e-3)

    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_per_step}), flush=True)
        return

    # coverage of the sharded batch (after timing): every rank's per-vector
    # round-trip errors, reassembled in global vector order
    rt = sharding.gather_rows(roundtrip_stats(c_dev, back), total, world, rank)
    coverage = {"vectors": int(rt.shape[0]), "global_batch": total,
                "max_roundtrip": float(rt.max()), "slice_rank0": [0, sharding.contiguous_slice(total, world, 0)[1]]}

    # correctness spot check of the timed output against the oracle (not timed)
    chk = None
    if rank == 0:
        v = 0
        ref_f = O.oracle_forward(wl["alpha"], wl["beta"], c_host[v]) if wl["n"] < 70000 else None
        if ref_f is not None:
            ref_i = O.oracle_inverse(wl["alpha"], wl["beta"], ref_f)
            chk = {"fwd": O.parity(cheb[v].cpu().numpy(), ref_f, c_host[v]),
                   "inv": O.parity(back[v].cpu().numpy(), ref_i, c_host[v]),
                   "oracle_plans": O.plan_source()}

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
    executed = {"fwd_rec": 2.0 * fst.rec_steps_executed * batch + 5.0 * fst.rec_steps_executed,
                "inv_rec": 2.0 * ist.rec_steps_executed * batch + 5.0 * ist.rec_steps_executed}
    for d, s_ in (("fwd", fst), ("inv", ist)):
        both = stages[f"{d}_blocks"] + stages[f"{d}_edge"]
        for sname in ("blocks", "edge"):
            share = stages[f"{d}_{sname}"] / both if both > 0 else 0.0
            executed[f"{d}_{sname}"] = 5.0 * s_.fft_points_per_vector * batch * share
    model = stage_model(fp.host, ip.host, batch)
    remap_half_exact(model, executed, fp.host, ip.host, batch)
    roofline = dominant_roofline(stages, model, executed, peak, args.config)
    roofline["step"] = step_roofline(survey_flops(fp.host, ip.host, batch), peak, sum(step_ms) / args.steps,
                                     float(batch * n1))

    # e2e through the public API: pinned host input -> pipeline(forward, inverse)
    # -> pinned host output, copies overlapped with compute across 2 streams
    e2e = None
    if not args.no_e2e:
        pin_in = torch.from_numpy(c_host).pin_memory()
        pin_outs = [torch.empty_like(pin_in).pin_memory() for _ in range(2)]
        chunk = max(batch // 4, min(batch, 64))
        # every step: H2D of its inputs, forward, inverse, D2H of its results;
        # steps are streamed (pipeline(sync=False): H2D, compute and D2H streams over 3 buffer slots),
        # so one step's copies run under its neighbours' transforms
        for w_ in range(2):
            cj.pipeline((fp, ip), pin_in, pin_outs[w_], chunk=chunk, streams=3, device=local, sync=False)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for k_ in range(args.steps):
            cj.pipeline((fp, ip), pin_in, pin_outs[k_ % 2], chunk=chunk, streams=3, device=local, sync=False)
        torch.cuda.synchronize(dev)
        e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
        pin_out = pin_outs[(args.steps - 1) % 2]
        nbytes = batch * n1 * 8
        ok = bool(np.array_equal(pin_out.numpy(), back.cpu().numpy())) if chunk == batch else None
        e2e = {"value": total * n1 / e2e_s, "unit": UNIT, "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "chunk": chunk, "matches_device_path": ok,
               "path": "paper_1602_02618_b200.pipeline((fwd_plan, inv_plan), pinned host in, pinned host out, "
                       "sync=False) per step: H2D, forward, inverse, D2H per chunk on three streams (copies in, "
                       "transforms, copies out) over 3 device buffer slots, one synchronize after the K steps; "
                       "host wall clock "
                       "per step, max over ranks (bytes are per rank)",
               "note": "streamed steps overlap on the two streams, so e2e can exceed the single-stream "
                       "device value (which serialises steps); every step still copies its inputs in and "
                       "its results out"}

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
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SURVEY.md 8(d))",
            "config": config_json(wl, args.config, total, world),
            "cuda_graph": graph is not None,
            "gpu_launches": int(launches), "clocks": clk.summary(), "roofline": roofline,
            "cpu_baseline": cpu, "e2e": e2e, "parity_check_vector0": chk, "coverage": coverage,
        }
        if getattr(ip.host, "half_gemm", False):
            line["numerics"] = ("fp64 throughout, except the alpha = beta = 1/2 inverse's first-order "
                                "correction to the reference's evaluation points (|M t| ~ 1e-12 ||t||_1): "
                                "bf16 operands with fp32 accumulation on the tensor cores, contributing "
                                "<= ~1e-15 ||t||_1; the exact conversion and the sum are fp64 (DESIGN.md 3.5)")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def ctypes_peak(L, st):
    import ctypes
    v = ctypes.c_double(0.0)
    rc = L.cjt_probe_fp64_peak(ctypes.byref(v), st)
    return v.value if rc == 0 else None


def config5_sample(draws, cores):
    """Bounded CPU sample of configuration 5: every 8th vector with N <= 16383
    (the reference's per-coefficient cost grows with N, so this overstates the
    CPU rate and understates the speed-up)."""
    idx = [i for i, (a, b, n) in enumerate(draws) if n <= 16383][::8][: 8 * cores]
    return [(5, draws[i][2], i, draws[i][0], draws[i][1]) for i in idx]


def run_reference5(args, wl):
    import cjt_oracle as O
    rank, _, world = dist_env()
    if rank != 0:
        return
    draws = O.config5_draws(wl["batch"])
    arm = CpuArm(wl, 5)
    tasks = config5_sample(draws, arm.cores)
    coeffs = sum(t[1] + 1 for t in tasks)
    arm.sample_tasks(tasks)   # warm-up: plans built and cached per worker
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        arm.sample_tasks(tasks)
        times.append(time.perf_counter() - t)
    arm.close()
    value = coeffs * args.steps / sum(times)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md 8(d))",
        "config": config5_json(world), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": arm.cores, "kind": arm.kind,
                         "sample": f"{len(tasks)} config-5 vectors with N <= 16383 (every 8th), fwd+inv, "
                                   f"{arm.cores} host processes, plans cached untimed"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config5_json(world):
    return {"workload": "config5: ragged fwd+inv CJT, 4096 vectors, (alpha, beta) uniform on "
                        "{-0.45,-0.2,0,0.25,0.5}^2, N uniform on {2^8..2^16}-1, c_n=z_n*(n+1)^-1.2, "
                        "225 plan pairs, groups LPT-sharded over GPUs",
            "global_batch": 4096, "parallelism": f"LPT group sharding x{world}",
            "l2": "flushed between timed steps (256 MiB write)"}


def run_ours5(args, wl):
    import torch
    import torch.distributed as dist

    import cjt_oracle as O
    from paper_1602_02618_b200 import _native as nat
    from paper_1602_02618_b200 import sharding
    from paper_1602_02618_b200.ragged import RaggedPlan

    rank, local, world = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    draws = O.config5_draws(wl["batch"])
    # shard whole groups by a cheap cost proxy (alpha = beta = 1/2 plans are pure O(N^2))
    keys = list(dict.fromkeys(draws))
    counts = {k: 0 for k in keys}
    for d in draws:
        counts[d] += 1
    proxy = np.array([counts[(a, b, n)] * (n + 1) ** 2 * (1.0 if (a == b == 0.5) else 0.08)
                      for a, b, n in keys])
    mine = sharding.lpt_assign(proxy, world)[rank]
    t0 = time.perf_counter()
    rp = RaggedPlan(draws, groups_subset=mine)
    plan_s = time.perf_counter() - t0
    vecs = {}
    for g, mem in enumerate(rp.members):
        for i in mem:
            vecs[i] = O.seeded_vector(5, i, draws[i][2])
    host = rp.pack(vecs)
    x = torch.from_numpy(host).to(dev)
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    rp.reserve()
    nstreams = int(os.environ.get("CJT_RAGGED_STREAMS", "4"))
    streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
    assignment = rp.assign(nstreams)

    def step_eager():
        rp.execute("forward", x, y, streams, assignment)
        rp.execute("inverse", y, z, streams, assignment)

    for _ in range(2):
        step_eager()
    torch.cuda.synchronize(dev)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step_eager()
    graph.replay()
    torch.cuda.synchronize(dev)
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup - 1, 0)):
        graph.replay()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            graph.replay()
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    total_ms = sum(s_.elapsed_time(e_) for s_, e_ in zip(starts, ends))
    coeffs = torch.tensor([float(rp.total)], dtype=torch.float64, device=dev)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.all_reduce(coeffs)
    ms_per_step = total_ms / args.steps
    value = float(coeffs.item()) / (ms_per_step * 1e-3)

    chk = None
    if rank == 0:
        zh, yh = z.cpu().numpy(), y.cpu().numpy()
        worst = {"fwd": 0.0, "inv": 0.0}
        for g, mem in enumerate(rp.members):
            a, b, n = rp.keys[g]
            if n > 2047:
                continue
            i0 = mem[0]
            off = rp.offsets[g]
            c = vecs[i0]
            rf = O.oracle_forward(a, b, c)
            worst["fwd"] = max(worst["fwd"], O.parity(yh[off:off + n + 1], rf, c))
            worst["inv"] = max(worst["inv"], O.parity(zh[off:off + n + 1], O.oracle_inverse(a, b, yh[off:off + n + 1]),
                                                     yh[off:off + n + 1]))
        chk = {"groups_checked_N_le_2047": worst}

    # per-stage sums over groups (sequential, one stream) for the roofline
    L = nat.lib()
    st = stream.cuda_stream
    stage_ms = {}
    # untimed pass first: per-stream workspaces and P arenas of this stream
    for k, (src, dst) in enumerate(((x, y), (y, z))):
        for g in range(len(rp.keys)):
            dp = rp.plans[g][k].device_plan(local)
            nat.check(L.cjt_execute_stage(dp.handle, rp.group_view(src, g).data_ptr(),
                                          rp.group_view(dst, g).data_ptr(), rp.sizes[g], nat.STAGE_ALL, st))
    torch.cuda.synchronize(dev)
    for sname, mask in (("rec", nat.STAGE_REC), ("blocks", nat.STAGE_BLOCKS), ("edge", nat.STAGE_EDGE)):
        for k, (src, dst) in enumerate(((x, y), (y, z))):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for g in range(len(rp.keys)):
                dp = rp.plans[g][k].device_plan(local)
                nat.check(L.cjt_execute_stage(dp.handle, rp.group_view(src, g).data_ptr(),
                                              rp.group_view(dst, g).data_ptr(), rp.sizes[g], mask, st))
            ev1.record(stream)
            torch.cuda.synchronize(dev)
            stage_ms[("fwd_" if k == 0 else "inv_") + sname] = ev0.elapsed_time(ev1)
    graph.replay()
    torch.cuda.synchronize(dev)
    peak = ctypes_peak(L, st)
    # SURVEY 8(d) algorithmic work summed over the groups, per stage
    model = {"flops": {k_: 0.0 for k_ in stage_ms}, "bytes": {k_: 0.0 for k_ in stage_ms}}
    executed = {k_: 0.0 for k_ in stage_ms}
    fft_exec = {"fwd": 0.0, "inv": 0.0}
    for g in range(len(rp.keys)):
        fh, ih = rp.plans[g][0].host, rp.plans[g][1].host
        m_ = stage_model(fh, ih, rp.sizes[g])
        ex_ = {}
        remap_half_exact(m_, ex_, fh, ih, rp.sizes[g])
        for k_ in stage_ms:
            model["flops"][k_] += m_["flops"][k_]
            model["bytes"][k_] += m_["bytes"][k_]
        for k, d in enumerate(("fwd", "inv")):
            s_ = rp.plans[g][k].device_plan(local).stats()
            executed[f"{d}_rec"] += 2.0 * s_.rec_steps_executed * rp.sizes[g] + 5.0 * s_.rec_steps_executed
            fft_exec[d] += 5.0 * s_.fft_points_per_vector * rp.sizes[g]
    for d in ("fwd", "inv"):
        both = stage_ms[f"{d}_blocks"] + stage_ms[f"{d}_edge"]
        for sname in ("blocks", "edge"):
            executed[f"{d}_{sname}"] = fft_exec[d] * (stage_ms[f"{d}_{sname}"] / both if both > 0 else 0.0)
    roofline = dominant_roofline(stage_ms, model, executed, peak, 5)
    roofline["note"] = ("stage times are the groups' stages run back to back on one stream; the timed step "
                        "overlaps groups on several streams")
    flop5 = sum(survey_flops(rp.plans[g][0].host, rp.plans[g][1].host, rp.sizes[g]) for g in range(len(rp.keys)))
    roofline["step"] = step_roofline(flop5, peak, ms_per_step, float(rp.total))
    e2e = None
    if not args.no_e2e:
        pin_in = torch.from_numpy(host).pin_memory()
        pin_out = torch.empty_like(pin_in).pin_memory()
        x.copy_(pin_in, non_blocking=True)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            x.copy_(pin_in, non_blocking=True)
            graph.replay()
            pin_out.copy_(z, non_blocking=True)
            torch.cuda.synchronize(dev)
        e2e_s = (time.perf_counter() - t0) / args.steps
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": float(coeffs.item()) / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(host.nbytes),
               "d2h_bytes_per_step": int(host.nbytes),
               "path": "packed pinned host -> device copy, CUDA-graph replay of RaggedPlan.execute "
                       "(forward then inverse of every group), device -> pinned host copy; host wall clock"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        arm = CpuArm(wl, 5)
        tasks = config5_sample(draws, arm.cores)
        arm.sample_tasks(tasks)
        t0 = time.perf_counter()
        arm.sample_tasks(tasks)
        wall = time.perf_counter() - t0
        arm.close()
        cpu = {"value": sum(t[1] + 1 for t in tasks) / wall, "unit": UNIT, "cores": arm.cores, "kind": arm.kind,
               "sample": f"{len(tasks)} config-5 vectors with N <= 16383 (every 8th), fwd+inv, {arm.cores} host "
                         "processes, plans cached untimed (overstates the CPU rate: cost per coefficient grows with N)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md 8(d))",
            "config": dict(config5_json(world), groups_this_rank=len(rp.keys), plan_seconds=round(plan_s, 1),
                           streams=nstreams, cuda_graph=True),
            "gpu_launches": int(rp.launches()), "clocks": clk.summary(), "roofline": roofline,
            "cpu_baseline": cpu, "e2e": e2e, "parity_check": chk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """`--gpus N` without a torchrun environment: re-launch this command as N
    ranks (one process per GPU) under torch.distributed.run on 127.0.0.1."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    wl = WORKLOADS[args.config]
    if args.config == 5:
        (run_reference5 if args.impl == "reference" else run_ours5)(args, wl)
    elif args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
