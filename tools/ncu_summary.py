"""Summarise ncu captures for profiles/ (run here, where ncu -i works without a GPU).

    python tools/ncu_summary.py gpurun_out/prof_c2_r01.ncu-rep > profiles/ncu_full_c2_r01.md
    python tools/ncu_summary.py --launches gpurun_out/launches_c2_r01.csv > profiles/launches_c2_r01.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time_us", 1e-3),
    ("dram__bytes_read.sum", "dram_rd_MB", 1.0),
    ("dram__bytes_write.sum", "dram_wr_MB", 1.0),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%", 1.0),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_%", 1.0),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%", 1.0),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%", 1.0),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_%", 1.0),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_inst_%", 1.0),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%", 1.0),
    ("launch__registers_per_thread", "regs", 1.0),
    ("launch__grid_size", "grid", 1.0),
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    idx = {name: head.index(name) for name, _, _ in METRICS if name in head}
    kname = head.index("Kernel Name")
    print(f"# ncu --set full summary: {path}\n")
    cols = [short for name, short, _ in METRICS if name in idx]
    print("| kernel | " + " | ".join(cols) + " |")
    print("|---|" + "---|" * len(cols))
    for r in rows[2:]:
        vals = []
        for name, short, scale in METRICS:
            if name not in idx:
                continue
            v = r[idx[name]].replace(",", "")
            unit = units[idx[name]]
            try:
                f = float(v)
                if unit == "byte" or unit == "Kbyte" or unit == "Mbyte" or unit == "Gbyte":
                    f *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[unit]
                elif short == "time_us":
                    f *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1.0)
                vals.append(f"{f:.4g}")
            except ValueError:
                vals.append(v)
        name = r[kname].split("(")[0].replace("void ", "").replace("cjt::<unnamed>::", "")
        print(f"| {name} | " + " | ".join(vals) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    tot = 0.0
    items = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("cjt::<unnamed>::", "")
        t = float(r[vi].replace(",", "")) * 1e-3
        items.append((int(r[ii]), name, t))
    print(f"# launch list (ncu gpu__time_duration, cold cache, serialised): {path}\n")
    print("| id | kernel | us |")
    print("|---|---|---|")
    for i, n, t in items:
        print(f"| {i} | {n} | {t:.1f} |")
    # per-execution share by kernel: plan-time kernels excluded, the profile run
    # executes the transform pair `execs` times (one per k_inverse_finish launch)
    plan_time = ("k_checkpoints", "k_build_inv_gen", "k_fp64_probe")
    execs = max(1, sum(1 for _, n, _ in items if n.startswith("k_inverse_finish")))
    agg = {}
    for _, n, t in items:
        if n.startswith(plan_time) or not n.startswith("k_"):
            continue
        base = n.split("<")[0]
        agg[base] = agg.get(base, 0.0) + t / execs
    tot = sum(agg.values())
    print(f"\n## per execution of (forward, inverse), by kernel ({execs} executions; plan-time kernels excluded)\n")
    print("| kernel | us | share |")
    print("|---|---|---|")
    for n, t in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"| {n} | {t:.1f} | {t / tot:.3f} |")
    print(f"| total | {tot:.1f} | 1.000 |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[1])
