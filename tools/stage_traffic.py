"""Sum ncu per-kernel DRAM bytes of one stage capture into profiles/ncu_traffic.json.

    python tools/stage_traffic.py CONFIG STAGE gpurun_out/x.csv [...]   (pairs of STAGE CSV)
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
cfg = sys.argv[1]
out = ROOT / "profiles" / "ncu_traffic.json"
data = json.loads(out.read_text()) if out.exists() else {}
args = sys.argv[2:]
for stage, path in zip(args[0::2], args[1::2]):
    rows = list(csv.reader(open(path)))
    hdr = next((i for i, r in enumerate(rows) if "Metric Name" in r), None)
    if hdr is None:   # the stage launches no kernel in this configuration
        data.setdefault(f"config{cfg}", {})[stage] = {"bytes": 0.0, "read": 0.0, "write": 0.0, "kernels": 0,
                                                      "ncu_us": 0.0, "source": path}
        continue
    h = rows[hdr]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = {"dram__bytes_read.sum": 0.0, "dram__bytes_write.sum": 0.0, "gpu__time_duration.sum": 0.0}
    kernels = 0
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] not in tot:
            continue
        v = float(r[vi].replace(",", ""))
        if r[mi].startswith("dram"):
            v *= scale.get(r[ui], 1)
        else:
            kernels += 1
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        tot[r[mi]] += v
    data.setdefault(f"config{cfg}", {})[stage] = {
        "bytes": tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"],
        "read": tot["dram__bytes_read.sum"], "write": tot["dram__bytes_write.sum"],
        "kernels": kernels, "ncu_us": tot["gpu__time_duration.sum"], "source": path}
out.write_text(json.dumps(data, indent=1) + "\n")
print(json.dumps(data, indent=1))
