"""Per-source-line totals of selected ncu source-page columns (run here).

    python tools/ncu_lines.py REPORT KERNEL_REGEX [N] [COLUMN ...]
SASS rows are folded into their CUDA source line.
"""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 12
cols = sys.argv[4:] or ["# Samples", "L1 Wavefronts Shared Excessive", "L1 Wavefronts Shared",
                        "L2 Theoretical Sectors Global Excessive", "stall_long_sb", "stall_barrier",
                        "stall_math", "stall_mio", "stall_short_sb"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", "regex:" + rx, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, path, cur, tot = None, "?", None, {}


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


for r in rows:
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        path = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0] not in ("", "-"):
        cur = (path, r[0], r[1].strip()[:90])
        tot.setdefault(cur, {})
        continue   # the CUDA line's own totals repeat its SASS rows
    if cur is None:
        continue
    d = tot[cur]
    for c in cols:
        if c in hdr:
            d[c] = d.get(c, 0.0) + num(r[hdr.index(c)])
for c in cols:
    s = sum(d.get(c, 0.0) for d in tot.values())
    print(f"== {c}: total {s:.0f}")
    for k, d in sorted(tot.items(), key=lambda kv: -kv[1].get(c, 0.0))[:n]:
        if d.get(c, 0.0) > 0:
            print(f"  {d[c]:12.0f} {100 * d[c] / max(s, 1):5.1f}%  {k[0]}:{k[1]}  {k[2]}")
