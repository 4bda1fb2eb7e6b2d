"""Top source lines by warp-stall samples from an ncu report (run here).

    python tools/ncu_hotlines.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
path, hdr, out = "?", None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            w = float(r[4] or 0)
        except ValueError:
            continue
        out.append((w, path, r[0], r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1.0
for w, p, ln, src in sorted(out, reverse=True)[:n]:
    print(f"{100 * w / tot:5.1f}%  {p}:{ln}  {src}")
