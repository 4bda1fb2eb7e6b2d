"""Plan-build phase times for config 5's plan pairs ($CJT_PLAN_TIMING=1 lines on
stderr, aggregated), serial, plus the host planner alone."""
import os, sys, time, json, re, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    import cjt_oracle as O
    from paper_1602_02618_b200 import planner as pl, engine
    torch.zeros(1, device="cuda")
    keys = sorted(set(O.config5_draws(4096)))
    th = 0.0
    keep = []
    t0 = time.perf_counter()
    for a, b, n in keys:
        for d in ("forward", "inverse"):
            t1 = time.perf_counter(); hp = pl.build(d, pl.JacobiParameters(a, b), n); th += time.perf_counter() - t1
            tp = engine.TransformPlan(hp); tp.device_plan(0); keep.append(tp)
    torch.cuda.synchronize()
    print(json.dumps({"host_planner_s": th, "total_s": time.perf_counter() - t0}), flush=True)
    sys.exit(0)
r = subprocess.run([sys.executable, __file__, "child"], capture_output=True, text=True,
                   env=dict(os.environ, CJT_PLAN_TIMING="1"), timeout=600)
agg = {}
for line in r.stderr.splitlines():
    m = re.match(r"\[cjt plan G=(\d+)\]\s+(\S+)\s+([\d.]+) ms", line)
    if m:
        agg[m.group(2)] = agg.get(m.group(2), 0.0) + float(m.group(3))
print(r.stdout.strip())
print(json.dumps({k: round(v, 1) for k, v in agg.items()}))
lines = [l for l in r.stderr.splitlines() if "upload" in l]
print("first uploads:", "\n".join(lines[:4]))
vals = sorted((float(re.search(r"([\d.]+) ms", l).group(1)), l) for l in lines)
print("largest uploads:", "\n".join(v[1] for v in vals[-6:]))
print("median upload ms:", vals[len(vals) // 2][0])
