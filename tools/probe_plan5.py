"""Per-plan host / device creation times of configuration 5's 225 plan pairs."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch
import cjt_oracle as O
import paper_1602_02618_b200 as cj
from paper_1602_02618_b200 import planner as pl, engine
torch.cuda.init(); torch.zeros(1, device="cuda")
keys = sorted(set(O.config5_draws(4096)))
rows = []
for a, b, n in keys:
    for d in ("forward", "inverse"):
        t0 = time.perf_counter(); hp = pl.build(d, pl.JacobiParameters(a, b), n); t1 = time.perf_counter()
        tp = engine.TransformPlan(hp); tp.device_plan(0); torch.cuda.synchronize(); t2 = time.perf_counter()
        rows.append((t2 - t0, t1 - t0, t2 - t1, a, b, n, d, hp.half_gemm, len(hp.blocks)))
rows.sort(reverse=True)
tot_h = sum(r[1] for r in rows); tot_d = sum(r[2] for r in rows)
print(json.dumps({"host_s": tot_h, "device_s": tot_d}))
for r in rows[:25]:
    print("%.3f host %.3f dev %.3f  (%g,%g) N=%d %s gemm=%s blocks=%d" % r)
