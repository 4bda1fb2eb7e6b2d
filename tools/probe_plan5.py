"""Plan-creation times of configuration 5's 225 plan pairs (host planner and
device upload separately, plans kept alive), and the threaded RaggedPlan."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch
import cjt_oracle as O
from paper_1602_02618_b200 import planner as pl, engine
from paper_1602_02618_b200.ragged import RaggedPlan
torch.zeros(1, device="cuda")
keys = sorted(set(O.config5_draws(4096)))
rows, keep = [], []
for a, b, n in keys:
    for d in ("forward", "inverse"):
        t0 = time.perf_counter(); hp = pl.build(d, pl.JacobiParameters(a, b), n); t1 = time.perf_counter()
        tp = engine.TransformPlan(hp); tp.device_plan(0); torch.cuda.synchronize(); t2 = time.perf_counter()
        keep.append(tp)
        rows.append((t2 - t0, t1 - t0, t2 - t1, a, b, n, d, hp.half_gemm, len(hp.blocks)))
rows.sort(reverse=True)
print(json.dumps({"serial_host_s": sum(r[1] for r in rows), "serial_device_s": sum(r[2] for r in rows)}))
del keep
torch.cuda.synchronize()
t0 = time.perf_counter(); rp = RaggedPlan(O.config5_draws(4096)); torch.cuda.synchronize()
print(json.dumps({"ragged_threaded_s": time.perf_counter() - t0}))
for r in rows[:12]:
    print("%.3f host %.3f dev %.3f  (%g,%g) N=%d %s gemm=%s blocks=%d" % r)
