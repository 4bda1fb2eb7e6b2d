"""Recurrence-stage timing vs batch (is K1/K2 producer- or DMMA-bound?).
    python tools/rec_probe.py [N] [alpha beta]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1602_02618_b200 as cj  # noqa: E402
from paper_1602_02618_b200 import _native as nat  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32767
a, b = (float(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (0.5, 0.5)
p = cj.JacobiParameters(a, b)
fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
dev = torch.device("cuda", 0)
L = nat.lib()
st = torch.cuda.current_stream()
for B in (8, 16, 24, 32, 48, 64, 96, 128):
    x = torch.randn(B, n + 1, dtype=torch.float64, device=dev)
    y = cj.forward_batched(fp, x)
    z = cj.inverse_batched(ip, y)
    res = {}
    for name, tp, src, dst in (("fwd", fp, x, y), ("inv", ip, y, z)):
        dp = tp.device_plan(0)
        def run():
            nat.check(L.cjt_execute_stage(dp.handle, src.data_ptr(), dst.data_ptr(), B, nat.STAGE_REC, st.cuda_stream))
        run(); run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        steps = dp.stats().rec_steps
        res[name] = (ms, 2.0 * steps * B / (ms * 1e-3) / 1e12)
    print(f"N={n} ({a},{b}) B={B:4d}  fwd {res['fwd'][0]:8.3f} ms {res['fwd'][1]:6.2f} TF/s   "
          f"inv {res['inv'][0]:8.3f} ms {res['inv'][1]:6.2f} TF/s", flush=True)
