"""e2e through pipeline() for configs 2 and 3 at several slot counts (host wall clock per step)."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np, torch
import paper_1602_02618_b200 as cj
for cfg, (a, b, n, B, chunk) in {2: (-0.25, 0.4, 16383, 64, 64), 3: (0.5, 0.5, 4095, 8192, 2048)}.items():
    p = cj.JacobiParameters(a, b)
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    rng = np.random.default_rng(0)
    pin_in = torch.from_numpy(rng.standard_normal((B, n + 1)) / np.arange(1, n + 2)).pin_memory()
    outs = [torch.empty_like(pin_in).pin_memory() for _ in range(2)]
    for slots in (1, 2, 3):
        for w in range(2):
            cj.pipeline((fp, ip), pin_in, outs[w], chunk=chunk, streams=slots, sync=False)
        torch.cuda.synchronize()
        K = 10
        t0 = time.perf_counter()
        for k in range(K):
            cj.pipeline((fp, ip), pin_in, outs[k % 2], chunk=chunk, streams=slots, sync=False)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / K
        print(json.dumps({"config": cfg, "slots": slots, "ms": dt * 1e3, "coeffs_per_s": B * (n + 1) / dt}), flush=True)
