"""e2e (pinned host in -> fwd+inv -> pinned host out) of config 3 through
pipeline() for several chunk sizes / stream counts; host wall clock per step."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np, torch
import paper_1602_02618_b200 as cj
n, B = 4095, 8192
p = cj.JacobiParameters(0.5, 0.5)
fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
rng = np.random.default_rng(0)
pin_in = torch.from_numpy(rng.standard_normal((B, n + 1)) * 0.999 ** np.arange(n + 1)).pin_memory()
outs = [torch.empty_like(pin_in).pin_memory() for _ in range(2)]
# raw copy bandwidths for reference
d = torch.empty_like(pin_in, device="cuda")
torch.cuda.synchronize()
for name, fn in (("h2d", lambda: d.copy_(pin_in, non_blocking=True)), ("d2h", lambda: outs[0].copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize(); print(json.dumps({name: pin_in.nbytes * 5 / (time.perf_counter() - t0) / 1e9}))
for chunk, streams in ((2048, 2), (2048, 3), (1024, 2), (1024, 3), (1024, 4), (512, 4), (4096, 2), (8192, 1)):
    for w in range(2):
        cj.pipeline((fp, ip), pin_in, outs[w], chunk=chunk, streams=streams, sync=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    K = 10
    for k in range(K):
        cj.pipeline((fp, ip), pin_in, outs[k % 2], chunk=chunk, streams=streams, sync=False)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K
    print(json.dumps({"chunk": chunk, "streams": streams, "ms_per_step": dt * 1e3, "coeffs_per_s": B * (n + 1) / dt}))
