"""Round-2 probe (GPU box): folded-inverse deviation vs the reference for
alpha = beta classes, and plan-time split (host planner vs device upload)."""
import json, os, sys, time
from concurrent.futures import ProcessPoolExecutor
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import cjt_oracle as O


def ref_pair(args):
    a, n, v = args
    ch = O.reference_package()
    from chebjac import engine
    p = ch.JacobiParameters(a, a)
    c = O.seeded_vector(5, v, n)
    f = engine.forward(engine.plan("forward", p, n), ch.jacobi(p, c)).data
    i = engine.inverse(engine.plan("inverse", p, n), ch.chebyshev(f)).data
    return a, n, v, c, f, i


def main():
    import torch
    import paper_1602_02618_b200 as cj
    from paper_1602_02618_b200 import planner as pl
    out = {"plan": {}, "fold": []}
    for name, (a, b, n) in {"c2": (-0.25, 0.4, 16383), "c3": (0.5, 0.5, 4095),
                            "c4": (0.3, -0.45, 2**20 - 1), "c5max": (-0.45, 0.5, 65535),
                            "c5half": (0.5, 0.5, 65535)}.items():
        for d in ("forward", "inverse"):
            t0 = time.perf_counter(); hp = pl.build(d, pl.JacobiParameters(a, b), n); t1 = time.perf_counter()
            tp = cj.engine.TransformPlan(hp); tp.device_plan(0); torch.cuda.synchronize(); t2 = time.perf_counter()
            tp.device_plan(0).reserve(16); torch.cuda.synchronize(); t3 = time.perf_counter()
            out["plan"][f"{name}_{d}"] = {"host_s": t1 - t0, "device_s": t2 - t1, "reserve16_s": t3 - t2}
            print(name, d, out["plan"][f"{name}_{d}"], flush=True)
            del tp, hp
    jobs = [(a, n, v) for a in (-0.45, -0.2, 0.0, 0.25, 0.5) for n in (1023, 4095, 16383, 65535) for v in range(2)]
    with ProcessPoolExecutor(min(16, os.cpu_count())) as ex:
        res = list(ex.map(ref_pair, jobs))
    for a, n, v, c, f, i in res:
        row = {"a": a, "n": n, "v": v}
        for fold in ("0", "1"):
            os.environ["CJT_FOLD_INVERSE"] = fold
            ip = cj.plan("inverse", cj.JacobiParameters(a, a), n)
            got = cj.inverse_batched(ip, torch.from_numpy(f[None]).cuda()).cpu().numpy()[0]
            row["fold" + fold] = O.parity(got, i, f)
        fp = cj.plan("forward", cj.JacobiParameters(a, a), n)
        row["fwd"] = O.parity(cj.forward_batched(fp, torch.from_numpy(c[None]).cuda()).cpu().numpy()[0], f, c)
        out["fold"].append(row)
        print(row, flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "probe_r2.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
