"""Reference engine on its own backends vs the B200 plugin.

Runs the UNMODIFIED reference engine (oracle/_ref: chebjac.engine.forward /
inverse) with its kernel backend set to "cython" (the reference's native
kernels) and then to "cuda" (paper_1602_02618_b200.backend registered into
chebjac.backend._BACKENDS), on the same seeded vectors, and prints one JSON
line: seconds per forward+inverse per vector for each backend, the share of
the time spent inside the plugin calls, and the max deviation.

    python tools/bench_plugin.py [--config 2] [--vectors 8]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import cjt_oracle as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--vectors", type=int, default=8)
    args = ap.parse_args()
    ch = O.reference_package()
    if ch is None:
        print(json.dumps({"unavailable": "oracle/_ref not built"}))
        return
    from chebjac import backend as rb
    from chebjac import engine
    import paper_1602_02618_b200 as cj
    from paper_1602_02618_b200 import backend as pb
    cj.register_with(rb)
    wl = O.CONFIGS[args.config]
    p = ch.JacobiParameters(wl["alpha"], wl["beta"])
    n = wl["n"]
    fp, ip = engine.plan("forward", p, n), engine.plan("inverse", p, n)
    vecs = [O.seeded_vector(args.config, v, n) for v in range(args.vectors)]
    out, res = {}, {}
    for name in ("cython", "cuda"):
        prev = rb.set_kernel_backend(name)
        try:
            # warm: plans' device state (cuda) / first-call costs
            engine.inverse(ip, engine.forward(fp, ch.jacobi(p, vecs[0])))
            kern = rb.kernels()
            spent = [0.0]

            def timed(fn):
                def w(*a):
                    t = time.perf_counter()
                    fn(*a)
                    spent[0] += time.perf_counter() - t
                return w
            wrapped = type("K", (), {"clenshaw_points": staticmethod(timed(kern.clenshaw_points)),
                                     "transpose_accumulate": staticmethod(timed(kern.transpose_accumulate))})
            rb._BACKENDS["_timed"] = wrapped
            rb.set_kernel_backend("_timed")
            t0 = time.perf_counter()
            res[name] = [engine.inverse(ip, engine.forward(fp, ch.jacobi(p, c))).data for c in vecs]
            dt = time.perf_counter() - t0
        finally:
            rb.set_kernel_backend(prev)
            rb._BACKENDS.pop("_timed", None)
        out[name] = {"s_per_vector": dt / len(vecs), "kernel_share": spent[0] / dt}
    dev = max(O.parity(a, b, c) for a, b, c in zip(res["cuda"], res["cython"], vecs))
    print(json.dumps({"config": args.config, "N": n, "vectors": len(vecs), "backends": out,
                      "speedup_cuda_vs_cython": out["cython"]["s_per_vector"] / out["cuda"]["s_per_vector"],
                      "max_dev_vs_cython_x_l1": dev, "plugin_cache_entries": len(pb._KCACHE)}))


if __name__ == "__main__":
    main()
