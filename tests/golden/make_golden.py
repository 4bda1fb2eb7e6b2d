"""Generate tests/golden/*.npz from the REAL reference (chebjac, Cython backend).

Run here (the reference is importable from oracle/_ref, built by
oracle/build_ref.sh); the fixtures are committed and the GPU box only reads
them.  Inputs are the seeded synthetic vectors of SURVEY.md 8(d)
(oracle.cjt_oracle.seeded_vector), at sizes a CPU finishes in seconds.

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
import cjt_oracle as O  # noqa: E402

ch = O.reference_package()
if ch is None:
    raise SystemExit("reference not built: run oracle/build_ref.sh first")
from chebjac import asymptotics as asy  # noqa: E402
from chebjac import engine, oracle  # noqa: E402

assert ch.kernel_backend() == "cython", ch.kernel_backend()

# (name, config id for seeds/envelopes, alpha, beta, N, number of vectors)
CASES = [
    ("cfg1", 1, 0.0, 0.0, 1023, 1),
    ("cfg2_small", 2, -0.25, 0.4, 2047, 2),
    ("cfg2_full", 2, -0.25, 0.4, 16383, 1),
    ("cfg3_full", 3, 0.5, 0.5, 4095, 2),
    ("cfg4_small", 4, 0.3, -0.45, 8191, 1),
    ("cfg5_a", 5, -0.45, 0.25, 255, 2),
    ("cfg5_b", 5, 0.5, -0.2, 511, 1),
    ("cfg5_c", 5, 0.0, 0.5, 2047, 1),
    ("cfg5_d", 5, 0.25, 0.25, 4095, 1),
    ("cfg5_e", 5, 0.5, 0.5, 1023, 1),
    ("tiny", 2, -0.25, 0.4, 3, 1),
    ("edge_n1", 1, 0.125, -0.375, 1, 1),
]


def table_digest(tp) -> str:
    h = hashlib.sha256()
    t = tp.tables
    for name in ("A", "B", "C", "rf_plus", "rf_minus", "rf_plus_inv", "rf_minus_inv"):
        h.update(np.ascontiguousarray(getattr(t, name)).tobytes())
    h.update(tp.cuts.tobytes())
    h.update(tp.regions.tobytes())
    h.update(tp.grid.angles.tobytes())
    if tp.weights is not None:
        h.update(tp.weights.w.tobytes())
        h.update(tp.scalings.tobytes())
    return h.hexdigest()


def main():
    layouts = {}
    for name, cfg, a, b, n, nvec in CASES:
        p = ch.JacobiParameters(a, b)
        fp = engine.plan("forward", p, n)
        ip = engine.plan("inverse", p, n)
        cs, fw, iv = [], [], []
        for v in range(nvec):
            c = O.seeded_vector(cfg, v, n)
            f = engine.forward(fp, ch.jacobi(p, c)).data
            i = engine.inverse(ip, ch.chebyshev(f)).data
            cs.append(c)
            fw.append(f)
            iv.append(i)
        extra = {}
        if n <= 2047 and cfg == 1:
            extra["dense"] = oracle.oracle_forward(p, cs[0])
        np.savez_compressed(HERE / f"{name}.npz", alpha=a, beta=b, n=n, c=np.array(cs),
                            fwd=np.array(fw), inv=np.array(iv), **extra)
        layouts[name] = {
            d: {"blocks": [[blk.j, blk.i1, blk.i2] for blk in tp.layout.blocks],
                "n_m": tp.layout.n_m, "tbar": tp.layout.theta_bar_index,
                "digest": table_digest(tp)}
            for d, tp in (("forward", fp), ("inverse", ip))
        }
        print(name, "done")
    # partitions of the full-size configurations (plan only)
    full = {"cfg4_full": (0.3, -0.45, 2**20 - 1), "cfg5_max": (0.5, -0.45, 65535),
            "frozen_2_14": (0.125, 0.375, 2**14)}
    for name, (a, b, n) in full.items():
        p = ch.JacobiParameters(a, b)
        entry = {}
        for d in ("forward", "inverse"):
            g = n if d == "forward" else 2 * n
            lay = asy.compute_partition(p, g, 7, engine.DEFAULT_EPS)
            entry[d] = {"blocks": [[blk.j, blk.i1, blk.i2] for blk in lay.blocks],
                        "n_m": lay.n_m, "tbar": lay.theta_bar_index}
        layouts[name] = entry
        print(name, "done")
    (HERE / "layouts.json").write_text(json.dumps(layouts, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
