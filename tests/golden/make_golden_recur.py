"""Generate tests/golden/recur.npz from the REAL reference (chebjac, Cython
backend): jacobi_forward / jacobi_forward_reinsch / clenshaw_smith /
clenshaw_smith_reinsch / evaluate_expansion (recurrences.py:74-171) on
seeded inputs, including the endpoints theta = 0 and pi.

    python tests/golden/make_golden_recur.py
"""

from __future__ import annotations

import math
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
from chebjac import recurrences as R  # noqa: E402

PARAMS = [(0.0, 0.0), (-0.5, 0.5), (0.3, -0.45), (0.5, 0.5), (2.25, -0.75)]
THETAS = [0.0, 1e-3, 0.3, math.pi / 4, 1.0, math.pi / 2, 2.0, 3 * math.pi / 4, 3.0, math.pi]
# evaluate_expansion: (alpha, beta, n_coeffs - 1, grid N)
EVAL_CASES = [(0.0, 0.0, 0, 4), (-0.25, 0.4, 63, 100), (0.5, 0.5, 511, 511), (0.3, -0.45, 1000, 257),
              (1.5, -0.5, 2047, 4096)]


def main():
    out = {}
    rng = np.random.default_rng(424242)
    for k, (a, b) in enumerate(PARAMS):
        p = ch.JacobiParameters(a, b)
        n_max = 40 + 50 * k
        c = rng.standard_normal(n_max + 1) / (np.arange(n_max + 1) + 1.0)
        out[f"pt{k}_ab"] = np.array([a, b])
        out[f"pt{k}_c"] = c
        fw, rp, rm, cs, crp, crm = [], [], [], [], [], []
        for th in THETAS:
            fw.append(R.jacobi_forward(p, n_max, th))
            rp.append(R.jacobi_forward_reinsch(p, n_max, th, 1))
            rm.append(R.jacobi_forward_reinsch(p, n_max, th, -1))
            cs.append(R.clenshaw_smith(p, c, th))
            crp.append(R.clenshaw_smith_reinsch(p, c, th, 1))
            crm.append(R.clenshaw_smith_reinsch(p, c, th, -1))
        out[f"pt{k}_fwd"] = np.array(fw)
        out[f"pt{k}_rfp"] = np.array(rp)
        out[f"pt{k}_rfm"] = np.array(rm)
        out[f"pt{k}_cs"] = np.array(cs)
        out[f"pt{k}_crp"] = np.array(crp)
        out[f"pt{k}_crm"] = np.array(crm)
    out["thetas"] = np.array(THETAS)
    for k, (a, b, n, g) in enumerate(EVAL_CASES):
        p = ch.JacobiParameters(a, b)
        c = np.stack([rng.standard_normal(n + 1) * 0.99 ** np.arange(n + 1) for _ in range(3)])
        out[f"ev{k}_abng"] = np.array([a, b, n, g])
        out[f"ev{k}_c"] = c
        out[f"ev{k}_vals"] = np.stack([R.evaluate_expansion(p, c[v], R.AngleGrid(g)) for v in range(3)])
    np.savez_compressed(HERE / "recur.npz", **out)
    print("wrote", HERE / "recur.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
