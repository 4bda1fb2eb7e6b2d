"""Generate tests/golden/shifts.npz from the REAL reference (chebjac):
integer parameter shifts, to_core / from_core and jacobi_to_jacobi
(engine.py:232-354) on seeded inputs.

    python tests/golden/make_golden_shifts.py
"""

from __future__ import annotations

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
from chebjac import engine  # noqa: E402

# single shifts: (alpha, beta, N); the first rows hit alpha + beta = -1 and N = 0
SHIFT_CASES = [(0.0, 0.0, 1), (-0.5, -0.5, 16), (0.25, -0.25, 0), (0.3, -0.45, 255),
               (-0.75, 1.5, 1023), (2.25, 0.125, 4096)]
OPS = ("increment_beta", "decrement_beta", "increment_alpha", "decrement_alpha")
# jacobi_to_jacobi: (source alpha, beta, target alpha, beta, N)
J2J_CASES = [(0.0, 0.0, 0.25, -0.25, 64), (1.5, -0.75, -0.25, 2.5, 255),
             (0.5, 0.5, 0.5, 0.5, 128), (2.75, 1.25, 0.0, 0.0, 1023)]


def seeded(seed, n):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(n + 1) / np.sqrt(np.arange(n + 1) + 1.0)


def main():
    out = {}
    for ci, (a, b, n) in enumerate(SHIFT_CASES):
        c = seeded(7000 + ci, n)
        out[f"shift{ci}_c"] = c
        out[f"shift{ci}_ab"] = np.array([a, b])
        for op in OPS:
            p = ch.JacobiParameters(a, b)
            try:
                r = getattr(engine, op)(ch.jacobi(p, c))
            except ch.ParameterRangeError:
                continue
            out[f"shift{ci}_{op}"] = r.data
            out[f"shift{ci}_{op}_ab"] = np.array([r.params.alpha, r.params.beta])
    for ci, (a, b, ta, tb, n) in enumerate(J2J_CASES):
        c = seeded(8000 + ci, n)
        p = ch.JacobiParameters(a, b)
        core = engine.to_core(ch.jacobi(p, c))
        r = engine.jacobi_to_jacobi(ch.jacobi(p, c), ch.JacobiParameters(ta, tb))
        out[f"j2j{ci}_c"] = c
        out[f"j2j{ci}_case"] = np.array([a, b, ta, tb])
        out[f"j2j{ci}_core"] = core.data
        out[f"j2j{ci}_core_ab"] = np.array([core.params.alpha, core.params.beta])
        out[f"j2j{ci}_out"] = r.data
        print("j2j", ci, "done")
    np.savez_compressed(HERE / "shifts.npz", **out)


if __name__ == "__main__":
    main()
