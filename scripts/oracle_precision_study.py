"""Precision study of the iteration count (reading R14): the oracle's eGl-QMR run in
80-bit extended precision (numpy longdouble: every block, product, update and reduction; only the
scalar norms pass through Python floats) next to its float64 runs, on config 3's operator at m^3
(s = 16, seed 2). The oracle's code is untouched: this script converts the run's blocks after
_Run.__init__ (the recurrences propagate the dtype). Calls only oracle/ and synth/.
    python scripts/oracle_precision_study.py 96 [method [config]]
Appends "m<k>:<method>:longdouble" to profiles/r02_count_ensemble.json.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import oracle.solvers as so  # noqa: E402
import synth  # noqa: E402


def main(m, method="egl_qmr", cfg=3):
    cfg = int(cfg)
    if cfg == 3:
        A = synth.conv_diff_3d(m, (50.0, 30.0, 10.0))
        B = synth.random_rhs(A.n, 16, 2)
    else:
        A, B = synth.make_config(cfg, m=m)
    cplx = np.iscomplexobj(B) or np.iscomplexobj(A.values)
    LD = np.clongdouble if cplx else np.longdouble
    As = A.to_scipy().astype(LD)
    orig = so._Run.__init__

    def init(self, *a, **kw):
        orig(self, *a, **kw)
        self.A = As
        self._AH = None
        self.dt = LD
        self.B = self.B.astype(LD)
        self.X = self.X.astype(LD)
        self.R0 = self.B - self.A @ self.X
    so._Run.__init__ = init
    t0 = time.time()
    r = oracle.solve(method, A.to_scipy(), B, tol=1e-8, maxit=2000, record=0)
    assert r.X.dtype == LD, r.X.dtype
    path = os.path.join(ROOT, "profiles", "r02_count_ensemble.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    key = (f"m{m}" if cfg == 3 else f"c{cfg}m{m}") + f":{method}:longdouble"
    data[key] = {"inputs_hash": synth.input_hash(A, B), "outcome": r.outcome, "iterations": r.iterations,
                 "final_true_rel_residual": float(r.final_true_rel_residual), "tol": 1e-8, "maxit": 2000,
                 "oracle_seconds": round(time.time() - t0, 1), "eps": float(np.finfo(np.longdouble).eps),
                 "crossings": [next((k + 1 for k, v in enumerate(r.history) if v <= 10.0 ** -j), None)
                               for j in range(1, 9)]}
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    print(key, data[key], flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]), *sys.argv[2:4])
