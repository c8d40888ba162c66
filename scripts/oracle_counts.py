"""Full-size oracle solves for iteration-count parity ("run once and
cache, keyed by input hash"). Calls only oracle/ and synth/ (no GPU path), and writes
tests/golden/oracle_counts.json: per (config, method) the input hash, the oracle's
outcome, iteration count and final true residual at tol 1e-8, maxit 2000.

    python scripts/oracle_counts.py cfg2 bl_bicg_rq       # ~1 h of numpy on 16 cores
    python scripts/oracle_counts.py cfg3 egl_qmr seq      # the second reduction order (SURVEY §8c.5 rule 3)
    python scripts/oracle_counts.py cfg3 egl_qmr pert0    # BLAS order on B·(1 + 1e-15·N(0,1)), seed 0: one more
                                                          # member of the oracle ensemble of tests/test_gpu_solvers.py
                                                          # (DESIGN §4 rule 2) where "seq" at 256³ would take > 5 h
    python scripts/oracle_counts.py m128 egl_qmr seq      # config 3's operator at 128³ (s = 16, seed 2): the mid-size
                                                          # ensemble study (profiles/r02_count_ensemble.json)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402


def _progress():
    """Print every 25th iteration's recursive residual (wraps _Run.step_done; no arithmetic)."""
    import oracle.solvers as so
    orig = so._Run.step_done

    def step_done(self, k, *a, **kw):
        out = orig(self, k, *a, **kw)
        if k % 25 == 0 and self.res.history:
            print(f"  it {k}: rel {self.res.history[-1]:.3e}", flush=True)
        return out
    so._Run.step_done = step_done


def main(cfg, method, order="blas"):
    _progress()
    import numpy as np
    if cfg.startswith("cfg"):
        A, B = synth.make_config(int(cfg[3:]))
        path = os.path.join(ROOT, "tests", "golden", "oracle_counts.json")
    elif cfg.startswith("c"):  # "c<cfg>m<k>": that config's operator and right-hand sides at grid size k
        num, mm = cfg[1:].split("m")
        A, B = synth.make_config(int(num), m=int(mm))
        path = os.path.join(ROOT, "profiles", "r02_count_ensemble.json")
    else:  # "m<k>": config 3's operator and right-hand sides at k^3 (the count-ensemble study)
        A = synth.conv_diff_3d(int(cfg[1:]), (50.0, 30.0, 10.0))
        B = synth.random_rhs(A.n, 16, 2)
        path = os.path.join(ROOT, "profiles", "r02_count_ensemble.json")
    Bs = B
    if order.startswith("pert"):  # the ensemble's perturbation recipe (tests/test_gpu_solvers.py)
        Bs = B * (1 + 1e-15 * np.random.default_rng(int(order[4:])).standard_normal(B.shape))
    t0 = time.time()
    r = oracle.solve(method, A.to_scipy(), Bs, tol=1e-8, maxit=2000, record=0,
                     order="blas" if order.startswith("pert") else order)
    data = json.load(open(path)) if os.path.exists(path) else {}
    key = f"{cfg}:{method}" + ("" if order == "blas" else f":{order}")
    data[key] = {"inputs_hash": synth.input_hash(A, B), "outcome": r.outcome,
                               "iterations": r.iterations, "half_step": r.half_step,
                               "final_true_rel_residual": r.final_true_rel_residual,
                               "tol": 1e-8, "maxit": 2000, "oracle_seconds": round(time.time() - t0, 1),
                               # first iteration with recursive relative residual <= 1e-1 ... 1e-8
                               "crossings": [next((k + 1 for k, v in enumerate(r.history) if v <= 10.0 ** -j), None)
                                             for j in range(1, 9)]}
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    print(key, data[key], flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:4])
