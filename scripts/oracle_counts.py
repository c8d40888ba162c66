"""Full-size oracle solves for iteration-count parity ("run once and
cache, keyed by input hash"). Calls only oracle/ and synth/ (no GPU path), and writes
tests/golden/oracle_counts.json: per (config, method) the input hash, the oracle's
outcome, iteration count and final true residual at tol 1e-8, maxit 2000.

    python scripts/oracle_counts.py cfg2 bl_bicg_rq       # ~1 h of numpy on 16 cores
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402


def main(cfg, method):
    num = int(cfg[3:])
    A, B = synth.make_config(num)
    t0 = time.time()
    r = oracle.solve(method, A.to_scipy(), B, tol=1e-8, maxit=2000, record=0)
    path = os.path.join(ROOT, "tests", "golden", "oracle_counts.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[f"{cfg}:{method}"] = {"inputs_hash": synth.input_hash(A, B), "outcome": r.outcome,
                               "iterations": r.iterations, "half_step": r.half_step,
                               "final_true_rel_residual": r.final_true_rel_residual,
                               "tol": 1e-8, "maxit": 2000, "oracle_seconds": round(time.time() - t0, 1)}
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    print(cfg, method, data[f"{cfg}:{method}"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
