"""Config 5 SpMM+Gram sweep (SURVEY §8(d).3 / BASELINE.json configs[4]): the power-law
operator (n = 2^22, ~67M nnz, uniform columns) times an n x s block for
s in {1, 2, 4, 8, 16, 32, 64}, alone and with the full s x s Gram Y^H (A P)
(fused into the SpMM epilogue for s <= 16, DMMA tensor-core Gram kernel after the
SpMM for s > 16), plus the standalone DMMA Gram. Times with CUDA events on the
library's stream (torch's current stream), warm, median of 10; writes
profiles/<tag>_cfg5_sweep.json.

    python scripts/sweep_cfg5.py r01
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1504_04395_b200 as srk  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main(tag):
    srk.load_library()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    A = synth.power_law(1 << 22, seed=4)
    M = srk.Matrix.from_csr(A, need_adjoint=False)
    n, nnz = A.n, A.nnz
    rows = []
    for s in (1, 2, 4, 8, 16, 32, 64):
        P = torch.from_numpy(synth.random_rhs(n, s, 4)).cuda()
        Y = torch.from_numpy(synth.random_rhs(n, s, 5)).cuda()
        Q = torch.empty_like(P)
        a_bytes = (n + 1) * 4 + nnz * 12
        b_spmm = a_bytes + 2 * n * s * 8           # A once, P read once, Q written once
        t_spmm = timed(lambda: srk.spmm_block(M, P, Q=Q))
        t_full = timed(lambda: srk.spmm_block(M, P, gram="full", Y=Y, Q=Q))
        t_gram = timed(lambda: srk.gram_block(Q, Y, "full"))
        flops = 2.0 * n * s * s
        b_full = b_spmm + n * s * 8                # + the Gram operand Y
        rows.append({
            "s": s, "spmm_ms": t_spmm, "spmm_gbs": b_spmm / t_spmm / 1e6, "spmm_frac": b_spmm / t_spmm / 1e6 / peak,
            "spmm_gram_ms": t_full, "spmm_gram_gbs": b_full / t_full / 1e6,
            "spmm_gram_frac": b_full / t_full / 1e6 / peak,
            "gram_path": "fused epilogue (FMA)" if s <= 16 else "SpMM + DMMA Gram kernel",
            "gram_only_ms": t_gram, "gram_only_tflops": flops / t_gram / 1e9,
            "gram_only_gbs": 2 * n * s * 8 / t_gram / 1e6,
        })
        print(json.dumps(rows[-1]), flush=True)
    out = {"config": "cfg5 power-law n=2^22 (synth.power_law seed 4)", "n": n, "nnz": nnz,
           "peak_hbm_gbs": peak, "dmma_peak_tflops_measured": 37.1, "rows": rows}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", f"{tag}_cfg5_sweep.json"), "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
