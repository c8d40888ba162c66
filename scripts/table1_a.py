"""Table 1's acceleration factor a on B200: the time of s single
matrix-vector products divided by the time of one matrix-block product with s columns,
unpreconditioned and with the right ILU(0) preconditioner (one preconditioned product =
M^-1 then A), on the paper's Ex. 1 (200^2, s = 4) and Ex. 2/3 operators (50^3, s = 19),
next to the paper's Matlab / i7-4770 values (a = 2.65 / 1.21, 2.66 / 1.69, 2.60 / 1.71).
CUDA events, median of 20 after warm-up. Writes profiles/<tag>_table1_a.json.

    python scripts/table1_a.py r02
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

PAPER = {"ex1": (2.65, 1.21), "ex2": (2.66, 1.69), "ex3": (2.60, 1.71)}


def med_ms(fn, reps=20):
    for _ in range(3):
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
    out = {}
    for ex in ("ex1", "ex2", "ex3"):
        if ex == "ex1":
            A, B = synth.paper_ex1(200)
        else:
            A, B = synth.paper_ex2(50, 1000.0 if ex == "ex2" else 10.0)
        s = B.shape[1]
        M = srk.Matrix.from_csr(A)
        Mi = srk.Matrix.from_csr(A).ilu0()
        P = torch.from_numpy(np.ascontiguousarray(B)).cuda()
        cols = [P[:, j:j + 1].contiguous() for j in range(s)]
        Q = torch.empty_like(P)
        q1 = torch.empty_like(cols[0])
        z1 = torch.empty_like(cols[0])
        Z = torch.empty_like(P)

        def singles():
            for c in cols:
                srk.spmm_block(M, c, Q=q1)

        def block():
            srk.spmm_block(M, P, Q=Q)

        def singles_prec():
            for c in cols:
                z = srk.precond_apply(Mi, c)
                srk.spmm_block(M, z, Q=q1)

        def block_prec():
            z = srk.precond_apply(Mi, P)
            srk.spmm_block(M, z, Q=Q)

        t1, tb = med_ms(singles), med_ms(block)
        t1p, tbp = med_ms(singles_prec), med_ms(block_prec)
        out[ex] = {"n": A.n, "nnz": A.nnz, "s": s, "a_noprec": t1 / tb, "a_prec": t1p / tbp,
                   "ms_s_singles": t1, "ms_block": tb, "ms_s_singles_prec": t1p, "ms_block_prec": tbp,
                   "paper_a_noprec": PAPER[ex][0], "paper_a_prec": PAPER[ex][1],
                   "rho": s * A.n / A.nnz}
        print(ex, out[ex], flush=True)
    out["note"] = ("B200 times with CUDA events (median of 20): the paper's a (P:679-686) measured Matlab on an "
                   "i7-4770; on the GPU these desk-size products are launch/latency-bound, so a measures how "
                   "many single products one block launch replaces")
    json.dump(out, open(os.path.join(ROOT, "profiles", f"{tag}_table1_a.json"), "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
