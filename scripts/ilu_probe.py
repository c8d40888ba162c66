"""Table 2 (lower half) entries of the unstabilised block methods under right ILU(0):
outcome, iterations and the true residual where they stop (tuning / reading aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1504_04395_b200 as srk  # noqa: E402
import synth  # noqa: E402

srk.load_library()
for ex in ("ex1", "ex2", "ex3"):
    A, B = synth.paper_ex1(200) if ex == "ex1" else synth.paper_ex2(50, 1000.0 if ex == "ex2" else 10.0)
    Q, _ = np.linalg.qr(B)
    Q = np.ascontiguousarray(Q)
    M = srk.Matrix.from_csr(A, need_adjoint=True).ilu0()
    for m in ("bl_bicg", "bl_bicgstab", "bl_bicg_rq", "bl_bicgstab_rq"):
        X, rep = srk.solve(M, torch.from_numpy(Q).cuda(), m, tol=1e-10, maxit=500)
        r = np.linalg.norm(Q - A.to_scipy() @ X.cpu().numpy()) / np.linalg.norm(Q)
        print(ex, m, rep.outcome, rep.iterations, f"{r:.2e}", flush=True)
