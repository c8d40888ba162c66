"""Wall time of ILU(0)-preconditioned solves of the paper's examples (second of two
identical solves, device-synchronised): A/B for the triangular-solve kernels
(SRK_TRSV_LEVELS=1: one launch per level)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1504_04395_b200 as srk  # noqa: E402
import synth  # noqa: E402

srk.load_library()
tag = "levels" if os.environ.get("SRK_TRSV_LEVELS") else "syncfree"
for ex in ("ex1", "ex2", "ex3"):
    A, B = synth.paper_ex1(200) if ex == "ex1" else synth.paper_ex2(50, 1000.0 if ex == "ex2" else 10.0)
    Q = np.ascontiguousarray(np.linalg.qr(B)[0])
    M = srk.Matrix.from_csr(A, need_adjoint=True).ilu0()
    Bd = torch.from_numpy(Q).cuda()
    for m in ("bl_bicgstab_rq", "egl_bicg"):
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            X, r = srk.solve(M, Bd, m, tol=1e-10, maxit=500)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"{tag} {ex} {m:15s} it {r.iterations:4d} {dt * 1e3:8.1f} ms  {dt * 1e3 / max(1, r.iterations):7.3f} ms/it", flush=True)
