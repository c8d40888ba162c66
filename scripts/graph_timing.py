"""Config 1 (n = 1024, latency-bound): solve time with and without CUDA-graph replay."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1504_04395_b200 as srk
A, B = synth.make_config(1)
for method in ("egl_bicg", "bl_bicgstab_rq"):
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    Bd = torch.from_numpy(B).cuda()
    for g in (False, True):
        for poll in (8, 32):
            best = 1e9
            for rep in range(5):
                sv = srk.Solver(M, 4, method, tol=1e-8, poll_every=poll, use_graph=g)
                sv.start(Bd)
                torch.cuda.synchronize()
                t = time.perf_counter()
                sv.iterate(2000)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t)
                r = sv.report()
                sv.close()
            print(f"{method:16s} graph={int(g)} poll={poll:3d} iters={r.iterations} {1e3*best:.2f} ms  "
                  f"{1e6*best/r.iterations:.1f} us/it  {4*r.iterations/best:.0f} RHS*it/s")
