"""Iteration counts of one full-size configuration under the library's alternative
reduction / update orders (tensor-core vs CUDA-core updates, Gram kernel choice):
the GPU's own rounding spread, next to the oracle's cached count.
    python scripts/count_spread.py 2 bl_bicgstab_rq
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = f"""
import sys; sys.path.insert(0, {ROOT!r})
import torch, synth, paper_1504_04395_b200 as srk
srk.load_library()
A, B = synth.make_config({int(sys.argv[1])})
M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[{sys.argv[2]!r}])
X, rep = srk.solve(M, torch.from_numpy(B).cuda(), {sys.argv[2]!r}, tol=1e-8, maxit=2000)
print(rep.outcome, rep.iterations, rep.final_true_rel_residual)
"""
for env in ({}, {"SRK_NO_DMMA_UPDATE": "1"}, {"SRK_GRAM_CTA": "1"}, {"SRK_NO_DMMA_UPDATE": "1", "SRK_GRAM_CTA": "1"}):
    out = subprocess.run([sys.executable, "-c", CODE], env={**os.environ, **env}, capture_output=True, text=True)
    print(env or "default", out.stdout.strip() or out.stderr[-300:], flush=True)
