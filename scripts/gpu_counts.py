"""GPU iteration counts of eGl-QMR (config 3's operator and right-hand sides at m^3, s = 16, seed 2)
under the library's alternative product kernels (plane-marching / banded / CSR SpMM): the GPU side of
the count-ensemble study (the oracle side: scripts/oracle_counts.py m<k> egl_qmr [seq|rev|pert<i>]).
    python scripts/gpu_counts.py 96 128 256
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = """
import sys; sys.path.insert(0, {root!r})
import torch, synth, paper_1504_04395_b200 as srk
srk.load_library()
if {cfg} == 3:
    A = synth.conv_diff_3d({m}, (50.0, 30.0, 10.0)); B = synth.random_rhs(A.n, 16, 2)
else:
    A, B = synth.make_config({cfg}, m={m})
M = srk.Matrix.from_csr(A, need_adjoint=True)
sv = srk.Solver(M, B.shape[1], {method!r}, tol=1e-8, maxit=2000, poll_every=8)
sv.start(torch.from_numpy(B).cuda())
sv.iterate(2000)
rep = sv.report()
h = sv.history(rep.iterations)
cross = [next((k + 1 for k, v in enumerate(h) if v <= 10.0 ** -j), None) for j in range(1, 9)]
print(rep.outcome, rep.iterations, rep.final_true_rel_residual, "crossings", cross)
"""
method = os.environ.get("COUNT_METHOD", "egl_qmr")
cfg = int(os.environ.get("COUNT_CFG", "3"))  # 3: config 3's operator at m^3 (s = 16); else make_config(cfg, m=m)
for m in sys.argv[1:]:
    for env in ({}, {"SRK_BAND_PLANE": "0"}, {"SRK_NO_BAND": "1"}, {"SRK_NO_DMMA_UPDATE": "1"}, {"SRK_GRAM_CTA": "1"}):
        out = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT, m=int(m), method=method, cfg=cfg)],
                             env={**os.environ, **env}, capture_output=True, text=True)
        print(m, method, env or "default", out.stdout.strip() or out.stderr[-300:], flush=True)
