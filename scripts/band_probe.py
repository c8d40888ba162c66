"""One config-3 banded SpMM (s = 16, eGl vector-sum epilogue) for an ncu capture, plus
CUDA-event timings of the band and CSR paths (SRK_NO_BAND is read at operator creation)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1504_04395_b200 as srk  # noqa: E402

m = int(os.environ.get("BAND_M", "256"))
s = int(os.environ.get("BAND_S", "16"))
reps = int(os.environ.get("BAND_REPS", "5"))
cplx = os.environ.get("BAND_CPLX") == "1"
A = synth.conv_diff_3d(m, (50.0, 30.0, 10.0), np.complex128, -0.1j) if cplx else synth.conv_diff_3d(m, (50.0, 30.0, 10.0))
dt = torch.complex128 if cplx else torch.float64
M = srk.Matrix.from_csr(A, need_adjoint=True)
print("format", M.format(), flush=True)
g = torch.Generator(device="cuda").manual_seed(1)
P = torch.randn((A.n, s), dtype=dt, device="cuda", generator=g)
y = torch.randn((A.n,), dtype=dt, device="cuda", generator=g)
Q = torch.empty_like(P)
for gram in ("none", "sumvec", "adjoint"):
    adj = gram == "adjoint"
    gram = "none" if adj else gram
    for _ in range(2):
        srk.spmm_block(M, P, adjoint=adj, gram=gram, Y=y if gram != "none" else None, Q=Q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        srk.spmm_block(M, P, adjoint=adj, gram=gram, Y=y if gram != "none" else None, Q=Q)
    e1.record()
    torch.cuda.synchronize()
    print(f"{M.format()[0]} gram={gram}{' adjoint' if adj else ''}: {e0.elapsed_time(e1) / reps:.3f} ms", flush=True)
