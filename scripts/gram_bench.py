"""Times srk_gram_block (FULL) on n x s blocks resident in HBM (each larger than L2):
distinct operands and X == Y, reporting algorithmic GB/s (the operand bytes read once).
Tuning aid: SRK_GRAM_CTA=1 switches narrow widths to the CTA-tiled kernel.

    python scripts/gram_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1504_04395_b200 as srk  # noqa: E402

srk.load_library()
n = 1 << 21
for cplx, s in ((True, 8), (False, 8), (False, 16), (True, 16), (False, 32)):
    dt = torch.complex128 if cplx else torch.float64
    X = torch.randn(n, s, dtype=dt, device="cuda")
    Y = torch.randn(n, s, dtype=dt, device="cuda")
    for same in (False, True):
        Yo = X if same else Y
        for _ in range(3):
            srk.gram_block(X, Yo, "full")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        K = 20
        for _ in range(K):
            srk.gram_block(X, Yo, "full")
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        byts = X.numel() * X.element_size() * (1 if same else 2)
        print(f"{'c128' if cplx else 'f64'} s={s:2d} same={int(same)}  {ms * 1e3:7.1f} us  {byts / ms / 1e6:7.0f} GB/s", flush=True)
