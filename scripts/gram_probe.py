"""One DMMA Gram launch (n = 2^22, s = 64, real) for the ncu capture of gram_mma_kernel
(scripts/gpu_ncu_gram.sh); checks the result against numpy on a few entries."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1504_04395_b200 as srk  # noqa: E402
import synth  # noqa: E402

srk.load_library()
Xh, Yh = synth.random_rhs(1 << 22, 64, 4), synth.random_rhs(1 << 22, 64, 5)
X, Y = torch.from_numpy(Xh).cuda(), torch.from_numpy(Yh).cuda()
g = srk.gram_block(X, Y, "full").cpu().numpy().reshape(64, 64)
ref = Yh[:, :2].T @ Xh[:, :2]
assert np.allclose(g[:2, :2], ref, rtol=1e-10, atol=1e-8)
print("ok")
