"""Helpers shared by the -m gpu parity tests (no method arithmetic here)."""
import numpy as np


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def to_np(t):
    return t.detach().cpu().numpy()


def csr_with_empty_rows(n, seed, cplx=False):
    """A ragged CSR: every 7th row empty, others with 0..9 random sorted columns."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(n):
        if i % 7 == 3:
            continue
        k = int(rng.integers(0, 10))
        c = np.unique(rng.integers(0, n, k))
        rows += [i] * len(c)
        cols += list(c)
    import scipy.sparse as sp
    v = rng.standard_normal(len(rows))
    if cplx:
        v = v + 1j * rng.standard_normal(len(rows))
    A = sp.csr_matrix((v, (np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64))), shape=(n, n))
    A.sort_indices()
    return A
