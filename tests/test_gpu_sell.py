"""SELL-32-sigma form (SURVEY §8(a) a0 "convert to SELL-C-sigma"; srk_matrix_sell_info): built for
irregular operators, used by narrow products (s * esz <= 32 B, one row per lane). The product and
every fused reduction against scipy / the oracle on power-law rows (ragged row count, empty rows,
rows longer than a chunk's neighbours), real and complex, A and A^H; the format's bookkeeping."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle.linalg as OL
import synth
from tests.gpu_util import rel, to_dev, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def srk():
    import paper_1504_04395_b200 as srk
    srk.load_library()
    return srk


def _power_law(n, seed, cplx):
    """Power-law rows (synth.power_law) with some rows emptied; complex values optionally."""
    A = synth.power_law(n, seed=seed).to_scipy().tolil()
    rng = np.random.default_rng(seed)
    for r in rng.choice(n, size=max(1, n // 50), replace=False):
        A.rows[r], A.data[r] = [], []
    A = A.tocsr()
    if cplx:
        A = A.astype(np.complex128)
        A.data = A.data * np.exp(1j * rng.uniform(0, 2 * np.pi, A.nnz))
    A.sort_indices()
    return A


def _rand(rng, n, s, cplx):
    X = rng.standard_normal((n, s))
    return X + 1j * rng.standard_normal((n, s)) if cplx else X


@pytest.mark.parametrize("n", [4099, 70001])
def test_sell_built_for_irregular_rows(srk, n):
    A = _power_law(n, 3, False)
    M = srk.Matrix.from_csr(A)
    info = M.sell_info()
    assert info is not None, "power-law rows must get the SELL form"
    nchunk, entries, sigma = info
    assert nchunk == (n + 31) // 32 and entries % 32 == 0
    assert A.nnz <= entries <= 1.25 * A.nnz  # padding bound of the build
    # a stencil stays out of the SELL form
    S = srk.Matrix.from_csr(synth.conv_diff_2d(20, (20.0, 20.0)))
    assert S.sell_info() is None


@pytest.mark.parametrize("cplx,s", [(False, 1), (False, 2), (False, 3), (False, 4), (True, 1), (True, 2)])
@pytest.mark.parametrize("n", [4099, 70001])
def test_sell_product_and_reductions(srk, n, s, cplx):
    A = _power_law(n, 7 + s, cplx)
    M = srk.Matrix.from_csr(A)
    assert M.sell_info() is not None
    rng = np.random.default_rng(s)
    P, Y = _rand(rng, n, s, cplx), _rand(rng, n, s, cplx)
    ref = A @ P
    scale = max(1.0, np.max(np.abs(ref)))
    Q = to_np(srk.spmm_block(M, to_dev(P)))
    assert np.max(np.abs(Q - ref)) <= 1e-13 * scale
    refH = A.conj().T @ P
    QH = to_np(srk.spmm_block(M, to_dev(P), adjoint=True))
    assert np.max(np.abs(QH - refH)) <= 1e-13 * max(1.0, np.max(np.abs(refH)))
    expect = {"trace": lambda: np.array([OL.trace_inner(ref, Y)]), "norm2": lambda: np.array([OL.fro2(ref)]),
              "colnorm2": lambda: np.sum(np.abs(ref) ** 2, axis=0), "diag": lambda: OL.col_inner(ref, Y),
              "sumvec": lambda: np.array([OL.sum_inner(Y[:, 0], ref)]), "full": lambda: OL.gram(Y, ref)}
    for mode, fn in expect.items():
        Yd = to_dev(Y[:, 0].copy()) if mode == "sumvec" else to_dev(Y)
        Q2, g = srk.spmm_block(M, to_dev(P), gram=mode, Y=Yd)
        assert np.array_equal(to_np(Q2), Q), mode  # the epilogue does not change the product
        e = fn()
        assert rel(to_np(g).reshape(e.shape), e) < 1e-11, mode


def test_sell_row_sum_order(srk):
    """One row per lane sums its entries in CSR order (the team-per-row kernel's butterfly does
    not): rows with one entry are exact products, every row within one rounding per term of the
    sequential sum."""
    n = 4099
    A = _power_law(n, 11, False).tolil()
    for r in range(5, n, 97):           # some rows with exactly one entry
        A.rows[r], A.data[r] = [int(r * 31 % n)], [1.0 + r / n]
    A = A.tocsr()
    A.sort_indices()
    M = srk.Matrix.from_csr(A)
    assert M.sell_info() is not None
    p = np.random.default_rng(0).standard_normal((n, 1))
    q = to_np(srk.spmm_block(M, to_dev(p)))[:, 0]
    lens = np.diff(A.indptr)
    seq = np.array([sum(A.data[j] * p[A.indices[j], 0] for j in range(A.indptr[i], A.indptr[i + 1])) for i in range(n)])
    one = lens == 1
    assert one.any() and np.array_equal(q[one], seq[one])
    mag = np.abs(A) @ np.abs(p[:, 0])
    assert np.all(np.abs(q - seq) <= 2.3e-16 * lens * mag)


@pytest.mark.parametrize("cplx,s", [(False, 1), (False, 2), (False, 3), (False, 4), (True, 1), (True, 2)])
@pytest.mark.parametrize("maxlen", [12, 29, 200])
def test_team_kernel_unsorted_variable_rows(srk, maxlen, s, cplx):
    """Narrow products on an operator with long but REGULAR row lengths (mean >= 12: the
    team-per-row kernel on the unsorted CSR, no SELL form): rows of differing lengths inside one
    team. The 16-byte two-rows-per-team instance faulted here (ptxas -O3; scripts/team_probe.cu)."""
    n = 4099
    rng = np.random.default_rng(maxlen)
    lens = rng.integers(maxlen // 2 + 6, maxlen + 1, n)      # max < 4 mean + 8: regular
    rp = np.concatenate([[0], np.cumsum(lens)])
    ci = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens])
    va = rng.standard_normal(rp[-1]) + (1j * rng.standard_normal(rp[-1]) if cplx else 0)
    A = sp.csr_matrix((va, ci, rp), shape=(n, n))
    M = srk.Matrix.from_csr(A)
    assert M.sell_info() is None and M.format()[0] == "csr"
    P = _rand(rng, n, s, cplx)
    for adj in (False, True):
        ref = (A.conj().T if adj else A) @ P
        Q = to_np(srk.spmm_block(M, to_dev(P), adjoint=adj))
        assert np.max(np.abs(Q - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))), adj
