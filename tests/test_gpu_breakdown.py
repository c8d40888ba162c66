"""Breakdown parity on the GPU (SURVEY §5 "forcing singular Grams in unit tests"): the
GPU's outcome, breakdown kind, breakdown iteration and frozen columns must equal the
oracle's when a Lanczos denominator vanishes, an s x s Gram is
singular, the residual block is rank deficient (reading G11) or one Li
column meets a Lanczos zero (reading G13). The inputs are integer-valued so the
vanishing quantities are EXACT zeros in floating point, whatever the summation order."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth
from tests.gpu_util import rel, to_dev, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def srk():
    import paper_1504_04395_b200 as srk
    srk.load_library()
    return srk


def _skew(n, seed):
    """Integer skew-symmetric CSR: x^T S x = 0 exactly for every integer x."""
    rng = np.random.default_rng(seed)
    T = sp.random(n, n, density=6.0 / n, random_state=seed, data_rvs=lambda k: rng.integers(1, 4, k).astype(float))
    S = sp.triu(T, 1) - sp.triu(T, 1).T
    S = S.tocsr()
    S.sort_indices()
    return S


def _gpu(srk, A, B, method, maxit=50):
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    X, rep = srk.solve(M, to_dev(B), method, tol=1e-10, maxit=maxit)
    return to_np(X), rep


def _assert_same_breakdown(rep, a):
    assert a.outcome == "breakdown", (a.outcome, a.iterations)
    assert rep.outcome == "breakdown", rep
    assert rep.breakdown_kind == a.breakdown_kind, (rep.breakdown_kind, a.breakdown_kind)
    assert rep.breakdown_iter == a.breakdown_iter, (rep.breakdown_iter, a.breakdown_iter)


@pytest.mark.parametrize("method", ["gl_bicg", "egl_bicg", "li_bicg", "gl_bicgstab"])
def test_lanczos_zero(srk, method):
    """A skew-symmetric operator with integer right-hand sides: <A P, R̂> = tr(R^T S R) = 0
    at the first iteration (s = 4 columns; the economic mean r̂ = R 1 / 4 is dyadic, so
    sum(r̂^T S R) = 4 r̂^T S r̂ = 0 exactly too). For Li every column freezes: breakdown."""
    n, s = 400, 4
    A = _skew(n, 3)
    B = np.random.default_rng(5).integers(-3, 4, (n, s)).astype(float)
    a = oracle.solve(method, A, B, tol=1e-10, maxit=50, record=0)
    X, rep = _gpu(srk, A, B, method)
    _assert_same_breakdown(rep, a)
    assert rel(X, a.X) <= 1e-12


@pytest.mark.parametrize("method", ["bl_bicg", "bl_bicgstab"])
def test_singular_gram(srk, method):
    """Two identical right-hand sides: every s x s Gram of the block methods is exactly
    singular (identical rows / columns give an exactly zero LU pivot)."""
    A = synth.conv_diff_3d(8).to_scipy()
    B = synth.random_rhs(A.shape[0], 3, 4)
    B[:, 2] = B[:, 0]
    a = oracle.solve(method, A, B, tol=1e-10, maxit=50, record=0)
    X, rep = _gpu(srk, A, B, method)
    _assert_same_breakdown(rep, a)


@pytest.mark.parametrize("method", ["bl_bicg_rq", "bl_bicgstab_rq", "bl_qmr"])
def test_rank_deficient_residual(srk, method):
    """The QR-normalised variants' thin QR of a rank-deficient R0 (a column that is the sum of two
    others, integer-valued): BREAKDOWN(rank) at the start (reading G11)."""
    A = synth.conv_diff_3d(8).to_scipy()
    n = A.shape[0]
    B = np.random.default_rng(7).integers(-3, 4, (n, 3)).astype(float)
    B[:, 2] = B[:, 0] + B[:, 1]
    a = oracle.solve(method, A, B, tol=1e-10, maxit=50, record=0)
    X, rep = _gpu(srk, A, B, method)
    _assert_same_breakdown(rep, a)


@pytest.mark.parametrize("cplx", [False, True])
def test_li_column_freeze(srk, cplx):
    """Li-BiCG on blockdiag(S, M): column 0 meets an exact Lanczos zero at iteration 1 and
    freezes (reading G13) while column 1 keeps iterating; the frozen column set, the X
    columns and the per-column iterates match the oracle."""
    rng = np.random.default_rng(21)
    m = 6
    Sk = np.triu(rng.integers(-3, 4, (m, m)), 1).astype(float)
    Sk = Sk - Sk.T
    Mb = synth.random_sparse(40, 4, 5, np.complex128 if cplx else np.float64, 0.8).to_scipy()
    A = sp.block_diag([sp.csr_matrix(Sk), Mb], format="csr")
    A.sort_indices()
    B = np.zeros((m + 40, 2), dtype=np.complex128 if cplx else np.float64)
    B[:m, 0] = rng.integers(-4, 5, m)
    B[:, 1] = synth.random_rhs(m + 40, 1, 8, cplx)[:, 0]
    k = 10
    a = oracle.solve("li_bicg", A, B, tol=1e-300, maxit=k, record=k)
    assert a.breakdown_cols == [0]
    M = srk.Matrix.from_csr(A)
    sv = srk.Solver(M, 2, "li_bicg", tol=1e-300, maxit=k, poll_every=1, check_true_residual=False)
    sv.start(to_dev(B))
    for it in range(k):
        sv.iterate(1)
        X = to_np(sv.x())
        assert np.all(X[:, 0] == 0)
        assert rel(X[:, 1], a.Xs[it][:, 1]) <= 1e-10, it
    assert sv.report().frozen_cols == len(a.breakdown_cols)
    sv.close()
