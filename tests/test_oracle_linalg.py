"""Pins for the oracle's block primitives (oracle/linalg.py) against textbook
identities and library routines — never against a retyped copy of the formula."""
import numpy as np
import pytest

from oracle import linalg as L


def _rand(rng, n, s, cplx):
    X = rng.standard_normal((n, s))
    if cplx:
        X = X + 1j * rng.standard_normal((n, s))
    return X


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("order", ["blas", "seq", "rev"])
def test_trace_flattening_identity(rng, cplx, order):
    """<x, y> = tr(Y^H X) with X = mat(x): the trace inner product of
    two blocks equals the plain vector dot product of their column stacks."""
    X, Y = _rand(rng, 37, 5, cplx), _rand(rng, 37, 5, cplx)
    x, y = X.ravel(order="F"), Y.ravel(order="F")
    assert abs(L.trace_inner(X, Y, order=order) - np.dot(y.conj(), x)) <= 1e-13 * np.linalg.norm(x) * np.linalg.norm(y)


@pytest.mark.parametrize("cplx", [False, True])
def test_sum_rank1_identity(rng, cplx):
    """tr(1 r̂^H R) = sum(r̂^H R): sum_inner equals the trace inner
    product against the rank-1 block r̂ 1^T."""
    R = _rand(rng, 29, 4, cplx)
    r = _rand(rng, 29, 1, cplx)[:, 0]
    Rh = np.repeat(r[:, None], 4, axis=1)
    assert abs(L.sum_inner(r, R) - L.trace_inner(R, Rh)) <= 1e-13 * np.linalg.norm(R) * np.linalg.norm(Rh)


@pytest.mark.parametrize("order", ["blas", "seq"])
def test_gram_orthonormal_and_s1(rng, order):
    """Orthonormal X gives Y^H X = I (SPEC block_gram S:94); s=1 is np.vdot."""
    Q, _ = np.linalg.qr(_rand(rng, 50, 6, True))
    assert np.allclose(L.gram(Q, Q, order=order), np.eye(6), atol=1e-14)
    x, y = _rand(rng, 50, 1, True), _rand(rng, 50, 1, True)
    assert abs(L.gram(y, x, order=order)[0, 0] - np.vdot(y[:, 0], x[:, 0])) < 1e-12
    # Gram vs the full trace: tr(Y^H X) = trace(gram)
    X, Y = _rand(rng, 50, 3, True), _rand(rng, 50, 3, True)
    assert abs(np.trace(L.gram(Y, X, order=order)) - np.vdot(Y.ravel(), X.ravel())) < 1e-11


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("order", ["blas", "seq"])
def test_thin_qr_vs_lapack(rng, cplx, order):
    """Thin QR with real non-negative diagonal is unique (reading G10): MGS2 must
    equal LAPACK Householder QR after phase normalisation; orthonormality and
    reconstruction bounds of SPEC thin_qr."""
    Z = _rand(rng, 60, 7, cplx)
    Q, C = L.thin_qr(Z, order=order)
    Ql, Rl = np.linalg.qr(Z)
    ph = np.diag(Rl) / np.abs(np.diag(Rl))
    Ql, Rl = Ql * ph[None, :], Rl * ph.conj()[:, None]
    assert np.allclose(Q, Ql, atol=1e-12) and np.allclose(C, Rl, atol=1e-12)
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(7)) <= 1e-13
    assert np.linalg.norm(Q @ C - Z) / np.linalg.norm(Z) <= 1e-14
    assert np.allclose(np.tril(C, -1), 0) and np.all(np.diag(C).real > 0) and np.allclose(np.diag(C).imag, 0)


def test_thin_qr_rank_deficient(rng):
    """[w | 2w] is rank deficient -> Breakdown('rank') (reading G11)."""
    w = rng.standard_normal((20, 1))
    with pytest.raises(L.Breakdown) as e:
        L.thin_qr(np.hstack([w, 2 * w]))
    assert e.value.kind == "rank"


def test_small_solve(rng):
    """LU-with-pivoting solve residual; singular Gram breaks down."""
    G = _rand(rng, 4, 4, True) + 4 * np.eye(4)
    M = _rand(rng, 4, 3, True)
    Zs = L.small_solve(G, M)
    assert np.linalg.norm(G @ Zs - M) <= 1e-12 * np.linalg.norm(M)
    assert np.allclose(L.small_solve(2 * np.eye(3), np.eye(3)), 0.5 * np.eye(3))
    Gh = L.small_solve_h(G, M)
    assert np.linalg.norm(G.conj().T @ Gh - M) <= 1e-12 * np.linalg.norm(M)
    with pytest.raises(L.Breakdown):
        L.small_solve(np.array([[1.0, 2.0], [2.0, 4.0]]), np.eye(2))


def test_unitary_qr_stack(rng):
    """M = Omega [R; 0] with Omega unitary and diag(R) real positive (App. A.3)."""
    M = _rand(rng, 8, 4, True)
    Om, R = L.unitary_qr_stack(M)
    assert np.linalg.norm(Om.conj().T @ Om - np.eye(8)) < 1e-13
    full = np.vstack([R, np.zeros((4, 4))])
    assert np.linalg.norm(Om @ full - M) < 1e-13
    assert np.all(np.diag(R).real > 0) and np.allclose(np.diag(R).imag, 0)


def test_cholqr2_alternative_equals_mgs2():
    """The oracle's alternative thin QR (CholQR2, order="cholqr", used only to measure the
    method's spread under the QR algorithm — reading G10) returns the same unique thin QR
    with real positive diagonal as MGS2, and detects rank deficiency."""
    import synth
    from oracle.linalg import Breakdown, thin_qr
    for cplx in (False, True):
        Z = synth.random_rhs(300, 6, 4, cplx)
        Q1, C1 = thin_qr(Z)
        Q2, C2 = thin_qr(Z, order="cholqr")
        assert np.linalg.norm(Q1 - Q2) < 1e-12 and np.linalg.norm(C1 - C2) < 1e-12 * np.linalg.norm(C1)
        assert np.all(np.diag(C2).real > 0) and np.allclose(np.diag(C2).imag, 0)
        Z[:, 5] = Z[:, 0] + Z[:, 1]
        with pytest.raises(Breakdown):
            thin_qr(Z, order="cholqr")
