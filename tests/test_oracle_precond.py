"""Pins of the oracle's ILU(0) and right preconditioning (oracle/precond.py;
PAPER.md P:670-676)."""
import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

import oracle
import oracle.precond as OP
import synth


def _tridiag(n, lo, d, up):
    return sp.diags([np.full(n - 1, lo), np.full(n, d), np.full(n - 1, up)], [-1, 0, 1], format="csr")


def test_ilu0_of_1d_laplacian_closed_form():
    """tridiag(-1, 2, -1) has no fill: ILU(0) = LU, u_kk = (k+1)/k, l_k+1,k = -k/(k+1)."""
    n = 50
    L, U = OP.ilu0(_tridiag(n, -1.0, 2.0, -1.0))
    k = np.arange(1, n + 1)
    assert np.allclose(U.diagonal(), (k + 1) / k, rtol=0, atol=1e-14)
    assert np.allclose(L.diagonal(-1), -k[:-1] / (k[:-1] + 1), rtol=0, atol=1e-14)


def test_ilu0_equals_lapack_lu_without_fill():
    """A nonsymmetric, complex, diagonally dominant tridiagonal matrix: no fill and no
    pivoting, so ILU(0) must equal LAPACK's LU factors."""
    n = 40
    rng = np.random.default_rng(3)
    A = sp.diags([rng.standard_normal(n - 1) + 1j * rng.standard_normal(n - 1), 5 + rng.random(n),
                  rng.standard_normal(n - 1)], [-1, 0, 1], format="csr")
    L, U = OP.ilu0(A)
    P, Lr, Ur = sla.lu(A.toarray())
    assert np.allclose(P, np.eye(n))
    assert np.max(np.abs(L.toarray() - Lr)) < 1e-14 and np.max(np.abs(U.toarray() - Ur)) < 1e-13


def test_ilu0_matches_a_on_its_pattern():
    """The defining property of ILU(0): (L U)_ij = A_ij for every (i, j) in the pattern of
    A (with fill elsewhere), on a 2D convection-diffusion operator and a random one."""
    for A in (synth.conv_diff_2d(12, (20.0, 10.0)).to_scipy(),
              synth.random_sparse(300, 5, seed=4, dominance=1.5).to_scipy()):
        L, U = OP.ilu0(A)
        LU = (L @ U).tocsr()
        A = A.tocsr()
        A.sort_indices()
        rows = np.repeat(np.arange(A.shape[0]), np.diff(A.indptr))
        got = np.asarray(LU[rows, A.indices]).ravel()
        assert np.max(np.abs(got - A.data)) < 1e-12 * np.max(np.abs(A.data))
        assert (LU - A).nnz > 0  # genuinely incomplete


def test_right_preconditioning_with_exact_factorisation():
    """M = A (ILU(0) exact for a tridiagonal operator): A M^-1 = I, every method
    converges in one iteration to X = A^-1 B."""
    n, s = 60, 3
    A = _tridiag(n, -1.3, 4.0, -0.7)
    B = synth.random_rhs(n, s, 2)
    Xd = np.linalg.solve(A.toarray(), B)
    for method in ("egl_bicg", "gl_bicgstab", "bl_bicg_rq", "li_qmr"):
        r = OP.solve_right(method, A, B, tol=1e-12, maxit=5)
        assert r.outcome == "converged" and r.iterations == 1, (method, r.outcome, r.iterations)
        assert np.max(np.abs(r.X - Xd)) < 1e-12


def test_right_preconditioned_iterates_stay_in_the_preconditioned_space():
    """Right preconditioning keeps the residual B - A X_k the method's residual of
    A M^-1 Y = B, and converges much faster than the plain method on Ex. 1's operator."""
    A, B = synth.paper_ex1(20)
    As = A.to_scipy()
    Q, _ = np.linalg.qr(B)
    plain = oracle.solve("gl_bicgstab", As, Q, tol=1e-10, maxit=500, record=0)
    prec = OP.solve_right("gl_bicgstab", As, Q, tol=1e-10, maxit=500, record=0)
    assert prec.outcome == "converged" and prec.iterations < plain.iterations
    assert np.linalg.norm(Q - As @ prec.X) / np.linalg.norm(Q) <= 1e-10


def test_apply_inv_and_adjoint_against_dense_inverse():
    """M^-1 P and M^-H P (the adjoint products of the BiCG / QMR families under
    right preconditioning, (A M^-1)^H = M^-H A^H) against the dense inverse of the product
    L U of a genuinely incomplete, complex factorisation: the triangular solves must come
    in the order U^-1 L^-1 and L^-H U^-H (swapping either order changes the result)."""
    A = synth.random_sparse(120, 5, seed=9, dtype=np.complex128, dominance=1.5).to_scipy()
    L, U = OP.ilu0(A)
    M = (L @ U).toarray()
    assert np.linalg.norm(M - A.toarray()) > 1e-3  # fill dropped: M != A
    P = synth.random_rhs(120, 3, 5, True)
    Minv = np.linalg.inv(M)
    assert np.max(np.abs(OP.apply_inv(L, U, P) - Minv @ P)) < 1e-11 * np.max(np.abs(Minv @ P))
    ref = Minv.conj().T @ P
    assert np.max(np.abs(OP.apply_inv_adj(L, U, P) - ref)) < 1e-11 * np.max(np.abs(ref))
    # the swapped orders really differ here (the pin is not vacuous)
    wrong = np.linalg.inv((U @ L).toarray()).conj().T @ P
    assert np.max(np.abs(wrong - ref)) > 1e-6 * np.max(np.abs(ref))
