"""Pins of the oracle's ILU(0) and right preconditioning (oracle/precond.py;
PAPER.md P:670-676)."""
import numpy as np
import pytest
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


# ------------------------------------------------------------------ ILUTP (R14)
def test_ilutp_without_dropping_equals_lapack_lu():
    """droptol = 0, thresh = 1 is LU with partial pivoting: the same P, L, U as LAPACK's
    getrf (scipy.linalg.lu) on a dense real matrix (no ties in |x|)."""
    import scipy.linalg as sla
    rng = np.random.default_rng(11)
    A = rng.standard_normal((40, 40))
    L, U, perm = OP.ilutp(sp.csr_matrix(A), 0.0)
    Pm, Ls, Us = sla.lu(A)
    assert np.array_equal(np.argmax(Pm, axis=0), perm)  # A = Pm L U: row perm[k] of A is row k of L U
    assert np.max(np.abs(L.toarray() - Ls)) < 1e-13 and np.max(np.abs(U.toarray() - Us)) < 1e-12


def test_ilutp_complex_exact_lu_and_bounded_multipliers():
    """Complex, droptol = 0: A[perm] = L U to rounding, L unit lower, U upper, and every
    multiplier |l_ij| <= 1 (the pivot is the largest candidate)."""
    rng = np.random.default_rng(12)
    A = rng.standard_normal((30, 30)) + 1j * rng.standard_normal((30, 30))
    L, U, perm = OP.ilutp(sp.csr_matrix(A), 0.0)
    Ld, Ud = L.toarray(), U.toarray()
    assert np.allclose(np.diag(Ld), 1) and np.all(np.triu(Ld, 1) == 0) and np.all(np.tril(Ud, -1) == 0)
    assert np.max(np.abs(A[perm] - Ld @ Ud)) < 1e-12 * np.max(np.abs(A))
    assert np.max(np.abs(np.tril(Ld, -1))) <= 1.0
    assert sorted(perm.tolist()) == list(range(30))


def _pivoting_sparse(n, seed, cplx=False):
    """Sparse, nonsymmetric, weak diagonal (so partial pivoting moves rows)."""
    rng = np.random.default_rng(seed)
    A = sp.random(n, n, density=6.0 / n, random_state=rng, format="csr")
    if cplx:
        A = A + 1j * sp.random(n, n, density=6.0 / n, random_state=rng, format="csr")
    A = A + sp.diags(0.05 * rng.standard_normal(n)) + sp.diags(np.ones(n - 1), -1)
    A = sp.csr_matrix(A)
    A.sort_indices()
    return A


@pytest.mark.parametrize("cplx", [False, True])
def test_ilutp_residual_is_exactly_the_dropped_entries(cplx):
    """Pi A - L U consists of the dropped entries only: below droptol ||A(:, j)|| in column j,
    and none at a position L or U stores (there the residual is rounding); every stored
    off-diagonal entry passed the drop test (|u_kj| >= tol_j, |l_ij u_jj| >= tol_j);
    multipliers bounded by 1."""
    A = _pivoting_sparse(150, 5, cplx)
    tolr = 5e-2
    L, U, perm = OP.ilutp(A, tolr)
    assert np.any(perm != np.arange(150))  # pivoting happened
    Ad = A.toarray()
    Ld, Ud = L.toarray(), U.toarray()
    R = Ad[perm] - Ld @ Ud
    tol = tolr * np.linalg.norm(Ad, axis=0)
    stored = (np.tril(Ld, -1) != 0) | (Ud != 0)
    scale = np.max(np.abs(Ad))
    assert np.max(np.abs(R[stored])) < 1e-12 * scale
    assert np.all(np.abs(R) < tol[None, :] + 1e-12 * scale)
    assert np.any(np.abs(R) > 1e-12 * scale)  # something was dropped
    off_u = np.triu(Ud, 1)
    assert np.all(np.abs(off_u[off_u != 0]) >= tol[np.nonzero(off_u)[1]])
    Ls = np.tril(Ld, -1)
    i, j = np.nonzero(Ls)
    assert np.all(np.abs(Ls[i, j] * np.diag(Ud)[j]) >= tol[j] * (1 - 1e-14))
    assert np.max(np.abs(Ls)) <= 1.0


def test_ilutp_thresh0_keeps_the_diagonal():
    """thresh = 0 never pivots while the diagonal candidate is nonzero; on a column
    diagonally dominant matrix partial pivoting also keeps it, so both equal LAPACK's LU."""
    import scipy.linalg as sla
    rng = np.random.default_rng(13)
    A = rng.standard_normal((25, 25))
    A += np.diag(np.sum(np.abs(A), axis=0) + 1.0)
    L0, U0, p0 = OP.ilutp(sp.csr_matrix(A), 0.0, thresh=0.0)
    L1, U1, p1 = OP.ilutp(sp.csr_matrix(A), 0.0)
    _, Ls, Us = sla.lu(A)
    assert np.array_equal(p0, np.arange(25)) and np.array_equal(p1, np.arange(25))
    assert np.max(np.abs(L0.toarray() - Ls)) < 1e-13 and np.max(np.abs(U0.toarray() - Us)) < 1e-12
    B = _pivoting_sparse(80, 6)
    _, _, pb = OP.ilutp(B, 5e-2, thresh=0.0)
    assert np.array_equal(pb, np.arange(80)) or np.all(B.diagonal()[pb != np.arange(80)] == 0)


def test_ilutp_apply_inv_against_dense_inverse():
    """M = Pi^T L U: apply_inv = inv(M) P and apply_inv_adj = inv(M)^H P with the permutation
    (a swapped or missing permutation fails)."""
    A = _pivoting_sparse(60, 7, True)
    L, U, perm = OP.ilutp(A, 5e-2)
    Pi = np.eye(60)[perm]
    M = Pi.T @ L.toarray() @ U.toarray()
    Minv = np.linalg.inv(M)
    P = np.random.default_rng(1).standard_normal((60, 3)) + 0j
    ref = Minv @ P
    assert np.max(np.abs(OP.apply_inv(L, U, P, perm) - ref)) < 1e-10 * np.max(np.abs(ref))
    refh = Minv.conj().T @ P
    assert np.max(np.abs(OP.apply_inv_adj(L, U, P, perm) - refh)) < 1e-10 * np.max(np.abs(refh))


def test_ilutp_preconditions_the_lattice():
    """Ex. 4's use: with ILUTP(5e-2) on the lattice operator the preconditioned
    Gl-BiCGStab reaches the tolerance in fewer iterations than without."""
    A = synth.lattice_4d(4, kappa=0.12, seed=3).to_scipy()
    B = synth.random_rhs(A.shape[0], 4, 0, True)
    L, U, perm = OP.ilutp(A, 5e-2)
    pre = OP.solve_right("gl_bicgstab", A, B, L, U, perm, tol=1e-8, maxit=500, record=0)
    plain = oracle.solve("gl_bicgstab", A, B, tol=1e-8, maxit=500, record=0)
    assert pre.outcome == "converged" and plain.outcome == "converged"
    assert pre.iterations < plain.iterations
    assert np.linalg.norm(B - A @ pre.X) <= 1e-8 * np.linalg.norm(B) * 1.01
