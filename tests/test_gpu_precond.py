"""GPU parity of the right ILU(0) preconditioner (srk_matrix_ilu0, srk_precond_apply,
preconditioned solves) against the oracle (oracle/precond.py)."""
import numpy as np
import pytest

import oracle.precond as OP
import synth
from tests.gpu_util import rel, to_dev, to_np

pytestmark = pytest.mark.gpu

K = 20


@pytest.fixture(scope="module")
def srk():
    import paper_1504_04395_b200 as srk
    srk.load_library()
    return srk


def _ops():
    return {
        "cd2": synth.conv_diff_2d(14, (20.0, 10.0)),
        "cd3c": synth.conv_diff_3d(6, (10.0, 5.0, 2.0), np.complex128, -0.1j),
        "rand": synth.random_sparse(700, 6, seed=5, dominance=1.5),
    }


def _pattern_values(L, U, A):
    import scipy.sparse as sp
    Fl = ((L.tocsr() - sp.identity(A.shape[0], format="csr")) + U).tocsr()
    A = A.tocsr()
    A.sort_indices()
    rows = np.repeat(np.arange(A.shape[0]), np.diff(A.indptr))
    return np.asarray(Fl[rows, A.indices]).ravel()


@pytest.mark.parametrize("name", ["cd2", "cd3c", "rand"])
def test_ilu0_factor_matches_oracle(srk, name):
    A = _ops()[name]
    As = A.to_scipy()
    M = srk.Matrix.from_csr(A, need_adjoint=True).ilu0()
    L, U = OP.ilu0(As)
    ref = _pattern_values(L, U, As)
    got = M.ilu0_factor()
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("name", ["cd2", "cd3c", "rand"])
@pytest.mark.parametrize("s", [1, 4, 19])
def test_precond_apply_matches_oracle(srk, name, s):
    A = _ops()[name]
    As = A.to_scipy()
    cplx = np.iscomplexobj(A.values)
    M = srk.Matrix.from_csr(A, need_adjoint=True).ilu0()
    L, U = OP.ilu0(As)
    P = synth.random_rhs(A.n, s, 9, cplx)
    Z = to_np(srk.precond_apply(M, to_dev(P)))
    assert rel(Z, OP.apply_inv(L, U, P)) < 1e-12
    ZH = to_np(srk.precond_apply(M, to_dev(P), adjoint=True))
    assert rel(ZH, OP.apply_inv_adj(L, U, P)) < 1e-12


METHODS = ["egl_bicg", "gl_bicg", "li_bicg", "bl_bicg_rq", "egl_qmr", "bl_qmr", "li_bicgstab", "gl_bicgstab",
           "bl_bicgstab", "bl_bicgstab_rq"]


@pytest.mark.parametrize("method", METHODS)
def test_preconditioned_lockstep_and_solve(srk, method):
    """Right-preconditioned iterates X_k = M^-1 Y_k in lock step with the oracle on
    Ex. 1's operator (30^2, s = 4, B -> Q), then the full solve to 1e-10."""
    A, B = synth.paper_ex1(30)
    Q, _ = np.linalg.qr(B)
    Q = np.ascontiguousarray(Q)
    As = A.to_scipy()
    L, U = OP.ilu0(As)
    a = OP.solve_right(method, As, Q, L, U, tol=1e-10, maxit=500, record=K, order="blas")
    b = OP.solve_right(method, As, Q, L, U, tol=1e-10, maxit=500, record=K, order="seq")
    d = [rel(x, y) for x, y in zip(a.Xs, b.Xs)]
    env = np.maximum(1e-10, 100 * np.maximum.accumulate(d)) if d else np.array([])
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method]).ilu0()
    sv = srk.Solver(M, Q.shape[1], method, tol=1e-10, maxit=500, poll_every=1)
    sv.start(to_dev(Q))
    for k in range(min(K, a.iterations)):
        st = sv.iterate(1)
        x = to_np(sv.x())
        if k < len(a.Xs):
            assert rel(x, a.Xs[k]) <= env[k], (method, k + 1, rel(x, a.Xs[k]), env[k])
        if st != 0:
            break
    sv.close()
    X, rep = srk.solve(M, to_dev(Q), method, tol=1e-10, maxit=500)
    assert rep.outcome == a.outcome, (rep.outcome, a.outcome)
    if rep.outcome == "converged":
        assert np.linalg.norm(Q - As @ to_np(X)) / np.linalg.norm(Q) <= 1e-10
        assert abs(rep.iterations - a.iterations) <= max(2, 0.05 * a.iterations)


def test_preconditioned_x0(srk):
    """A nonzero X0 enters as Y0 = M X0: the solver's initial residual is B - A X0 and
    its iterate maps back to X0; the solve from there converges."""
    A, B = synth.paper_ex1(16)
    As = A.to_scipy()
    X0 = synth.random_rhs(A.n, B.shape[1], 11)
    M = srk.Matrix.from_csr(A, need_adjoint=True).ilu0()
    sv = srk.Solver(M, B.shape[1], "gl_bicgstab", tol=1e-10, maxit=200, poll_every=1)
    sv.start(to_dev(B), to_dev(X0))
    assert rel(to_np(sv.residual()), B - As @ X0) < 1e-12
    assert rel(to_np(sv.x()), X0) < 1e-12
    sv.iterate(200)
    rep = sv.report()
    assert rep.outcome == "converged"
    assert np.linalg.norm(B - As @ to_np(sv.x())) <= 1e-10 * np.linalg.norm(B - As @ X0) * 1.01
    sv.close()


def test_precond_apply_large_many_levels(srk):
    """The sync-free triangular solves at the paper's Ex. 2 size (50^3 = 125,000 rows,
    ~150 levels, every CTA of the grid taking rows): M^-1 P against the oracle's
    triangular solves, and bitwise equal to the one-launch-per-level schedule
    (SRK_TRSV_LEVELS=1, run in a subprocess: the switch is read once)."""
    import os
    import subprocess
    import sys
    A, _ = synth.paper_ex2(50, 1000.0)
    As = A.to_scipy()
    M = srk.Matrix.from_csr(A, need_adjoint=True).ilu0()
    L, U = OP.ilu0(As)
    P = synth.random_rhs(A.n, 4, 13)
    Z = to_np(srk.precond_apply(M, to_dev(P)))
    assert rel(Z, OP.apply_inv(L, U, P)) < 1e-12
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (f"import sys; sys.path.insert(0, {root!r})\n"
            "import numpy as np, torch, synth, paper_1504_04395_b200 as srk\n"
            "srk.load_library()\n"
            "A, _ = synth.paper_ex2(50, 1000.0)\n"
            "M = srk.Matrix.from_csr(A, need_adjoint=True).ilu0()\n"
            "P = synth.random_rhs(A.n, 4, 13)\n"
            "Z = srk.precond_apply(M, torch.from_numpy(P).cuda()).cpu().numpy()\n"
            "sys.stdout.buffer.write(Z.tobytes())\n")
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "SRK_TRSV_LEVELS": "1"},
                         capture_output=True, timeout=600)
    Zl = np.frombuffer(out.stdout, dtype=np.float64).reshape(Z.shape)
    assert np.array_equal(Z, Zl)


# ------------------------------------------------------------- ILUTP (R14)
def _pivoting_sparse(n, seed, cplx=False):
    """Sparse, nonsymmetric, weak diagonal: partial pivoting moves rows (as in the oracle pins)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    A = sp.random(n, n, density=6.0 / n, random_state=rng, format="csr")
    if cplx:
        A = A + 1j * sp.random(n, n, density=6.0 / n, random_state=rng, format="csr")
    A = A + sp.diags(0.05 * rng.standard_normal(n)) + sp.diags(np.ones(n - 1), -1) + 2.0 * sp.identity(n)
    A = sp.csr_matrix(A)
    A.sort_indices()
    return A


def _ilutp_ops():
    import scipy.sparse as sp
    weak = _pivoting_sparse(400, 21)
    weak = sp.csr_matrix(weak - 2.0 * sp.identity(400))  # weak diagonal: rows move
    weak.sort_indices()
    return {
        "pivot": weak,
        "pivot_c": _pivoting_sparse(300, 22, True),
        "lattice": synth.lattice_4d(4, kappa=0.12, seed=3).to_scipy(),  # Ex. 4's operator at 4^4
    }


@pytest.mark.parametrize("name", ["pivot", "pivot_c", "lattice"])
def test_ilutp_factor_matches_oracle(srk, name):
    """The library's ILUTP (host factorisation) against the oracle's: the same pivot order
    and the same L, U entries (to rounding)."""
    A = _ilutp_ops()[name]
    M = srk.Matrix.from_csr(A, need_adjoint=True).ilutp(5e-2)
    L, U, perm = OP.ilutp(A, 5e-2)
    Lg, Ug, pg = M.ilutp_factor()
    kind, nz, pivoted = M.prec_info()
    assert kind == "ilutp" and pivoted == bool(np.any(perm != np.arange(A.shape[0])))
    assert np.array_equal(pg, perm)
    assert (Lg != 0).sum() == (L != 0).sum() and (Ug != 0).sum() == (U != 0).sum()
    assert rel(Lg.toarray(), L.toarray()) <= 1e-12 and rel(Ug.toarray(), U.toarray()) <= 1e-12
    if name == "pivot":
        assert pivoted


@pytest.mark.parametrize("name", ["pivot", "pivot_c", "lattice"])
def test_ilutp_apply_matches_oracle(srk, name):
    """Z = M^-1 P = U^-1 L^-1 (Pi P) and M^-H P = Pi^T L^-H U^-H P on the device (the row
    permutation kernels around the level-scheduled solves) against the oracle's, from the
    oracle's factor."""
    A = _ilutp_ops()[name]
    cplx = A.dtype == np.complex128
    M = srk.Matrix.from_csr(A, need_adjoint=True).ilutp(5e-2)
    L, U, perm = OP.ilutp(A, 5e-2)
    for s in (1, 4, 7):
        P = synth.random_rhs(A.shape[0], s, s, cplx)
        Z = to_np(srk.precond_apply(M, to_dev(P)))
        assert rel(Z, OP.apply_inv(L, U, P, perm)) <= 1e-11, (name, s)
        ZH = to_np(srk.precond_apply(M, to_dev(P), adjoint=True))
        assert rel(ZH, OP.apply_inv_adj(L, U, P, perm)) <= 1e-11, (name, s)


@pytest.mark.parametrize("method", ["gl_bicgstab", "bl_bicgstab_rq", "egl_qmr", "bl_bicg_rq"])
def test_ilutp_preconditioned_lockstep(srk, method):
    """Right-ILUTP-preconditioned iterates in lock step with the oracle on a pivoting operator
    (X_k = M^-1 Y_k, M = Pi^T L U; A^H products through M^-H), then the full solve on Ex. 4's
    lattice operator (preconditioning reduces the iteration count)."""
    import oracle
    A = _ilutp_ops()["pivot"]
    B = synth.random_rhs(A.shape[0], 4, 3)
    L, U, perm = OP.ilutp(A, 5e-2)
    a = OP.solve_right(method, A, B, L, U, perm, tol=1e-10, maxit=300, record=10, order="blas")
    b = OP.solve_right(method, A, B, L, U, perm, tol=1e-10, maxit=300, record=10, order="seq")
    d = [rel(x, y) for x, y in zip(a.Xs, b.Xs)]
    env = np.maximum(1e-10, 100 * np.maximum.accumulate(d)) if d else np.array([])
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method]).ilutp(5e-2)
    sv = srk.Solver(M, 4, method, tol=1e-10, maxit=300, poll_every=1)
    sv.start(to_dev(B))
    for k in range(min(10, len(a.Xs))):
        st = sv.iterate(1)
        assert rel(to_np(sv.x()), a.Xs[k]) <= env[k], (method, k + 1)
        if st != 0:
            break
    sv.close()
    Al = _ilutp_ops()["lattice"]
    Bl = synth.random_rhs(Al.shape[0], 4, 0, True)
    Ml = srk.Matrix.from_csr(Al, need_adjoint=srk.NEEDS_ADJOINT[method]).ilutp(5e-2)
    Lq, Uq, pq = OP.ilutp(Al, 5e-2)
    ref = OP.solve_right(method, Al, Bl, Lq, Uq, pq, tol=1e-8, maxit=500, record=0)
    plain = oracle.solve(method, Al, Bl, tol=1e-8, maxit=500, record=0)
    X, rep = srk.solve(Ml, to_dev(Bl), method, tol=1e-8, maxit=500)
    assert rep.outcome == ref.outcome == "converged"
    assert abs(rep.iterations - ref.iterations) <= max(2, 0.05 * ref.iterations)
    assert rep.iterations < plain.iterations
    assert np.linalg.norm(Bl - Al @ to_np(X)) / np.linalg.norm(Bl) <= 1e-8
