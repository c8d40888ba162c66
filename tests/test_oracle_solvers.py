"""Pins for the oracle solvers (oracle/solvers.py) against what the paper and
the mathematics fix: the s=1 reduction to SciPy's single-RHS
bicg/qmr/bicgstab, the loop-interchange equivalence, the Kronecker
lift of the global methods, the rank-1 shadow equivalence of the
economic methods, the exact-arithmetic equivalence of
the rQ variants (Eqs. (4)-(7)) and the norm identity ‖R‖ = ‖C‖
(P:589-597), Petrov-Galerkin, block Krylov membership (P:210-219,
P:313-316), brute-force quasi-minimisation (QMR), finite termination,
dense direct solves and Proposition 1's counts."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
import synth
from oracle import solvers as S

BICG = ["li_bicg", "gl_bicg", "egl_bicg", "bl_bicg", "bl_bicg_rq"]
QMR = ["li_qmr", "gl_qmr", "egl_qmr", "bl_qmr"]
STAB = ["li_bicgstab", "gl_bicgstab", "bl_bicgstab", "bl_bicgstab_rq"]
SCIPY = {**{m: spla.bicg for m in BICG}, **{m: spla.qmr for m in QMR}, **{m: spla.bicgstab for m in STAB}}


def problem(n=48, s=3, seed=0, cplx=False, dominance=0.6):
    A = synth.random_sparse(n, 4, seed, np.complex128 if cplx else np.float64, dominance).to_scipy()
    B = synth.random_rhs(n, s, seed, cplx)
    return A, B


def scipy_iterates(fn, A, b, k):
    xs = []
    fn(A, b, rtol=1e-300, atol=0.0, maxiter=k, callback=lambda x: xs.append(np.array(x, copy=True)))
    return xs


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("method", oracle.METHODS)
def test_s1_reduces_to_single_rhs(method, cplx):
    """'All resulting simultaneous methods reduce to the single r.h.s. method for s=1'."""
    A, B = problem(s=1, cplx=cplx, seed=3)
    K = 8
    r = oracle.solve(method, A, B, tol=1e-300, maxit=K, record=K, shadow=None)
    ref = scipy_iterates(SCIPY[method], A, B[:, 0], K)
    assert len(r.Xs) == K and len(ref) == K
    for k in range(K):
        assert rel(r.Xs[k][:, 0], ref[k]) < 1e-10, (method, k)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("method", ["li_bicg", "li_qmr", "li_bicgstab"])
def test_loop_interchange_per_column(method, cplx):
    """Column i of Li-X is the single-RHS method on (A, b_i)."""
    A, B = problem(s=4, cplx=cplx, seed=5)
    K = 10
    r = oracle.solve(method, A, B, tol=1e-300, maxit=K, record=K)
    for i in range(B.shape[1]):
        ref = scipy_iterates(SCIPY[method], A, B[:, i], K)
        for k in range(K):
            assert rel(r.Xs[k][:, i], ref[k]) < 1e-10, (method, i, k)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("method", ["gl_bicg", "gl_qmr", "gl_bicgstab"])
def test_global_is_kronecker_lift(method, cplx):
    """Gl-X on (A, B) is X on (I⊗A) x = vec(B), mat by columns (Eq. (2))."""
    A, B = problem(n=30, s=3, cplx=cplx, seed=7)
    s = B.shape[1]
    K = 10
    r = oracle.solve(method, A, B, tol=1e-300, maxit=K, record=K)
    big = sp.kron(sp.identity(s), A).tocsr()
    ref = scipy_iterates(SCIPY[method], big, B.ravel(order="F"), K)
    for k in range(K):
        assert rel(r.Xs[k].ravel(order="F"), ref[k]) < 1e-10, (method, k)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("pair", [("egl_bicg", "gl_bicg"), ("egl_qmr", "gl_qmr")])
def test_economic_equals_global_rank1_shadow(pair, cplx):
    """With R̂0 = r̂0 1^T the shadow blocks keep this structure, so the
    economic variant reproduces the global one."""
    A, B = problem(n=40, s=4, cplx=cplx, seed=11)
    K = 15
    e = oracle.solve(pair[0], A, B, tol=1e-300, maxit=K, record=K)
    g = oracle.solve(pair[1], A, B, tol=1e-300, maxit=K, record=K, shadow="mean")
    for k in range(K):
        assert rel(e.Xs[k], g.Xs[k]) < 1e-11, k
    assert e.matvec_cols_AH == K and g.matvec_cols_AH == K * B.shape[1]


@pytest.mark.parametrize("cplx", [False, True])
def test_bl_bicg_rq_equals_bl_bicg(cplx):
    """Eqs. (4)-(7): Alg. 5 produces Alg. 3's iterates in exact arithmetic; and
    ‖R^(k)‖_F = ‖C^(k)‖_F."""
    A, B = problem(n=40, s=3, cplx=cplx, seed=13, dominance=0.6)
    K = 8
    a = oracle.solve("bl_bicg", A, B, tol=1e-300, maxit=K, record=K)
    b = oracle.solve("bl_bicg_rq", A, B, tol=1e-300, maxit=K, record=K)
    for k in range(K):
        assert rel(b.Xs[k], a.Xs[k]) < 1e-8, k
        true = np.linalg.norm(B - A @ b.Xs[k])
        assert abs(np.linalg.norm(b.Rs[k]) - true) <= 1e-10 * np.linalg.norm(B), k


@pytest.mark.parametrize("cplx", [False, True])
def test_bl_bicgstab_rq_equals_bl_bicgstab(cplx):
    """Bl-BiCGStab-rQ (App. A.5) equals Bl-BiCGStab (A.4) in exact arithmetic,
    and its ‖C‖_F is the true residual norm."""
    A, B = problem(n=40, s=3, cplx=cplx, seed=17, dominance=0.6)
    K = 8
    a = oracle.solve("bl_bicgstab", A, B, tol=1e-300, maxit=K, record=K)
    b = oracle.solve("bl_bicgstab_rq", A, B, tol=1e-300, maxit=K, record=K)
    for k in range(K):
        assert rel(b.Xs[k], a.Xs[k]) < 1e-8, k
        assert abs(np.linalg.norm(b.Rs[k]) - np.linalg.norm(B - A @ b.Xs[k])) <= 1e-10 * np.linalg.norm(B)


def test_bl_bicg_petrov_galerkin():
    """Residuals are orthogonal to K_k(A^H, R̂0): (R̂^(i))^H R^(j) = 0, i != j."""
    A, B = problem(n=40, s=3, seed=19, dominance=0.8)
    K = 5
    r = oracle.solve("bl_bicg", A, B, tol=1e-300, maxit=K, record=K)
    # shadow residuals: recompute with the adjoint problem's Krylov space instead
    AH = A.conj().T.tocsr()
    R0 = B.copy()
    basis = [R0]
    for _ in range(K):
        basis.append(AH @ basis[-1])
    # R_j must be orthogonal to span{R0, A^H R0, ..., (A^H)^{j-1} R0}
    for j in range(1, K + 1):
        Rj = r.Rs[j - 1]
        Kspace = np.hstack(basis[:j])
        Qk, _ = np.linalg.qr(Kspace)
        assert np.linalg.norm(Qk.conj().T @ Rj) <= 1e-8 * np.linalg.norm(B), j


@pytest.mark.parametrize("method", ["bl_bicg", "bl_bicg_rq", "bl_bicgstab", "bl_bicgstab_rq", "bl_qmr"])
def test_block_finite_termination(method):
    """dim K_k(A, R0) = sk: n=12, s=3 terminates within ceil(n/s)+2 = 6
    iterations and matches the dense direct solve."""
    rng = np.random.default_rng(23)
    Ad = rng.standard_normal((12, 12)) + 6 * np.eye(12)
    A = sp.csr_matrix(Ad)
    B = rng.standard_normal((12, 3))
    r = oracle.solve(method, A, B, tol=1e-10, maxit=6)
    assert r.outcome == "converged" and r.iterations <= 6, (r.outcome, r.iterations)
    assert rel(r.X, np.linalg.solve(Ad, B)) < 1e-8


@pytest.mark.parametrize("method", ["bl_bicgstab", "gl_bicgstab"])
def test_bicgstab_krylov_membership(method):
    """x_i^(k) ∈ x_i^(0) + K_2k(A, R0)."""
    A, B = problem(n=30, s=2, seed=29, dominance=0.6)
    K = 3
    r = oracle.solve(method, A, B, tol=1e-300, maxit=K, record=K)
    Ad = A.toarray()
    for k in range(1, K + 1):
        blocks = [B]
        for _ in range(2 * k - 1):
            blocks.append(Ad @ blocks[-1])
        Qk, _ = np.linalg.qr(np.hstack(blocks))
        Xk = r.Xs[k - 1]
        assert np.linalg.norm(Xk - Qk @ (Qk.T @ Xk)) <= 1e-8 * np.linalg.norm(Xk), k


@pytest.mark.parametrize("cplx", [False, True])
def test_bl_qmr_quasi_minimal(cplx):
    """Bl-QMR's X_k = X0 + 𝐏_k Z with Z the least-squares minimiser of
    ‖E1 ρ1 − L_k Z‖_F in the nested bi-orthogonal basis: checked by a
    dense lstsq, plus the Lanczos relation A 𝐏_k = 𝐕_{k+1} L_k and block
    bi-orthogonality W_j^H V_i = 0 (i != j)."""
    A, B = problem(n=36, s=3, cplx=cplx, seed=31, dominance=0.6)
    s = B.shape[1]
    K = 5
    tr = []
    r = S.bl_qmr(A, B, tol=1e-300, maxit=K + 1, record=K + 1, trace=tr)
    assert len(tr) == K + 1
    Vs = [t["V"] for t in tr]
    Ws = [t["W"] for t in tr]
    for i in range(K + 1):
        for j in range(K + 1):
            if i != j:
                assert np.linalg.norm(Ws[j].conj().T @ Vs[i]) < 1e-8, (i, j)
    rho1 = Vs[0].conj().T @ B
    for k in range(1, K + 1):
        L = np.zeros(((k + 1) * s, k * s), dtype=complex)
        for i in range(k):
            L[i * s:(i + 1) * s, i * s:(i + 1) * s] = tr[i]["beta"]
            L[(i + 1) * s:(i + 2) * s, i * s:(i + 1) * s] = tr[i]["rho_next"]
        Pk = np.hstack([tr[i]["P"] for i in range(k)])
        Vk1 = np.hstack(Vs[:k + 1])
        assert np.linalg.norm(A @ Pk - Vk1 @ L) <= 1e-10 * np.linalg.norm(A @ Pk)
        rhs = np.zeros(((k + 1) * s, s), dtype=complex)
        rhs[:s] = rho1
        Z = np.linalg.lstsq(L, rhs, rcond=None)[0]
        assert rel(Pk @ Z, r.Xs[k - 1]) < 1e-9, k


def test_proposition1_counts():
    """Prop. 1: per iteration two block products (one with A, one with
    A^H) and 7s (Li, Gl) or 7s^2 (Bl) vector operations; eGl needs one A^H
    vector; BiCGStab two A products and no A^H."""
    A, B = problem(n=40, s=4, seed=37)
    s, K = 4, 6
    for m in ("li_bicg", "gl_bicg"):
        r = oracle.solve(m, A, B, tol=1e-300, maxit=K)
        assert r.vector_ops == 7 * s * K and r.matvec_cols_A == s * K and r.matvec_cols_AH == s * K
    r = oracle.solve("bl_bicg", A, B, tol=1e-300, maxit=K)
    assert r.vector_ops == 7 * s * s * K and r.matvec_cols_A == s * K and r.matvec_cols_AH == s * K
    r = oracle.solve("egl_bicg", A, B, tol=1e-300, maxit=K)
    assert r.matvec_cols_A == s * K and r.matvec_cols_AH == K
    for m in STAB:
        r = oracle.solve(m, A, B, tol=1e-300, maxit=K)
        assert r.matvec_cols_A == 2 * s * K and r.matvec_cols_AH == 0, m


def test_trivial_cases():
    """A = I converges in one iteration with X = B; B = 0 needs none."""
    A = sp.identity(10, format="csr")
    B = np.random.default_rng(1).standard_normal((10, 2))
    for m in oracle.METHODS:
        r = oracle.solve(m, A, B, tol=1e-12, maxit=5)
        assert r.outcome == "converged" and r.iterations == 1 and rel(r.X, B) < 1e-14, m
        z = oracle.solve(m, A, np.zeros((10, 2)), tol=1e-12, maxit=5)
        assert z.outcome == "converged" and z.iterations == 0, m


@pytest.mark.parametrize("method", oracle.METHODS)
def test_config1_matches_direct_solve(method):
    """Config 1 (n=1024): every variant converges to tol 1e-8, its final true
    residual is <= 1e-8 and X is the direct solution within cond·tol."""
    A, B = synth.make_config(1)
    As = A.to_scipy()
    r = oracle.solve(method, As, B, tol=1e-8, maxit=2000)
    assert r.outcome == "converged" and r.final_true_rel_residual <= 1e-8
    Xs = spla.spsolve(As.tocsc(), B)
    assert rel(r.X, Xs) < 1e-5


def test_table1_rho_golden():
    """Table 1's ρ = s·n/nnz (Eq. (8); values P:687) from the paper-size
    stencils: Ex. 1 (200^2, s=4) and Ex. 2/3 (50^3, s=19). Fixture tests/golden/table1_rho.txt."""
    import os
    rows = {}
    with open(os.path.join(os.path.dirname(__file__), "golden", "table1_rho.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                ex, s, rho = line.split()
                rows[ex] = (int(s), float(rho))
    A1 = synth.conv_diff_2d(200)
    s, rho = rows["ex1"]
    assert round(s * A1.n / A1.nnz, 2) == rho
    A2 = synth.conv_diff_3d(50)
    s, rho = rows["ex2"]
    assert round(s * A2.n / A2.nnz, 2) == rho


@pytest.mark.parametrize("method,bound", [("egl_bicg", 1e-11), ("egl_qmr", 1e-11), ("li_qmr", 1e-11),
                                          ("gl_bicgstab", 1e-9)])
def test_reduction_order_spread_economic(method, bound):
    """on config 1 the economic/Li/global variants are insensitive to
    the reduction order over 20 iterations (Gl-BiCGStab sits near 1e-10), unlike
    the block variants — the basis of the parity envelope."""
    A, B = synth.make_config(1)
    As = A.to_scipy()
    a = oracle.solve(method, As, B, tol=1e-300, maxit=20, record=20, order="blas")
    b = oracle.solve(method, As, B, tol=1e-300, maxit=20, record=20, order="seq")
    assert max(rel(x, y) for x, y in zip(a.Xs, b.Xs)) < bound


def test_lattice_generator_structure():
    """Config 4 generator (reading G23): 8 dof*dof neighbour blocks + identity per
    row (8*12 + 1 = 97 entries), periodic nearest-neighbour pattern (block (x, y)
    present iff (y, x) present), and spectral radius of H close to the circular-law
    value sqrt(8 * 12 * 1/6) = 4 for i.i.d. CN(0, 1/6) blocks (4.06)."""
    import scipy.sparse.linalg as sla
    A = synth.lattice_4d(4)
    As = A.to_scipy()
    assert A.nnz == 97 * A.n
    assert np.allclose(As.diagonal(), 1.0)
    pat = (As != 0).astype(np.int8)
    assert (pat != pat.T).nnz == 0
    H = (sp.identity(A.n) - As) / 0.12
    rho = abs(sla.eigs(H.tocsc(), k=1, which="LM", return_eigenvectors=False)[0])
    assert 3.5 < rho < 4.6


@pytest.mark.parametrize("method", ["li_bicgstab", "gl_bicgstab", "bl_bicgstab", "bl_bicgstab_rq"])
def test_lattice_bicgstab_converges(method):
    """Config 4's methods on a 4^4 lattice converge to the direct solution."""
    A, B = synth.make_config(4, m=4)
    As = A.to_scipy()
    r = oracle.solve(method, As, B, tol=1e-10, maxit=200)
    assert r.outcome == "converged"
    Xs = spla.spsolve(As.tocsc(), B)
    assert rel(r.X, Xs) < 1e-8


def test_lattice_bsr_form_is_the_same_operator():
    """synth.lattice_4d_bsr (block-sparse, implied unit diagonal) describes exactly
    the matrix of synth.lattice_4d (scalar CSR): I + BSR assembled by scipy equals
    the CSR entry for entry (same RNG draws)."""
    import scipy.sparse as sp
    for L in (3, 4):
        A = synth.lattice_4d(L)
        brp, bcol, blocks = synth.lattice_4d_bsr(L)
        assert blocks.shape == (8 * L ** 4, 12, 12) and len(brp) == L ** 4 + 1
        assert np.all(np.diff(bcol.reshape(-1, 8), axis=1) > 0)  # sorted unique block columns
        B = sp.bsr_matrix((blocks, bcol, brp), shape=(A.n, A.n)) + sp.identity(A.n, dtype=np.complex128)
        D = (A.to_scipy() - B.tocsr()).tocsr()
        D.eliminate_zeros()
        assert D.nnz == 0


def test_li_freeze_policy_unit():
    """Reading G13 applied per column: a zero denominator OR a non-finite quotient
    freezes the column with coefficient 0; frozen columns stay at 0; others divide."""
    num = np.array([1.0, 1e300, 2.0, 3.0, np.nan])
    den = np.array([0.0, 1e-300, 4.0, 5.0, 1.0])
    frozen = np.array([False, False, False, True, False])
    q, newly = S._safe_div(num, den, frozen)
    assert np.array_equal(newly, [True, True, False, False, True])
    assert np.array_equal(q, [0.0, 0.0, 0.5, 0.0, 0.0])


def _skew_block_problem(cplx=False):
    """A = blockdiag(S, M): S an integer skew-symmetric block, M diagonally dominant.
    Column 0 of B lives on S with integer entries, so <q_0, p̂_0> = b_0^T S b_0 = 0
    EXACTLY in floating point: the Lanczos denominator of Li-BiCG's column 0 vanishes
    at the first iteration, while column 1 is an ordinary BiCG problem."""
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
    return A, B


@pytest.mark.parametrize("cplx", [False, True])
def test_li_bicg_column_freeze_on_lanczos_zero(cplx):
    """Li-BiCG with one column meeting an exact Lanczos zero (reading G13):
    that column freezes at iteration 1 (X column stays 0, reported in breakdown_cols)
    while the other column's iterates are SciPy's single-RHS bicg on (A, b_1)."""
    A, B = _skew_block_problem(cplx)
    q0 = A @ B[:, 0]
    assert np.vdot(B[:, 0], q0) == 0  # the exact zero the test relies on
    k = 12
    r = S.li_bicg(A, B, tol=1e-300, maxit=k, record=k)
    assert r.breakdown_cols == [0]
    assert all(np.all(X[:, 0] == 0) for X in r.Xs)
    ref = scipy_iterates(spla.bicg, A, B[:, 1], k)
    for j, x in enumerate(ref):
        assert rel(r.Xs[j][:, 1], x) < 1e-10, j


# ---------------------------------------------------------------- f3: QR of search directions
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("pair", [("bl_bicg", "bl_bicg_sq"), ("bl_bicgstab", "bl_bicgstab_sq")])
def test_search_direction_qr_equals_plain_block_method(pair, cplx):
    """Orthonormalising the search directions ([Oleary80]) changes only the
    basis the s x s coefficients act on: X_k equals Alg. 3 / App. A.4 in exact arithmetic
    (to the rounding the block recurrences amplify, as for the rQ pin)."""
    plain, sq = pair
    A, B = problem(cplx=cplx)
    a = oracle.solve(plain, A, B, tol=1e-10, maxit=200, record=8)
    b = S.SOLVERS[sq](A, B, tol=1e-10, maxit=200, record=8)
    for k in range(4):
        assert rel(b.Xs[k], a.Xs[k]) < 1e-11, k
    for k in range(4, 8):
        assert rel(b.Xs[k], a.Xs[k]) < 1e-6, k


@pytest.mark.parametrize("sq,base", [("bl_bicg_sq", spla.bicg), ("bl_bicgstab_sq", spla.bicgstab)])
def test_search_direction_qr_s1(sq, base):
    """s = 1: the orthonormal search direction is p/‖p‖, a rescaling — SciPy's BiCG / BiCGStab."""
    A, B = problem(s=1)
    r = S.SOLVERS[sq](A, B, tol=1e-300, maxit=10, record=10)
    ref = scipy_iterates(base, A, B[:, 0], 10)
    for k in range(min(len(ref), len(r.Xs))):
        assert rel(r.Xs[k][:, 0], ref[k]) < 1e-9, k


def test_search_direction_qr_converges_on_config1():
    A, B = synth.make_config(1)
    r = S.SOLVERS["bl_bicgstab_sq"](A.to_scipy(), B, tol=1e-8, maxit=2000, record=0)
    assert r.outcome == "converged" and r.final_true_rel_residual <= 1e-8


# ---------------------------------------------------------------- f4: rank-deficiency continuation
def test_counter_generator_is_splitmix64():
    """The replacement vectors' generator is SplitMix64 (its published first output for
    state 0 is 0xE220A8397B1DCDAF); entries are uniform in [-1, 1), keyed and repeatable."""
    from oracle.linalg import _splitmix64, counter_uniform
    assert int(_splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF
    u = counter_uniform(10000, 3, False)
    assert u.min() >= -1 and u.max() < 1 and abs(u.mean()) < 0.05 and abs(u.var() - 1 / 3) < 0.02
    assert np.array_equal(u, counter_uniform(10000, 3, False))
    assert not np.array_equal(u, counter_uniform(10000, 4, False))
    z = counter_uniform(100, 3, True)
    assert np.array_equal(z.real, u[:100]) and not np.array_equal(z.real, z.imag)
    assert np.array_equal(counter_uniform(50, 3, False, row0=50), u[50:100])


@pytest.mark.parametrize("cplx", [False, True])
def test_thin_qr_continuation_is_qr_of_the_replaced_block(cplx):
    """Z = [w, 2w, u]: column 1 is deficient; with continuation Q is the (unique) thin QR
    factor of Z' = [w, ρ, u], ρ the replacement vector, C[1, 1] = 0 and Z = Q C."""
    from oracle.linalg import counter_uniform, thin_qr
    rng = np.random.default_rng(2)
    n = 30
    w, u = synth.random_rhs(n, 2, 5, cplx).T
    Z = np.stack([w, 2 * w, u], axis=1)
    with pytest.raises(oracle.Breakdown):
        thin_qr(Z)
    fill = lambda j: counter_uniform(n, 7 * 64 + j, cplx)  # noqa: E731
    Q, C = thin_qr(Z, fill=fill)
    assert C[1, 1] == 0 and np.all(np.diag(C).real >= 0)
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(3)) < 1e-13
    assert np.linalg.norm(Q @ C - Z) < 1e-13 * np.linalg.norm(Z)
    Zp = Z.copy()
    Zp[:, 1] = fill(1)
    Qr, Rr = np.linalg.qr(Zp)
    ph = np.diag(Rr) / np.abs(np.diag(Rr))
    assert np.linalg.norm(Qr * ph[None, :] - Q) < 1e-12
    del rng


@pytest.mark.parametrize("cplx", [False, True])
def test_rank_continuation_equals_full_rank_run(cplx):
    """R0 = [b1, b2, b1 + b2] (exact deflation): continued Bl-BiCG-rQ runs on the
    orthonormal factor of B' = [b1, b2, ρ] (ρ the replacement) and only its C differs —
    α, β (Eqs. (4)-(7)) depend on the Q's alone — so X_k(B) = X_k(B') T with B = B' T:
    the deflation is hidden ([Dub01])."""
    from oracle.linalg import counter_uniform
    A, _ = problem(n=60, cplx=cplx)
    B = synth.random_rhs(60, 3, 3, cplx)
    B[:, 2] = B[:, 0] + B[:, 1]
    d = S.bl_bicg_rq(A, B, tol=1e-10, maxit=300, record=6, deflate=True)
    Bp = B.copy()
    Bp[:, 2] = counter_uniform(60, 2, cplx)
    T = np.linalg.lstsq(Bp, B, rcond=None)[0]
    assert np.linalg.norm(Bp @ T - B) < 1e-12 * np.linalg.norm(B)
    f = S.bl_bicg_rq(A, Bp, tol=1e-10, maxit=300, record=6)
    for k in range(4):
        assert rel(d.Xs[k], f.Xs[k] @ T) < 1e-9, k


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("method", ["bl_bicg_rq", "bl_bicgstab_rq"])
def test_rank_continuation_invariants(method, cplx):
    """With continuation the rQ methods run through an exactly rank-deficient R0 (plain
    policy: BREAKDOWN(rank), reading G11): every update right-multiplies by C, and
    C^(0) = Q^H B inherits b3 = b1 + b2, so x3 = x1 + x2 at every iterate; the norm
    identity ‖C_k‖_F = ‖B - A X_k‖_F holds throughout; the solve converges."""
    A, _ = problem(n=60, cplx=cplx)
    B = synth.random_rhs(60, 3, 3, cplx)
    B[:, 2] = B[:, 0] + B[:, 1]
    assert S.SOLVERS[method](A, B, tol=1e-10).outcome == "breakdown"
    d = S.SOLVERS[method](A, B, tol=1e-10, maxit=300, record=8, deflate=True)
    for X, C in zip(d.Xs, d.Rs):
        assert rel(X[:, 2], X[:, 0] + X[:, 1]) < 1e-10
        true = np.linalg.norm(B - A @ X)
        assert abs(np.linalg.norm(C) - true) <= 1e-8 * np.linalg.norm(B)
    assert d.outcome == "converged" and d.final_true_rel_residual <= 1e-10
    assert rel(d.X[:, 2], d.X[:, 0] + d.X[:, 1]) < 1e-8
