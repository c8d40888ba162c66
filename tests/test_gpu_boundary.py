"""The §8(b) boundary options on the GPU against the oracle: the shadow residual choices
(P:419-422), the QR preprocessing of the right-hand sides, the breakdown
thresholds, and the report's Proposition-1 vector-operation count."""
import numpy as np
import pytest

import oracle
from oracle import solvers as OS
import synth
from tests.gpu_util import rel, to_dev, to_np

pytestmark = pytest.mark.gpu
K = 12


@pytest.fixture(scope="module")
def srk():
    import paper_1504_04395_b200 as srk
    srk.load_library()
    return srk


@pytest.fixture(scope="module")
def cplx_problem():
    A = synth.conv_diff_3d(10, (50.0, 30.0, 10.0), np.complex128, -0.1j)
    return A, synth.random_rhs(A.n, 3, 1, True)


def _lockstep(srk, A, B, method, n_it, **opts):
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    sv = srk.Solver(M, B.shape[1], method, tol=1e-8, maxit=2000, poll_every=1, **opts)
    sv.start(to_dev(B))
    xs = []
    for _ in range(n_it):
        st = sv.iterate(1)
        xs.append(to_np(sv.x()))
        if st != 0:
            break
    sv.close()
    return xs


def _env(method, As, B, shadow):
    a = OS.SOLVERS[method](As, B, tol=1e-8, maxit=2000, record=K, order="blas", shadow=shadow)
    b = OS.SOLVERS[method](As, B, tol=1e-8, maxit=2000, record=K, order="seq", shadow=shadow)
    d = [rel(x, y) for x, y in zip(a.Xs, b.Xs)]
    return a, np.maximum(1e-10, 100 * np.maximum.accumulate(d))


SHADOW_METHODS = ["gl_bicg", "egl_bicg", "bl_bicg", "bl_bicg_rq", "li_qmr", "egl_qmr", "bl_qmr",
                  "gl_bicgstab", "bl_bicgstab", "bl_bicgstab_rq", "bl_bicg_sq", "bl_bicgstab_sq"]


@pytest.mark.parametrize("method", SHADOW_METHODS)
@pytest.mark.parametrize("shadow", ["conj", "given"])
def test_shadow_options(srk, cplx_problem, method, shadow):
    """R̂0 = conj(R0) (economic: conj of the mean) or a caller-given shadow."""
    A, B = cplx_problem
    As = A.to_scipy()
    econ = method.startswith("egl")
    if shadow == "given":
        S0 = synth.random_rhs(A.n, 1 if econ else B.shape[1], 9, True)
        S0 = S0[:, 0].copy() if econ else S0
        a, env = _env(method, As, B, S0)
        xs = _lockstep(srk, A, B, method, min(K, a.iterations), shadow="given", shadow_given=to_dev(S0))
    else:
        a, env = _env(method, As, B, "conj")
        xs = _lockstep(srk, A, B, method, min(K, a.iterations), shadow="conj")
    for k in range(min(len(xs), len(a.Xs))):
        assert rel(xs[k], a.Xs[k]) <= env[k], (method, shadow, k + 1, rel(xs[k], a.Xs[k]), env[k])


@pytest.mark.parametrize("method", ["gl_bicg", "li_bicgstab", "gl_qmr"])
def test_shadow_mean(srk, cplx_problem, method):
    """The rank-one block shadow r̂0 1^T on a non-economic variant."""
    A, B = cplx_problem
    As = A.to_scipy()
    a, env = _env(method, As, B, "mean")
    xs = _lockstep(srk, A, B, method, min(K, a.iterations), shadow="mean")
    for k in range(min(len(xs), len(a.Xs))):
        assert rel(xs[k], a.Xs[k]) <= env[k], (method, k + 1)


@pytest.mark.parametrize("method", ["egl_qmr", "bl_bicg_rq", "bl_bicgstab_rq"])
def test_preprocess_rhs(srk, cplx_problem, method):
    """B = Q C_B, solve A Y = Q, return X = Y C_B: the GPU's X equals the oracle's
    solve on Q times C_B, and X solves A X = B."""
    A, B = cplx_problem
    As = A.to_scipy()
    Q, C = oracle.thin_qr(B)
    a = oracle.solve(method, As, Q, tol=1e-8, maxit=2000, record=0)
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    X, rep = srk.solve(M, to_dev(B), method, tol=1e-8, maxit=2000, preprocess_rhs=True)
    X = to_np(X)
    assert rep.outcome == a.outcome == "converged"
    assert abs(rep.iterations - a.iterations) <= max(2, 0.02 * a.iterations)
    assert rel(X, a.X @ C) <= 1e-6
    assert np.linalg.norm(B - As @ X) / np.linalg.norm(B) <= 1e-7


@pytest.mark.parametrize("method", list(oracle.METHODS) + list(OS.SQ_METHODS))
def test_vector_ops_proposition1(srk, method):
    """The report's vector-operation count equals the oracle's counter after k iterations
    that end at maxit (Prop. 1: 7s for Li / Gl-BiCG and 7s^2 for Bl-BiCG per iteration)."""
    A = synth.conv_diff_3d(8)
    As = A.to_scipy()
    for s in (2, 3):
        B = synth.random_rhs(A.n, s, 1)
        a = OS.SOLVERS[method](As, B, tol=1e-300, maxit=4, record=0)
        M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
        X, rep = srk.solve(M, to_dev(B), method, tol=1e-300, maxit=4)
        assert rep.iterations == a.iterations == 4
        assert rep.vector_ops == a.vector_ops, (method, s, rep.vector_ops, a.vector_ops)
        if method in ("li_bicg", "gl_bicg"):
            assert rep.vector_ops == 7 * s * 4
        if method == "bl_bicg":
            assert rep.vector_ops == 7 * s * s * 4


def test_breakdown_threshold_option(srk):
    """eps_brk moves the singular-Gram test (reading G12): A = diag(1..50), B = [e1, e2,
    e1 + d e3] gives G = B^T A B with LU pivots 1, 2, 3 d^2 — at d = 1e-5 a relative pivot of
    1.5e-10 passes the default 1e-14 and breaks down at eps_brk = 1e-6."""
    import scipy.sparse as sp
    n, d = 50, 1e-5
    A = sp.diags(np.arange(1.0, n + 1), format="csr")
    B = np.zeros((n, 3))
    B[0, 0] = B[1, 1] = B[0, 2] = 1.0
    B[2, 2] = d
    M = srk.Matrix.from_csr(A)
    _, r0 = srk.solve(M, to_dev(B), "bl_bicg", tol=1e-12, maxit=1)
    assert r0.outcome != "breakdown", r0
    _, r1 = srk.solve(M, to_dev(B), "bl_bicg", tol=1e-12, maxit=1, eps_brk=1e-6)
    assert r1.outcome == "breakdown" and r1.breakdown_kind == "gram" and r1.breakdown_iter == 1, r1


def test_breakdown_col_reports_li_freeze(srk):
    import scipy.sparse as sp
    rng = np.random.default_rng(21)
    m = 6
    Sk = np.triu(rng.integers(-3, 4, (m, m)), 1).astype(float)
    Sk = Sk - Sk.T
    Mb = synth.random_sparse(40, 4, 5, np.float64, 0.8).to_scipy()
    A = sp.block_diag([sp.csr_matrix(Sk), Mb], format="csr")
    A.sort_indices()
    B = np.zeros((m + 40, 2))
    B[:m, 1] = rng.integers(-4, 5, m)        # column 1 meets the Lanczos zero this time
    B[:, 0] = synth.random_rhs(m + 40, 1, 8)[:, 0]
    M = srk.Matrix.from_csr(A)
    _, rep = srk.solve(M, to_dev(B), "li_bicg", tol=1e-300, maxit=5)
    assert rep.frozen_cols == 1 and rep.breakdown_col == 1


@pytest.mark.parametrize("method", ["egl_qmr", "bl_bicgstab_rq", "li_bicg"])
def test_trace_iterates_callback(srk, method):
    """srk_opts.trace_iterates / on_iter ("an iteration callback"): the callback's
    X_k and R_k (C_k for the rQ variant) are the stepping interface's, bitwise, and the oracle's
    within 1e-10 over the first iterations; its residual norm is the history's; the solve then
    runs on to convergence exactly as without the callback."""
    import oracle
    A = synth.conv_diff_2d(24, (20.0, 20.0))
    B = synth.random_rhs(A.n, 4, 3)
    M = srk.Matrix.from_csr(A)
    K = 6
    seen = []
    X, rep = srk.solve(M, to_dev(B), method, tol=1e-9, maxit=500, trace_iterates=K,
                       on_iter=lambda k, xk, rk, rel, state: seen.append((k, to_np(xk), to_np(rk), rel, state)))
    assert [t[0] for t in seen] == list(range(1, K + 1))
    sv = srk.Solver(M, 4, method, tol=1e-9, maxit=500, poll_every=1)
    sv.start(to_dev(B))
    ref = oracle.solve(method, A.to_scipy(), B, tol=1e-9, maxit=500, record=K)
    for k, xk, rk, rel, state in seen:
        sv.iterate(1)
        assert np.array_equal(xk, to_np(sv.x()))
        assert np.array_equal(rk, to_np(sv.residual()))
        assert np.linalg.norm(xk - ref.Xs[k - 1]) <= 1e-10 * np.linalg.norm(ref.Xs[k - 1])
        assert rk.shape == ref.Rs[k - 1].shape
        assert abs(rel - ref.history[k - 1]) <= 1e-9 * ref.history[k - 1] and state == 0
    X0, rep0 = srk.solve(M, to_dev(B), method, tol=1e-9, maxit=500)
    assert rep.outcome == rep0.outcome == "converged" and rep.iterations == rep0.iterations
    assert np.array_equal(to_np(X), to_np(X0))
