"""GPU parity of SURVEY §8(f) f3 and f4.

f3 — QR of the search directions (the [O'Leary] stabilisation the paper names and rejects,
P:486-496): Bl-BiCG-sQ and Bl-BiCGStab-sQ against the oracle's bl_bicg_sq /
bl_bicgstab_sq, iterate by iterate (X_k, R_k, §8c.5 envelope) and full solves.

f4 — rank-deficiency continuation of the rQ variants' thin QR:
with rank_policy="continue" a deficient column of Q is replaced by the counter-based
vector both sides generate, C_jj = 0, and the method runs on; the GPU must follow the
oracle's deflate=True run (X_k, C_k) and report the replaced column count."""
import numpy as np
import pytest

import oracle
from oracle import solvers as OS
import synth
from tests.gpu_util import rel, to_dev, to_np

pytestmark = pytest.mark.gpu
K = 20


@pytest.fixture(scope="module")
def srk():
    import paper_1504_04395_b200 as srk
    srk.load_library()
    return srk


def _problem(name):
    if name == "cfg1":
        return synth.make_config(1)
    if name == "cplx":
        A = synth.conv_diff_3d(10, (50.0, 30.0, 10.0), np.complex128, -0.1j)
        return A, synth.random_rhs(A.n, 3, 1, True)
    if name == "wide":  # s = 12 real: the DMMA Gram and update paths
        A = synth.conv_diff_3d(12)
        return A, synth.random_rhs(A.n, 12, 5)
    raise ValueError(name)


def _envelope(fn, As, B, k=K, **kw):
    a = fn(As, B, tol=1e-8, maxit=2000, record=k, order="blas", **kw)
    b = fn(As, B, tol=1e-8, maxit=2000, record=k, order="seq", **kw)
    d = [max(rel(x, y), rel(r, q)) for x, y, r, q in zip(a.Xs, b.Xs, a.Rs, b.Rs)]
    return a, np.maximum(1e-10, 100 * np.maximum.accumulate(d)) if d else np.array([])


def _lockstep(srk, A, B, method, n_it, **opts):
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    sv = srk.Solver(M, B.shape[1], method, tol=1e-8, maxit=2000, poll_every=1, **opts)
    sv.start(to_dev(B))
    xs, rs = [], []
    for _ in range(n_it):
        st = sv.iterate(1)
        xs.append(to_np(sv.x()))
        rs.append(to_np(sv.residual()))
        if st != 0:
            break
    return sv, xs, rs


@pytest.mark.parametrize("prob", ["cfg1", "cplx", "wide"])
@pytest.mark.parametrize("method", OS.SQ_METHODS)
def test_sq_lockstep(srk, method, prob):
    A, B = _problem(prob)
    As = A.to_scipy()
    a, env = _envelope(OS.SOLVERS[method], As, B)
    sv, xs, rs = _lockstep(srk, A, B, method, min(K, a.iterations))
    n_cmp = min(len(xs), len(a.Xs))
    assert n_cmp >= 1
    for k in range(n_cmp):
        assert rel(xs[k], a.Xs[k]) <= env[k], (method, prob, k + 1, "X", rel(xs[k], a.Xs[k]), env[k])
        if a.half_step and k == a.iterations - 1:
            continue
        assert rel(rs[k], a.Rs[k]) <= env[k], (method, prob, k + 1, "R", rel(rs[k], a.Rs[k]), env[k])
    sv.close()


@pytest.mark.parametrize("method", OS.SQ_METHODS)
def test_sq_full_solve(srk, method):
    """Outcome, count (within max(2%, |it_O - it_O'| + 2)) and the oracle-recomputed true
    residual on the complex stand-in for config 2."""
    A, B = _problem("cplx")
    As = A.to_scipy()
    a = OS.SOLVERS[method](As, B, tol=1e-8, maxit=2000, record=0, order="blas")
    b = OS.SOLVERS[method](As, B, tol=1e-8, maxit=2000, record=0, order="seq")
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    X, rep = srk.solve(M, to_dev(B), method, tol=1e-8, maxit=2000)
    assert rep.outcome == a.outcome, (rep, a.outcome)
    slack = max(0.02 * a.iterations, abs(a.iterations - b.iterations) + 2)
    assert abs(rep.iterations - a.iterations) <= slack
    if rep.outcome == "converged":
        true = np.linalg.norm(B - As @ to_np(X)) / np.linalg.norm(B)
        assert true <= 1e-8


def _deficient(cplx, n_m=10):
    A = synth.conv_diff_3d(n_m, (50.0, 30.0, 10.0), np.complex128 if cplx else np.float64, -0.1j if cplx else 0.0)
    B = synth.random_rhs(A.n, 4, 6, cplx)
    B[:, 3] = B[:, 0] + B[:, 1]   # rank 3 (exact up to the rounding of the sum)
    return A, B


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("method", ["bl_bicg_rq", "bl_bicgstab_rq"])
def test_rank_continuation_lockstep(srk, method, cplx):
    A, B = _deficient(cplx)
    As = A.to_scipy()
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    X, rep = srk.solve(M, to_dev(B), method, tol=1e-8, maxit=2000)
    assert rep.outcome == "breakdown" and rep.breakdown_kind == "rank" and rep.breakdown_iter == 0
    a, env = _envelope(OS.SOLVERS[method], As, B, deflate=True)
    sv, xs, rs = _lockstep(srk, A, B, method, min(K, a.iterations), rank_policy="continue")
    for k in range(min(len(xs), len(a.Xs))):
        assert rel(xs[k], a.Xs[k]) <= env[k], (method, k + 1, "X", rel(xs[k], a.Xs[k]), env[k])
        if a.half_step and k == a.iterations - 1:
            continue
        assert rel(rs[k], a.Rs[k]) <= env[k], (method, k + 1, "C", rel(rs[k], a.Rs[k]), env[k])
    assert sv.report().deflated_cols == 1
    sv.close()
    X, rep = srk.solve(M, to_dev(B), method, tol=1e-8, maxit=2000, rank_policy="continue")
    assert rep.outcome == "converged" and rep.deflated_cols == 1, rep
    X = to_np(X)
    assert np.linalg.norm(B - As @ X) / np.linalg.norm(B) <= 1e-8
    assert rel(X[:, 3], X[:, 0] + X[:, 1]) <= 1e-6


def test_rank_policy_rejected_for_other_methods(srk):
    A, B = _problem("cfg1")
    M = srk.Matrix.from_csr(A)
    with pytest.raises(srk.SrkError):
        srk.solve(M, to_dev(B), "bl_bicg", rank_policy="continue")
