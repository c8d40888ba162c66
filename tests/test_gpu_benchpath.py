"""Parity on the exact path bench.py times (config 3: eGl-QMR and Gl-BiCGStab, FP64,
s = 16, unpreconditioned, multi-kernel): the same operator family (3D 7-point
convection-diffusion, c = (50, 30, 10)) at 48^3 (n = 110,592, above
the single-CTA small-operator limit of 16,384 rows), the same kernels and launch
configuration — the SpMM with the fused eGl vector-sum epilogue, the 6-input / 4-output
block update — compared with the oracle over 20 iterations: X_k, R_k and the recursive
residual history under the §8c.5 envelope, then a full solve under the count rule
(within max(2%, |it_O - it_O'| + 2) of the oracle's two reduction orders) and the
oracle-recomputed true residual."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel, to_dev, to_np

pytestmark = pytest.mark.gpu

K = 20
M3 = 48
S = 16


@pytest.fixture(scope="module")
def srk():
    import paper_1504_04395_b200 as srk
    srk.load_library()
    return srk


@pytest.fixture(scope="module")
def problem():
    A = synth.conv_diff_3d(M3, (50.0, 30.0, 10.0))
    B = synth.random_rhs(A.n, S, 2)
    assert A.n > 16384
    return A, A.to_scipy(), B


@pytest.mark.parametrize("method", ["egl_qmr", "gl_bicgstab"])
def test_benchpath_lockstep(srk, problem, method):
    A, As, B = problem
    a = oracle.solve(method, As, B, tol=1e-8, maxit=2000, record=K, order="blas")
    b = oracle.solve(method, As, B, tol=1e-8, maxit=2000, record=K, order="seq")
    d = [max(rel(x, y), rel(r, q)) for x, y, r, q in zip(a.Xs, b.Xs, a.Rs, b.Rs)]
    env = np.maximum(1e-10, 100 * np.maximum.accumulate(d))
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    sv = srk.Solver(M, S, method, tol=1e-8, maxit=2000, poll_every=1)
    sv.profile(True)
    sv.start(to_dev(B))
    n_it = min(K, len(a.Xs))
    for it in range(n_it):
        assert sv.iterate(1) == 0
        ex = rel(to_np(sv.x()), a.Xs[it])
        er = rel(to_np(sv.residual()), a.Rs[it])
        assert ex <= env[it] and er <= env[it], (method, it + 1, ex, er, env[it])
    h = sv.history(n_it)
    ho = np.array(a.history[:n_it])
    assert np.all(np.abs(h - ho) / ho <= env[:n_it]), (h, ho)
    # the timed kernels ran: the s = 16 SpMM and (eGl-QMR) the 6-input / 4-output update
    launches = sv.profile_launches()
    sigs = {(t, g) for t, g, _, _ in launches}
    assert ("spmm", S) in sigs
    if method == "egl_qmr":
        assert ("update", 16 * 6 + 4) in sigs, sorted(sigs)
        assert ("spmm_adj", 1) in sigs  # the economic A^H vector product
    sv.close()


@pytest.mark.parametrize("method", ["egl_qmr", "gl_bicgstab"])
def test_benchpath_full_solve(srk, problem, method):
    A, As, B = problem
    a = oracle.solve(method, As, B, tol=1e-8, maxit=2000, record=0, order="blas")
    b = oracle.solve(method, As, B, tol=1e-8, maxit=2000, record=0, order="seq")
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    X, rep = srk.solve(M, to_dev(B), method, tol=1e-8, maxit=2000)
    assert rep.outcome == a.outcome == "converged"
    slack = max(0.02 * a.iterations, abs(a.iterations - b.iterations) + 2)
    assert abs(rep.iterations - a.iterations) <= slack, (rep.iterations, a.iterations, b.iterations)
    assert rep.half_step == a.half_step or abs(rep.iterations - a.iterations) > 0
    X = to_np(X)
    true = np.linalg.norm(B - As @ X) / np.linalg.norm(B)
    assert true <= 1e-8
    assert abs(true - rep.final_true_rel_residual) <= 1e-12 + 1e-6 * true
