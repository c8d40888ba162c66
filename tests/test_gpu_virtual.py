"""Distributed (row-partitioned) solver path on ONE GPU through the virtual-partition
transport (SURVEY §4 "Multi-GPU without a cluster", §8(e)): k virtual ranks, each with
its own context, stream and host thread, run the library's distributed code — halo
exchange of P rows into the ghost tail before every SpMM, one allreduce of the per-rank
partials per reduction point (staged out of place) — and the concatenated iterates must
match the oracle under the §8c.5 envelope, X_k and R_k, for k = 2, 4, 8 ranks.
"""
import threading

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel

pytestmark = pytest.mark.gpu

K = 12


@pytest.fixture(scope="module")
def srk():
    import paper_1504_04395_b200 as srk
    srk.load_library()
    return srk


def run_virtual(srk, A, B, method, k, n_it=K, full=False, tol=1e-8, maxit=2000, bsr=None):
    """k threads, one virtual rank each; returns per-iteration global X_k and R_k (lock
    step) or the final X and every rank's report (full solve). bsr = (block_row_ptr,
    block_col, blocks): the BSR-12 operator split by block rows (t-slabs)."""
    import torch
    torch.cuda.synchronize()
    if bsr is not None:
        boff = srk.partition_rows(bsr[0], k)
        off = boff * 12
    else:
        off = srk.partition_rows(A.row_ptr, k)
    grp = srk.VirtualGroup(k)
    out = [None] * k
    errs = []

    def worker(r):
        try:
            ctx = srk.Context(stream=torch.cuda.Stream())
            grp.attach(ctx, r)
            if bsr is not None:
                M = srk.DistMatrix.from_bsr(*bsr, boff, r, unit_diag=True, ctx=ctx)
            else:
                M = srk.DistMatrix(A, off, r, need_adjoint=srk.NEEDS_ADJOINT[method], ctx=ctx)
            Bl = torch.from_numpy(np.ascontiguousarray(B[off[r]:off[r + 1]])).cuda()
            torch.cuda.synchronize()
            if full:
                X, rep = srk.solve(M, Bl, method, tol=tol, maxit=maxit)
                torch.cuda.synchronize()
                out[r] = (X.cpu().numpy(), rep)
            else:
                sv = srk.Solver(M, B.shape[1], method, tol=tol, maxit=maxit, poll_every=1)
                sv.start(Bl)
                xs, rs = [], []
                for _ in range(n_it):
                    st = sv.iterate(1)
                    xs.append(sv.x().cpu().numpy())
                    rs.append(sv.residual().cpu().numpy())
                    if st != 0:
                        break
                out[r] = (xs, rs)
                sv.close()
            M.close()
            ctx.close()
        except Exception as e:  # surfaced in the main thread
            errs.append((r, repr(e)))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(k)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "virtual ranks hung"
    grp.close()
    assert not errs, errs
    return off, out


def _problem(name):
    if name == "real":      # 3D 7-point conv-diff 12^3 (config 3's stencil), s = 4
        A = synth.conv_diff_3d(12)
        return A, synth.random_rhs(A.n, 4, 2)
    if name == "cplx":      # config 2's operator at 10^3, s = 3 complex
        A = synth.conv_diff_3d(10, (50.0, 30.0, 10.0), np.complex128, -0.1j)
        return A, synth.random_rhs(A.n, 3, 1, True)
    if name == "irregular":  # power-law rows (config 5's structure), ragged partition
        A = synth.power_law(3000, 5)
        return A, synth.random_rhs(A.n, 4, 4)
    raise ValueError(name)


def envelope(method, As, B, tol=1e-8, k=K):
    a = oracle.solve(method, As, B, tol=tol, maxit=2000, record=k, order="blas")
    b = oracle.solve(method, As, B, tol=tol, maxit=2000, record=k, order="seq")
    d = [max(rel(x, y), rel(r, q)) for x, y, r, q in zip(a.Xs, b.Xs, a.Rs, b.Rs)]
    env = np.maximum(1e-10, 100 * np.maximum.accumulate(d)) if d else np.array([])
    return a, env


@pytest.mark.parametrize("k", [2, 4, 8])
@pytest.mark.parametrize("method,prob", [("egl_qmr", "real"), ("bl_bicgstab_rq", "real"), ("egl_qmr", "cplx"),
                                         ("bl_bicg_rq", "cplx"), ("gl_bicgstab", "irregular"),
                                         ("li_bicg", "real")])
def test_virtual_lockstep(srk, method, prob, k):
    A, B = _problem(prob)
    As = A.to_scipy()
    a, env = envelope(method, As, B)
    off, out = run_virtual(srk, A, B, method, k, n_it=min(K, a.iterations))
    n_cmp = min(len(out[0][0]), len(a.Xs))
    assert n_cmp >= 1
    rq = method.endswith("_rq")
    for it in range(n_cmp):
        X = np.concatenate([out[r][0][it] for r in range(k)])
        err = rel(X, a.Xs[it])
        assert err <= env[it], (method, prob, k, it + 1, "X", err, env[it])
        if a.half_step and it == a.iterations - 1:
            continue  # a half-step exit records S, which the GPU never materialises
        if rq:  # C_k is s x s, replicated on every rank
            for r in range(k):
                assert rel(out[r][1][it], a.Rs[it]) <= env[it], (method, k, it + 1, "C", r)
        else:
            R = np.concatenate([out[r][1][it] for r in range(k)])
            err = rel(R, a.Rs[it])
            assert err <= env[it], (method, prob, k, it + 1, "R", err, env[it])


@pytest.mark.parametrize("k", [2, 4])
@pytest.mark.parametrize("method", ["egl_qmr", "bl_bicgstab_rq", "gl_bicgstab"])
def test_virtual_full_solve(srk, method, k):
    """Full distributed solve: every rank reports the same outcome and count, the count
    agrees with the oracle's two reduction orders (|it_O - it_O'| + 2, and 2%), and the
    oracle's SpMM recomputes the true residual from the gathered X."""
    A, B = _problem("real")
    As = A.to_scipy()
    tol = 1e-8
    a = oracle.solve(method, As, B, tol=tol, maxit=2000, record=0, order="blas")
    b = oracle.solve(method, As, B, tol=tol, maxit=2000, record=0, order="seq")
    off, out = run_virtual(srk, A, B, method, k, full=True, tol=tol)
    reps = [o[1] for o in out]
    assert len({(r.outcome, r.iterations, r.half_step) for r in reps}) == 1, reps
    rep = reps[0]
    assert rep.outcome == a.outcome == "converged"
    slack = max(0.02 * a.iterations, abs(a.iterations - b.iterations) + 2)
    assert abs(rep.iterations - a.iterations) <= slack, (rep.iterations, a.iterations, b.iterations)
    X = np.concatenate([o[0] for o in out])
    true = np.linalg.norm(B - As @ X) / np.linalg.norm(B)
    assert true <= tol
    assert abs(true - rep.final_true_rel_residual) <= 1e-12 + 1e-6 * true


def test_virtual_deterministic_and_one_rank_equal(srk):
    """Bitwise rerun determinism at a fixed rank count; one virtual rank is the plain
    single-GPU operator (no transport at all)."""
    A, B = _problem("real")
    _, o1 = run_virtual(srk, A, B, "egl_qmr", 4, n_it=6)
    _, o2 = run_virtual(srk, A, B, "egl_qmr", 4, n_it=6)
    for r in range(4):
        for x, y in zip(o1[r][0], o2[r][0]):
            assert np.array_equal(x, y)
    _, one = run_virtual(srk, A, B, "egl_qmr", 1, n_it=6)
    import torch
    M = srk.Matrix.from_csr(A)
    sv = srk.Solver(M, B.shape[1], "egl_qmr", poll_every=1)
    sv.start(torch.from_numpy(B).cuda())
    for it in range(6):
        sv.iterate(1)
        # same kernels except the small-operator kernel the plain operator may take
        assert rel(sv.x().cpu().numpy(), one[0][0][it]) <= 1e-12
    sv.close()


@pytest.mark.parametrize("k", [2, 4])
@pytest.mark.parametrize("method", ["gl_bicgstab", "bl_bicgstab_rq", "li_bicgstab"])
def test_virtual_bsr_lattice(srk, method, k):
    """Config 4's operator (4D lattice, 12 complex dof per site, A = I - kappa H) as BSR-12
    split into t-slabs over k virtual ranks: lock-step X_k / R_k against the
    oracle on the same operator in scalar CSR form, then a full solve's count and residual."""
    A, B = synth.make_config(4, m=4)
    bsr = synth.lattice_4d_bsr(4)
    As = A.to_scipy()
    a, env = envelope(method, As, B)
    off, out = run_virtual(srk, A, B, method, k, n_it=min(K, a.iterations), bsr=bsr)
    n_cmp = min(len(out[0][0]), len(a.Xs))
    rq = method.endswith("_rq")
    for it in range(n_cmp):
        X = np.concatenate([out[r][0][it] for r in range(k)])
        assert rel(X, a.Xs[it]) <= env[it], (method, k, it + 1, "X", rel(X, a.Xs[it]), env[it])
        if a.half_step and it == a.iterations - 1:
            continue
        if not rq:
            R = np.concatenate([out[r][1][it] for r in range(k)])
            assert rel(R, a.Rs[it]) <= env[it], (method, k, it + 1, "R")
    off, out = run_virtual(srk, A, B, method, k, full=True, bsr=bsr)
    rep = out[0][1]
    assert rep.outcome == "converged" and abs(rep.iterations - a.iterations) <= max(2, 0.02 * a.iterations)
    X = np.concatenate([o[0] for o in out])
    assert np.linalg.norm(B - As @ X) / np.linalg.norm(B) <= 1e-8
