"""GPU lock-step parity of all 13 methods against the oracle (SURVEY §8c.5
envelope rule): per-iteration iterates X_k (k <= 20) agree
to max(1e-10, 100 * delta_k), where delta_k is the oracle's own spread between
two reduction orders; iteration counts agree within max(2%, |it - it'| + 2);
the final true residual, recomputed by the oracle from the GPU's X, is <= tol."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import rel, to_dev, to_np

pytestmark = pytest.mark.gpu

K = 20


@pytest.fixture(scope="module")
def srk():
    import paper_1504_04395_b200 as srk
    srk.load_library()
    return srk


def crel(a, b, method):
    """Relative error of a block: whole-block Frobenius ratio, or for the Li variants
    (s independent column recurrences) the worst per-column ratio, so a
    column-local error in a small-norm column is not diluted by the others."""
    if method.startswith("li_") and np.ndim(b) == 2:
        return max(rel(a[:, j], b[:, j]) for j in range(b.shape[1]))
    return rel(a, b)


def envelope(method, As, B, tol, maxit=2000, k=K):
    """SURVEY §8c.5 rule 2: the per-iteration bound max(1e-10, 100 max_{j<=k} delta_j),
    delta the oracle's own spread between two reduction orders over X_k and R_k (C_k)."""
    a = oracle.solve(method, As, B, tol=tol, maxit=maxit, record=k, order="blas")
    b = oracle.solve(method, As, B, tol=tol, maxit=maxit, record=k, order="seq")
    d = [max(crel(x, y, method), crel(r, q, method)) for x, y, r, q in zip(a.Xs, b.Xs, a.Rs, b.Rs)]
    env = np.maximum(1e-10, 100 * np.maximum.accumulate(d)) if d else np.array([])
    return a, b, env


def lockstep(srk, M, B, method, n_it, tol):
    sv = srk.Solver(M, B.shape[1], method, tol=tol, maxit=2000, poll_every=1)
    sv.start(to_dev(B))
    xs, rs = [], []
    for _ in range(n_it):
        st = sv.iterate(1)
        xs.append(to_np(sv.x()))
        rs.append(to_np(sv.residual()))
        if st != 0:
            break
    sv.rs = rs
    return sv, xs


def _problem(name):
    if name == "cfg1":
        A, B = synth.make_config(1)
        return A, B
    if name == "cplx":  # small complex stand-in for config 2 (3D conv-diff 10^3, shift -0.1i, s=3)
        A = synth.conv_diff_3d(10, (50.0, 30.0, 10.0), np.complex128, -0.1j)
        B = synth.random_rhs(A.n, 3, 1, True)
        return A, B
    if name == "lattice":  # config 4 at 4^4 sites (n = 3072, s = 12 complex)
        return synth.make_config(4, m=4)
    if name == "cfg2s":  # config 2 operator at 16^3 with its s = 8 complex RHS
        return synth.make_config(2, m=16)
    raise ValueError(name)


@pytest.mark.parametrize("prob", ["cfg1", "cplx"])
@pytest.mark.parametrize("method", oracle.METHODS)
def test_lockstep_parity(srk, method, prob):
    A, B = _problem(prob)
    As = A.to_scipy()
    tol = 1e-8
    a, b, env = envelope(method, As, B, tol)
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    sv, xs = lockstep(srk, M, B, method, min(K, a.iterations), tol)
    n_cmp = min(len(xs), len(a.Xs))
    assert n_cmp >= 1
    for k in range(n_cmp):
        err = crel(xs[k], a.Xs[k], method)
        assert err <= env[k], (method, prob, k + 1, "X", err, env[k])
        if a.half_step and k == a.iterations - 1:
            continue  # a half-step exit records S (never materialised on the GPU): X only
        err = crel(sv.rs[k], a.Rs[k], method)
        assert err <= env[k], (method, prob, k + 1, "R" if a.Rs[k].shape == B.shape else "C", err, env[k])
    sv.close()


def oracle_ensemble(method, As, B, tol, n_pert=4):
    """The method's own outcome spread under rounding: three
    reduction orders plus 1e-15 relative perturbations of B. Block variants are
    chaotic on config 1 (the paper reports Bl-BiCG diverging on Ex. 1)."""
    runs = [oracle.solve(method, As, B, tol=tol, maxit=2000, record=0, order=o) for o in ("blas", "seq", "rev")]
    for seed in range(n_pert):
        Bp = B * (1 + 1e-15 * np.random.default_rng(seed).standard_normal(B.shape))
        runs.append(oracle.solve(method, As, Bp, tol=tol, maxit=2000, record=0))
    return runs


@pytest.mark.parametrize("prob", ["cfg1", "cplx"])
@pytest.mark.parametrize("method", oracle.METHODS)
def test_full_solve(srk, method, prob):
    A, B = _problem(prob)
    As = A.to_scipy()
    tol = 1e-8
    runs = oracle_ensemble(method, As, B, tol)
    a = runs[0]
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    X, rep = srk.solve(M, to_dev(B), method, tol=tol, maxit=2000)
    X = to_np(X)
    outcomes = {r.outcome for r in runs}
    assert rep.outcome in outcomes, (rep, outcomes)
    same = [r for r in runs if r.outcome == rep.outcome]
    lo = min(r.iterations for r in same)
    hi = max(r.iterations for r in same)
    if rep.outcome == "converged":
        # SURVEY §8c.5 rule 3: within max(2%, spread + 2) of the oracle's count, the spread
        # being the oracle ensemble's own (its reduction orders and 1e-15 perturbations of
        # B; |it_O - it_O'| in the rule's two-order form)
        slack = max(0.02 * a.iterations, (hi - lo) + 2)
        assert abs(rep.iterations - a.iterations) <= slack, (rep.iterations, a.iterations, lo, hi)
        # the oracle's own SpMM recomputes the true residual from the GPU's X
        true = np.linalg.norm(B - As @ X) / np.linalg.norm(B)
        assert true <= tol
        assert abs(true - rep.final_true_rel_residual) <= 1e-12 + 1e-6 * true
    if rep.iterations == a.iterations and rep.half_step == a.half_step and rep.outcome == a.outcome:
        assert rep.matvec_cols_A == a.matvec_cols_A and rep.matvec_cols_AH == a.matvec_cols_AH


def test_solve_host_matches_device(srk):
    A, B = synth.make_config(1)
    M = srk.Matrix.from_csr(A)
    Xd, rd = srk.solve(M, to_dev(B), "egl_bicg")
    Xh, rh = srk.solve_host(M, B, "egl_bicg")
    assert rd.iterations == rh.iterations
    assert np.array_equal(to_np(Xd), Xh)  # same kernels, same order: bitwise


def test_determinism(srk):
    A, B = synth.make_config(1)
    M = srk.Matrix.from_csr(A)
    X1, r1 = srk.solve(M, to_dev(B), "bl_bicgstab_rq")
    X2, r2 = srk.solve(M, to_dev(B), "bl_bicgstab_rq")
    assert r1.iterations == r2.iterations and np.array_equal(to_np(X1), to_np(X2))


@pytest.mark.parametrize("method", oracle.METHODS)
def test_trivial_identity_and_zero_rhs(srk, method):
    import scipy.sparse as sp
    A = sp.identity(300, format="csr")
    B = np.random.default_rng(1).standard_normal((300, 2))
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    X, rep = srk.solve(M, to_dev(B), method, tol=1e-12, maxit=5)
    assert rep.outcome == "converged" and rep.iterations == 1 and rel(to_np(X), B) < 1e-14, (method, rep)
    X, rep = srk.solve(M, to_dev(np.zeros((300, 2))), method, tol=1e-12, maxit=5)
    assert rep.outcome == "converged" and rep.iterations == 0


def test_prop1_counters(srk):
    A, B = synth.make_config(1)
    s = B.shape[1]
    for method, (ca, cah) in {"gl_bicg": (s, s), "egl_bicg": (s, 1), "bl_bicg": (s, s),
                              "gl_bicgstab": (2 * s, 0), "egl_qmr": (s, 1)}.items():
        M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
        sv = srk.Solver(M, s, method, tol=1e-300, maxit=7)
        sv.start(to_dev(B))
        sv.iterate(7)
        r = sv.report()
        assert r.iterations == 7 and r.matvec_cols_A == 7 * ca and r.matvec_cols_AH == 7 * cah, method


def test_distributed_operator_single_rank_matches(srk):
    """srk_matrix_create_dist with one rank (plan = whole matrix, no ghosts) runs the
    same kernels: the solve is bitwise identical to the plain operator's."""
    A, B = synth.make_config(1)
    off = srk.partition_rows(A.row_ptr, 1)
    Md = srk.DistMatrix(A, off, 0, need_adjoint=True)
    M = srk.Matrix.from_csr(A)
    X1, r1 = srk.solve(M, to_dev(B), "egl_qmr")
    X2, r2 = srk.solve(Md, to_dev(B), "egl_qmr")
    assert r1.iterations == r2.iterations and np.array_equal(to_np(X1), to_np(X2))


LATTICE_METHODS = ["li_bicgstab", "gl_bicgstab", "bl_bicgstab", "bl_bicgstab_rq"]


@pytest.mark.parametrize("method", LATTICE_METHODS)
def test_lattice_lockstep_and_solve(srk, method):
    """Config 4's methods on the 4^4 lattice (complex, s = 12): lock-step parity and full solve."""
    test_lockstep_parity(srk, method, "lattice")
    test_full_solve(srk, method, "lattice")


@pytest.mark.parametrize("method", LATTICE_METHODS)
def test_lattice_bsr_lockstep_and_solve(srk, method):
    """Config 4's methods with the operator in BSR-12 form (unit diagonal implied,
    tensor-core block product): lock-step parity with the oracle (scalar CSR) and
    the full solve on the 4^4 lattice."""
    A, B = _problem("lattice")
    As = A.to_scipy()
    tol = 1e-8
    a, _, env = envelope(method, As, B, tol)
    brp, bcol, blocks = synth.lattice_4d_bsr(4)
    M = srk.Matrix.from_bsr(brp, bcol, blocks, unit_diag=True)
    sv, xs = lockstep(srk, M, B, method, min(K, a.iterations), tol)
    for k in range(min(len(xs), len(a.Xs))):
        assert rel(xs[k], a.Xs[k]) <= env[k], (method, k + 1)
    sv.close()
    X, rep = srk.solve(M, to_dev(B), method, tol=tol, maxit=2000)
    assert rep.outcome == "converged"
    assert np.linalg.norm(B - As @ to_np(X)) / np.linalg.norm(B) <= tol


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("method", ["bl_bicg", "bl_bicg_rq", "bl_qmr", "bl_bicgstab", "bl_bicgstab_rq"])
def test_block_methods_wide(srk, method, cplx):
    """Block methods at s = 19 (the paper's Ex. 2/3 width): s x s coefficient
    updates in the capacity-32 kernels and the s x s Grams on the tensor cores;
    lock-step parity and the full solve on a 3D convection-diffusion operator."""
    A = synth.conv_diff_3d(9, (10.0, 5.0, 2.0), np.complex128 if cplx else np.float64, -0.1j if cplx else 0.0)
    B = synth.random_rhs(A.n, 19, 3, cplx)
    As = A.to_scipy()
    tol = 1e-8
    a, _, env = envelope(method, As, B, tol)
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    sv, xs = lockstep(srk, M, B, method, min(K, a.iterations), tol)
    for k in range(min(len(xs), len(a.Xs))):
        assert rel(xs[k], a.Xs[k]) <= env[k], (method, k + 1, rel(xs[k], a.Xs[k]), env[k])
    sv.close()
    X, rep = srk.solve(M, to_dev(B), method, tol=tol, maxit=2000)
    if rep.outcome == "converged":
        assert np.linalg.norm(B - As @ to_np(X)) / np.linalg.norm(B) <= tol
    else:  # the oracle must see the same outcome
        assert rep.outcome in {r.outcome for r in oracle_ensemble(method, As, B, tol, n_pert=1)}


@pytest.mark.parametrize("method", ["bl_bicg_rq", "bl_qmr", "bl_bicgstab_rq"])
def test_config2_block_methods(srk, method):
    """Config 2's methods (block BiCG / QMR / BiCGStab with QR) on its operator at 16^3, s = 8 complex."""
    test_lockstep_parity(srk, method, "cfg2s")
    test_full_solve(srk, method, "cfg2s")


def test_config5_egl_bicg_s32(srk):
    """Config 5's full solve (eGl-BiCG, s = 32) on the power-law operator at n = 2^14."""
    A = synth.power_law(1 << 14, seed=4)
    B = synth.random_rhs(A.n, 32, 4)
    As = A.to_scipy()
    a = oracle.solve("egl_bicg", As, B, tol=1e-8, maxit=2000, record=20)
    M = srk.Matrix.from_csr(A)
    sv, xs = lockstep(srk, M, B, "egl_bicg", min(20, a.iterations), 1e-8)
    for k in range(min(len(xs), len(a.Xs))):
        assert rel(xs[k], a.Xs[k]) < 1e-10, k
    X, rep = srk.solve(M, to_dev(B), "egl_bicg", tol=1e-8)
    assert rep.outcome == "converged"
    runs = oracle_ensemble("egl_bicg", As, B, 1e-8, n_pert=1)
    its = [r.iterations for r in runs]
    slack = max(2, 0.02 * a.iterations)
    if max(its) - min(its) <= slack:  # BiCG over ~700 iterations: compare only if the oracle itself is stable
        assert min(its) - slack <= rep.iterations <= max(its) + slack, (rep.iterations, its)
    assert np.linalg.norm(B - As @ to_np(X)) / np.linalg.norm(B) <= 1e-8


@pytest.mark.parametrize("method", ["egl_bicg", "bl_bicgstab_rq", "gl_qmr", "bl_qmr"])
def test_cuda_graph_replay_is_bitwise_identical(srk, method):
    """The iterations between two polls replayed as one captured CUDA graph give the
    same bits, iteration count and report as launching them one by one."""
    A, B = synth.make_config(1)
    M = srk.Matrix.from_csr(A, need_adjoint=srk.NEEDS_ADJOINT[method])
    out = []
    for g in (False, True):
        sv = srk.Solver(M, B.shape[1], method, tol=1e-8, maxit=2000, poll_every=16, use_graph=g)
        sv.start(to_dev(B))
        sv.iterate(2000)
        r = sv.report()
        out.append((to_np(sv.x()), r.iterations, r.outcome))
        sv.close()
    assert out[0][1] == out[1][1] and out[0][2] == out[1][2]
    assert np.array_equal(out[0][0], out[1][0])


@pytest.mark.parametrize("method", ["egl_bicg", "egl_qmr"])
@pytest.mark.parametrize("cplx", [False, True])
def test_small_operator_single_kernel_iteration(srk, cplx, method):
    """eGl-BiCG / eGl-QMR on a small operator run their iterations as ONE single-CTA
    kernel (egl_bicg_small_kernel / egl_qmr_small_kernel: the steps of Alg. 4 / App. A.2
    separated by CTA barriers, the coefficient phases the same device code): one launch
    per iterate() call, iterates in lock step with the oracle (envelope rule), and the
    same outcome as the multi-kernel sequence
    (SRK_NO_SMALL_KERNEL=1, checked in a subprocess: the switch is read once)."""
    import os
    import subprocess
    import sys
    A, B = _problem("cplx" if cplx else "cfg1")
    M = srk.Matrix.from_csr(A, need_adjoint=True)
    sv = srk.Solver(M, B.shape[1], method, tol=1e-8, maxit=2000, poll_every=1)
    sv.start(to_dev(B))
    sv.iterate(2)
    sv.profile(True)
    sv.iterate(5)
    recs = sv.profile_launches()
    assert len(recs) == 1, recs  # the five iterations (end-of-iteration steps included) in one launch
    sv.profile(False)
    assert sv.report().iterations == 7
    sv.close()
    a, _, env = envelope(method, A.to_scipy(), B, 1e-8)
    sv, xs = lockstep(srk, M, B, method, min(K, a.iterations), 1e-8)
    for k, x in enumerate(xs):
        assert rel(x, a.Xs[k]) <= env[k], (k, rel(x, a.Xs[k]), env[k])
    sv.close()
    X, rep = srk.solve(M, to_dev(B), method, tol=1e-8, maxit=2000)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (f"import sys; sys.path.insert(0, {root!r})\n"
            "import numpy as np, torch, paper_1504_04395_b200 as srk\n"
            "from tests.test_gpu_solvers import _problem\n"
            "srk.load_library()\n"
            f"A, B = _problem({'cplx' if cplx else 'cfg1'!r})\n"
            "M = srk.Matrix.from_csr(A, need_adjoint=True)\n"
            f"X, rep = srk.solve(M, torch.from_numpy(B).cuda(), {method!r}, tol=1e-8, maxit=2000)\n"
            "print(rep.outcome, rep.iterations)\n")
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "SRK_NO_SMALL_KERNEL": "1"},
                         capture_output=True, text=True, timeout=600)
    outcome, its = out.stdout.split()[-2:]
    assert outcome == rep.outcome and abs(int(its) - rep.iterations) <= max(2, 0.02 * rep.iterations), \
        (out.stdout, out.stderr[-400:], rep)


@pytest.mark.parametrize("method", ["egl_bicg", "egl_qmr"])
@pytest.mark.parametrize("s", [1, 12])
def test_small_operator_widths(srk, method, s):
    """The single-CTA kernels at the widths their register paths do not cover by
    default (s = 1; s = 12 > 8 takes the column-loop product), on a ragged row count
    (n = 29^2 = 841, not a multiple of the CTA's warps): lock step with the oracle
    over 20 iterations, then a full solve meeting the tolerance."""
    A = synth.conv_diff_2d(29, (20.0, 20.0))
    B = synth.random_rhs(A.n, s, 5)
    M = srk.Matrix.from_csr(A, need_adjoint=True)
    a, _, env = envelope(method, A.to_scipy(), B, 1e-8)
    sv, xs = lockstep(srk, M, B, method, min(K, a.iterations), 1e-8)
    for k, x in enumerate(xs):
        assert rel(x, a.Xs[k]) <= env[k], (k, rel(x, a.Xs[k]), env[k])
    sv.close()
    X, rep = srk.solve(M, to_dev(B), method, tol=1e-8, maxit=2000)
    assert rep.outcome == "converged"
    assert np.linalg.norm(B - A.to_scipy() @ to_np(X)) / np.linalg.norm(B) <= 1e-8
