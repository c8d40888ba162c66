"""Parity on the exact path bench.py times (config 3: eGl-QMR and Gl-BiCGStab, FP64,
s = 16, unpreconditioned, multi-kernel): the same operator family (3D 7-point
convection-diffusion, c = (50, 30, 10)) at 48^3 (n = 110,592, above
the single-CTA small-operator limit of 16,384 rows), the same kernels and launch
configuration — the SpMM with the fused eGl vector-sum epilogue, the 7-input / 5-output
fused tail (D, S, X, R of iteration k and P of iteration k+1, qmr_tail.cu) — compared with the oracle over 20 iterations: X_k, R_k and the recursive
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
    # the timed kernels ran: the s = 16 SpMM and (eGl-QMR) the 7-input / 5-output fused tail
    launches = sv.profile_launches()
    sigs = {(t, g) for t, g, _, _ in launches}
    assert ("spmm", S) in sigs
    if method == "egl_qmr":
        assert ("update", 16 * 7 + 5) in sigs, sorted(sigs)
        # P is formed standalone only in the first iteration (2 in / 1 out at width s appears once
        # besides the Ṽ update of every iteration)
        n_tail = sum(1 for t, g, _, _ in launches if (t, g) == ("update", 16 * 7 + 5))
        assert n_tail == n_it
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


_FUSE_CODE = """
import sys; sys.path.insert(0, {root!r})
import numpy as np, torch, synth, paper_1504_04395_b200 as srk
srk.load_library()
A = synth.conv_diff_3d({m}, (20.0, 10.0, 5.0), {dt})
B = synth.random_rhs(A.n, {s}, 2, {cplx})
M = srk.Matrix.from_csr(A, need_adjoint=True)
sv = srk.Solver(M, {s}, {method!r}, tol=1e-8, maxit=2000, poll_every={poll}, use_graph={graph})
sv.start(torch.from_numpy(B).cuda())
sv.iterate({k})
np.save({out!r}, np.stack([sv.x().cpu().numpy(), sv.residual().cpu().numpy()]))
X, rep = srk.solve(M, torch.from_numpy(B).cuda(), {method!r}, tol=1e-8, maxit=2000)
print(rep.outcome, rep.iterations)
"""


@pytest.mark.parametrize("method", ["egl_qmr", "gl_qmr"])
@pytest.mark.parametrize("cplx,s", [(False, 16), (True, 8), (False, 5), (False, 6), (True, 3)])
def test_qmr_fused_tail_equals_separate_updates(srk, tmp_path, method, cplx, s):
    """The fused tail (qmr_tail.cu: D, S, X, R of iteration k and P of iteration k+1 in one
    pass, next iteration's 1/rho and c1 from coefficient phase 4) keeps the per-element FMA
    order of the two separate updates: X_k and R_k after 12 iterations — stepped one by one
    and inside a replayed CUDA graph — are bitwise those of the unfused plan
    (SRK_NO_QMR_FUSE=1, a subprocess: the switches are read once), and the full solves agree in
    outcome and count. eGl-QMR at whole 16-byte units per row also carries its n-vectors in the
    block kernels (qmr_vt_kernel and the tail's vector part), which changes the summation order
    of ||Ṽ||^2, <Ṽ, W̃>, ||W̃||^2: bitwise with that switched off (SRK_NO_QMR_VEC_FUSE=1), within
    1e-11 with it on (the operator is the 28^3 stencil with c = (20, 10, 5), on which the oracle's
    own two summation orders differ by 4e-16 / 1e-14 in X / R at iteration 12 and its counts do not
    move under 1e-15 perturbations of B; with c = (50, 30, 10) at this size a near-breakdown at
    iteration 9 spreads the oracle itself by 4e-10 and its counts by 6%; the lock step against the
    oracle is test_benchpath_lockstep). Widths 5 / 6 / 3
    give ragged last CTAs, rows of 3 units (the division path) and the no-vector fallback."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    m = 28  # n = 21,952 > the single-CTA limit
    res = {}
    novec = {"SRK_NO_QMR_VEC_FUSE": "1"}
    for tag, env, poll in (("fused", novec, 1), ("graph", novec, 4), ("plain", {"SRK_NO_QMR_FUSE": "1"}, 1),
                           ("vec", {}, 1), ("vecgraph", {}, 4)):
        out = str(tmp_path / f"{tag}.npy")
        code = _FUSE_CODE.format(root=root, m=m, dt="np.complex128" if cplx else "np.float64", s=s, cplx=cplx,
                                 method=method, poll=poll, graph=tag.endswith("graph"), k=12, out=out)
        r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-800:]
        res[tag] = (np.load(out), r.stdout.split()[-2:])
    ref = res["plain"][0]
    assert np.isfinite(ref).all()
    assert np.array_equal(res["fused"][0], ref)
    assert np.array_equal(res["graph"][0], ref)
    assert res["fused"][1] == res["plain"][1] == res["graph"][1], (res["fused"][1], res["plain"][1])
    assert np.array_equal(res["vec"][0], res["vecgraph"][0])
    for j in range(2):
        assert rel(res["vec"][0][j], ref[j]) <= 1e-11, (j, rel(res["vec"][0][j], ref[j]))
    assert res["vec"][1][0] == res["plain"][1][0] == "converged"
    it_v, it_p = int(res["vec"][1][1]), int(res["plain"][1][1])
    assert abs(it_v - it_p) <= max(2, 0.02 * it_p), (it_v, it_p)


@pytest.mark.parametrize("method", ["gl_bicgstab", "egl_bicg"])
@pytest.mark.parametrize("cplx,s", [(False, 16), (True, 12), (False, 5), (False, 6), (True, 3)])
def test_flat_plans_equal_generic_updates(srk, tmp_path, method, cplx, s):
    """eGl-BiCG's two block updates as lean flat kernels that carry r̂ and p̂ (egl_flat.cu) and
    Gl-BiCGStab's three updates as flat plans (flat_upd.cu: the FMA order of the generic
    upd_kernel per element, another summation order in ||S||^2, <R, R~>, ||R||^2) against the
    generic kernels (SRK_NO_FLAT_UPDATE=1, a subprocess: the switch is read once): X_k and R_k
    after 12 iterations within 1e-11 (well-conditioned operator, see the QMR test above),
    stepped and graph-replayed runs bitwise equal, full solves with the same outcome and counts
    within 2. Width 12 complex is config 4's; 5 / 3 give ragged last CTAs."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for tag, env, poll in (("flat", {}, 1), ("flatgraph", {}, 4), ("plain", {"SRK_NO_FLAT_UPDATE": "1"}, 1)):
        out = str(tmp_path / f"{tag}.npy")
        code = _FUSE_CODE.format(root=root, m=28, dt="np.complex128" if cplx else "np.float64", s=s, cplx=cplx,
                                 method=method, poll=poll, graph=tag.endswith("graph"), k=12, out=out)
        r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-800:]
        res[tag] = (np.load(out), r.stdout.split()[-2:])
    ref = res["plain"][0]
    assert np.isfinite(ref).all()
    assert np.array_equal(res["flat"][0], res["flatgraph"][0])
    for j in range(2):
        assert rel(res["flat"][0][j], ref[j]) <= 1e-11, (j, rel(res["flat"][0][j], ref[j]))
    assert res["flat"][1][0] == res["plain"][1][0] == "converged"
    it_f, it_p = int(res["flat"][1][1]), int(res["plain"][1][1])
    assert abs(it_f - it_p) <= max(2, 0.02 * it_p), (it_f, it_p)
