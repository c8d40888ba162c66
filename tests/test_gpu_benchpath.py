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


_DUMP_CODE = """
import sys; sys.path.insert(0, {root!r})
import numpy as np, torch, synth, paper_1504_04395_b200 as srk
srk.load_library()
out = {{}}
for method, cplx, s in {cases!r}:
    A = synth.conv_diff_3d(28, (20.0, 10.0, 5.0), np.complex128 if cplx else np.float64)  # n = 21,952 > the single-CTA limit
    B = synth.random_rhs(A.n, s, 2, cplx)
    M = srk.Matrix.from_csr(A, need_adjoint=True)
    for tag, poll, graph in (("step", 1, False), ("graph", 4, True)):
        sv = srk.Solver(M, s, method, tol=1e-8, maxit=2000, poll_every=poll, use_graph=graph)
        sv.start(torch.from_numpy(B).cuda())
        sv.iterate(12)
        out[f"{{method}}_{{int(cplx)}}_{{s}}_{{tag}}"] = np.stack([sv.x().cpu().numpy(), sv.residual().cpu().numpy()])
        sv.close()
    X, rep = srk.solve(M, torch.from_numpy(B).cuda(), method, tol=1e-8, maxit=2000)
    out[f"{{method}}_{{int(cplx)}}_{{s}}_count"] = np.array([rep.iterations if rep.outcome == "converged" else -1])
np.savez({path!r}, **out)
print("DUMP_OK")
"""

QMR_CASES = [(m, c, s) for m in ("egl_qmr", "gl_qmr") for c, s in ((False, 16), (True, 8), (False, 5), (False, 6), (True, 3))]
FLAT_CASES = [(m, c, s) for m in ("gl_bicgstab", "egl_bicg", "gl_bicg", "gl_qmr")
              for c, s in ((False, 16), (True, 12), (False, 5), (False, 6), (True, 3))]


def _dump(tmp, name, cases, env):
    """X_12, R_12 (stepped one by one, and with the last 8 iterations replayed as a CUDA graph) and
    the full-solve count of every case, in ONE subprocess per switch setting (the A/B switches
    are read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = str(tmp / f"{name}.npz")
    code = _DUMP_CODE.format(root=root, cases=cases, path=path)
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=1800)
    assert r.returncode == 0 and "DUMP_OK" in r.stdout, r.stderr[-800:]
    return dict(np.load(path))


@pytest.fixture(scope="module")
def qmr_dumps(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("qmr_fuse")
    return {"vec": _dump(tmp, "vec", QMR_CASES, {}),
            "fused": _dump(tmp, "fused", QMR_CASES, {"SRK_NO_QMR_VEC_FUSE": "1"}),
            "plain": _dump(tmp, "plain", QMR_CASES, {"SRK_NO_QMR_FUSE": "1"})}


@pytest.fixture(scope="module")
def flat_dumps(tmp_path_factory):
    tmp = tmp_path_factory.mktemp("flat")
    return {"flat": _dump(tmp, "flat", FLAT_CASES, {}),
            "plain": _dump(tmp, "plain", FLAT_CASES, {"SRK_NO_FLAT_UPDATE": "1"})}


@pytest.mark.parametrize("method,cplx,s", QMR_CASES)
def test_qmr_fused_tail_equals_separate_updates(qmr_dumps, method, cplx, s):
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
    oracle is test_benchpath_lockstep). Widths 5 / 6 / 3 give ragged last CTAs, rows of 3 units
    (the division path) and the no-vector fallback."""
    key = f"{method}_{int(cplx)}_{s}_"
    ref = qmr_dumps["plain"][key + "step"]
    assert np.isfinite(ref).all()
    assert np.array_equal(qmr_dumps["fused"][key + "step"], ref)
    assert np.array_equal(qmr_dumps["fused"][key + "graph"], ref)
    assert np.array_equal(qmr_dumps["plain"][key + "graph"], ref)
    it_p = int(qmr_dumps["plain"][key + "count"][0])
    assert it_p > 0 and int(qmr_dumps["fused"][key + "count"][0]) == it_p
    vec = qmr_dumps["vec"][key + "step"]
    assert np.array_equal(vec, qmr_dumps["vec"][key + "graph"])
    for j in range(2):
        assert rel(vec[j], ref[j]) <= 1e-11, (j, rel(vec[j], ref[j]))
    it_v = int(qmr_dumps["vec"][key + "count"][0])
    assert it_v > 0 and abs(it_v - it_p) <= max(2, 0.02 * it_p), (it_v, it_p)


@pytest.mark.parametrize("method,cplx,s", FLAT_CASES)
def test_flat_plans_equal_generic_updates(flat_dumps, method, cplx, s):
    """eGl-BiCG's two block updates as lean flat kernels that carry r̂ and p̂ (egl_flat.cu) and
    Gl-BiCGStab's three updates, Gl-BiCG's (X, R, R̂) update and Gl-QMR's (Ṽ, W̃) update as flat plans (flat_upd.cu: the FMA order of the
    generic upd_kernel per element, another summation order in the fused reductions) against the
    generic kernels (SRK_NO_FLAT_UPDATE=1, a subprocess: the switch is read once): X_k and R_k
    after 12 iterations within 1e-11 (well-conditioned operator, see the QMR test above),
    stepped and graph-replayed runs bitwise equal, full solves converged with counts
    within 2. Width 12 complex is config 4's; 5 / 6 / 3 give ragged last CTAs, rows of 3 units
    and (eGl-BiCG at odd real width) the generic fallback."""
    key = f"{method}_{int(cplx)}_{s}_"
    ref = flat_dumps["plain"][key + "step"]
    flat = flat_dumps["flat"][key + "step"]
    assert np.isfinite(ref).all()
    assert np.array_equal(flat, flat_dumps["flat"][key + "graph"])
    for j in range(2):
        assert rel(flat[j], ref[j]) <= 1e-11, (j, rel(flat[j], ref[j]))
    it_f, it_p = int(flat_dumps["flat"][key + "count"][0]), int(flat_dumps["plain"][key + "count"][0])
    assert it_f > 0 and it_p > 0 and abs(it_f - it_p) <= max(2, 0.02 * it_p), (it_f, it_p)
