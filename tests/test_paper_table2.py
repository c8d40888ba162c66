"""The paper's Table 2 (block methods, Ex. 1-3 at the paper's sizes and protocol;
fixture tests/golden/table2_block.txt) against the GPU path (fast, -m gpu), the oracle
against the paper (slow; opt-in with SRK_SLOW=1: ~6 minutes of numpy), and the GPU
against the oracle on the converged entries (-m gpu, not opt-in).

Agreement asserted: converged vs not converged within 500 iterations for every entry,
and the iteration count within 10% where the paper's method converged. One entry
differs and is marked: Ex. 3's plain Bl-BiCGStab converges in 111 iterations in the
paper, which used the Bl-BiCGStab of its reference [Jbilou05]; the App. A.4 form built
here (after [ELg03]) stagnates, while its QR-stabilised form —
mathematically the same iterates — converges in 98 (paper: 101). DESIGN.md §3."""
import os

import numpy as np
import pytest

import synth

HERE = os.path.dirname(__file__)


def _table(fname="table2_block.txt"):
    rows = []
    with open(os.path.join(HERE, "golden", fname)) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                ex, method, it, res = line.split()
                rows.append((ex, method, int(it), None if res == "div" else float(res)))
    return rows


def _problem(ex):
    A, B = synth.paper_ex1(200) if ex == "ex1" else synth.paper_ex2(50, 1000.0 if ex == "ex2" else 10.0)
    Q, _ = np.linalg.qr(B)
    return A, np.ascontiguousarray(Q)


def _paper_converged(it, res):
    return it < 500 and res is not None and res <= 1e-9


KNOWN = {("ex3", "bl_bicgstab")}
# the unstabilised block methods are rounding-sensitive where they barely converge in the
# paper; their QR-stabilised forms (the same iterates in exact arithmetic) match it
KNOWN_ILU = {
    # CUDA-core updates: stagnated at 2.1e-10 against the 1e-10 tolerance; tensor-core
    # updates: converges in 117 (paper: 113)
    ("ex1", "bl_bicgstab"): "stagnates near the tolerance depending on rounding (paper: 113 its)",
    ("ex2", "bl_bicg"): "singular s x s Gram (G12 breakdown test) at iteration 30, true residual 1.7e-6, with the "
                        "tensor-core updates (27 iterations, converged, with the CUDA-core ones; paper: 28)",
    ("ex3", "bl_bicg"): "singular s x s Gram (G12 breakdown test) at iteration 46-48 (paper: converged in 50)",
}


# Ex. 1's Bl-BiCGStab-rQ converges only after a long plateau, and where it leaves the
# plateau depends on rounding: the oracle takes 394 iterations on Q, 349 and 352 on Q with
# its columns reversed / pair-swapped (the same iterates in exact arithmetic), the GPU
# 356 (CUDA-core updates) or 428 (tensor-core updates); the paper 355. Only "converged
# within 500" is asserted for it. Ex. 3's Bl-BiCGStab-rQ is sensitive too, less so: 97
# iterations on Q, but with Q's columns reversed the oracle stalls at 1.7e-10 (500
# iterations); the GPU takes 95-98 (paper 101). Counts elsewhere: within 10%.
ROUNDING_SENSITIVE = {("ex1", "bl_bicgstab_rq")}


def _check(ex, method, it, res, outcome, iters):
    conv = outcome == "converged"
    if (ex, method) in KNOWN:
        pytest.xfail("Ex. 3 plain Bl-BiCGStab: [Jbilou05]'s variant in the paper vs App. A.4 here (DESIGN.md §3)")
    assert conv == _paper_converged(it, res), (ex, method, outcome, iters, it, res)
    if conv and (ex, method) not in ROUNDING_SENSITIVE:
        assert abs(iters - it) <= 0.10 * it, (ex, method, iters, it)


def test_golden_fixture_shape():
    for fname in ("table2_block.txt", "table2_block_ilu.txt"):
        rows = _table(fname)
        assert len(rows) == 12 and {r[0] for r in rows} == {"ex1", "ex2", "ex3"}


@pytest.mark.gpu
@pytest.mark.parametrize("row", _table(), ids=lambda r: f"{r[0]}-{r[1]}")
def test_table2_gpu(row):
    import torch

    import paper_1504_04395_b200 as srk
    srk.load_library()
    ex, method, it, res = row
    A, Q = _problem(ex)
    M = srk.Matrix.from_csr(A, need_adjoint=True)
    X, rep = srk.solve(M, torch.from_numpy(Q).cuda(), method, tol=1e-10, maxit=500)
    _check(ex, method, it, res, rep.outcome, rep.iterations)


@pytest.mark.gpu
@pytest.mark.parametrize("row", _table("table2_block_ilu.txt"), ids=lambda r: f"{r[0]}-{r[1]}")
def test_table2_ilu_gpu(row):
    """The lower half of Table 2: right ILU(0) (srk_matrix_ilu0). Converged vs not, and
    the count within 10% (the factorisation, not only the summation order, now
    differs from Matlab's in rounding)."""
    import torch

    import paper_1504_04395_b200 as srk
    srk.load_library()
    ex, method, it, res = row
    A, Q = _problem(ex)
    M = srk.Matrix.from_csr(A, need_adjoint=True).ilu0()
    X, rep = srk.solve(M, torch.from_numpy(Q).cuda(), method, tol=1e-10, maxit=500)
    conv = rep.outcome == "converged"
    ok = conv == _paper_converged(it, res) and (not conv or abs(rep.iterations - it) <= max(2, 0.10 * it))
    if not ok and (ex, method) in KNOWN_ILU:  # the rounding-sensitive entries: run, xfail if they miss
        pytest.xfail(KNOWN_ILU[(ex, method)])
    assert ok, (ex, method, rep.outcome, rep.iterations, it, res)


@pytest.mark.slow
@pytest.mark.parametrize("row", [r for r in _table() if _paper_converged(r[2], r[3])], ids=lambda r: f"{r[0]}-{r[1]}")
def test_table2_oracle(row):
    if os.environ.get("SRK_SLOW") != "1":
        pytest.skip("slow (numpy at the paper's sizes): set SRK_SLOW=1")
    import oracle
    ex, method, it, res = row
    A, Q = _problem(ex)
    r = oracle.solve(method, A.to_scipy(), Q, tol=1e-10, maxit=500, record=0)
    _check(ex, method, it, res, r.outcome, r.iterations)


@pytest.mark.gpu
@pytest.mark.parametrize("row", [r for r in _table() if _paper_converged(r[2], r[3]) and (r[0], r[1]) not in KNOWN
                                 and (r[0], r[1]) not in ROUNDING_SENSITIVE], ids=lambda r: f"{r[0]}-{r[1]}")
def test_table2_gpu_vs_oracle(row):
    """The GPU against the oracle on the paper's grid (not opt-in): for every entry the paper
    reports converged (and that is not marked rounding-sensitive above), the same outcome and
    the count within max(2%, 2) — or, where the oracle itself moves with the reduction
    order, within the oracle's spread + 2 (SURVEY §8c.5 rule 3) — and the oracle's SpMM
    recomputes the GPU's true residual."""
    import torch

    import oracle
    import paper_1504_04395_b200 as srk
    srk.load_library()
    ex, method, it, res = row
    A, Q = _problem(ex)
    As = A.to_scipy()
    a = oracle.solve(method, As, Q, tol=1e-10, maxit=500, record=0)
    M = srk.Matrix.from_csr(A, need_adjoint=True)
    X, rep = srk.solve(M, torch.from_numpy(Q).cuda(), method, tol=1e-10, maxit=500)
    assert rep.outcome == a.outcome, (rep.outcome, a.outcome)
    slack = max(2, 0.02 * a.iterations)
    alts = []
    if abs(rep.iterations - a.iterations) > slack:  # the oracle's own spread over its orders (R10)
        alts = [oracle.solve(method, As, Q, tol=1e-10, maxit=500, record=0, order=o) for o in ("seq", "rev", "cholqr")]
        alts = [b.iterations for b in alts if b.outcome == a.outcome]
        if alts:
            slack = max(slack, max(abs(a.iterations - b) for b in alts) + 2)
    assert abs(rep.iterations - a.iterations) <= slack, (rep.iterations, a.iterations, alts)
    Xh = X.cpu().numpy()
    assert np.linalg.norm(Q - As @ Xh) / np.linalg.norm(Q) <= 1e-10
