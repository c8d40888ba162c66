"""GPU parity of the kernel-level C-ABI calls (srk_spmm_block, srk_gram_block,
srk_block_update, srk_tsqr, the A^H build) against the oracle (oracle/linalg.py
and scipy products), element by element, on seeded inputs spanning several
CTAs and a ragged tail, plus empty rows."""
import numpy as np
import pytest

import oracle.linalg as OL
import synth
from tests.gpu_util import csr_with_empty_rows, rel, to_dev, to_np

pytestmark = pytest.mark.gpu

S_LIST = [1, 2, 3, 4, 8, 12, 16, 19, 32, 64]


@pytest.fixture(scope="module")
def srk():
    import paper_1504_04395_b200 as srk
    srk.load_library()
    return srk


def _rand(rng, n, s, cplx):
    X = rng.standard_normal((n, s))
    if cplx:
        X = X + 1j * rng.standard_normal((n, s))
    return X


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("s", S_LIST)
def test_spmm_matches_scipy(srk, s, cplx):
    A = csr_with_empty_rows(5003, seed=s, cplx=cplx)
    M = srk.Matrix.from_csr(A)
    rng = np.random.default_rng(s)
    P = _rand(rng, A.shape[0], s, cplx)
    Q = to_np(srk.spmm_block(M, to_dev(P)))
    ref = A @ P
    # summation order of one row differs at most by nnz_row * eps
    assert np.max(np.abs(Q - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)))
    QH = to_np(srk.spmm_block(M, to_dev(P), adjoint=True))
    refH = A.conj().T @ P
    assert np.max(np.abs(QH - refH)) <= 1e-13 * max(1.0, np.max(np.abs(refH)))


@pytest.mark.parametrize("cplx", [False, True])
def test_adjoint_is_conj_transpose(srk, cplx):
    A = csr_with_empty_rows(2001, seed=5, cplx=cplx)
    M = srk.Matrix.from_csr(A)
    rp, ci, va = (to_np(t) for t in M.adjoint_csr())
    AH = A.conj().T.tocsr()
    AH.sort_indices()
    assert np.array_equal(rp, AH.indptr) and np.array_equal(ci, AH.indices)
    assert np.array_equal(va, AH.data)  # a pure permutation + conjugation: bit-exact


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("s", [1, 3, 4, 8, 12, 16])
@pytest.mark.parametrize("mode", ["norm2", "colnorm2", "diag", "trace", "sumvec", "full"])
def test_spmm_fused_reductions(srk, s, cplx, mode):
    A = synth.random_sparse(3001, 6, seed=2, dtype=np.complex128 if cplx else np.float64).to_scipy()
    M = srk.Matrix.from_csr(A)
    rng = np.random.default_rng(7)
    P = _rand(rng, A.shape[0], s, cplx)
    Y = _rand(rng, A.shape[0], s, cplx)
    y = Y[:, 0].copy()
    Yd = to_dev(y) if mode == "sumvec" else to_dev(Y)
    Q, g = srk.spmm_block(M, to_dev(P), gram=mode, Y=Yd)
    Q = to_np(Q)
    g = to_np(g)
    ref = {
        "norm2": lambda: np.array([OL.fro2(Q)]),
        "colnorm2": lambda: np.real(OL.col_inner(Q, Q)),
        "diag": lambda: OL.col_inner(Q, Y),
        "trace": lambda: np.array([OL.trace_inner(Q, Y)]),
        "sumvec": lambda: np.array([OL.sum_inner(y, Q)]),
        "full": lambda: OL.gram(Y, Q),
    }[mode]()
    assert rel(g.reshape(ref.shape), ref) < 1e-12


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("s", [1, 2, 5, 8, 16, 17, 24, 32, 33, 48, 64])
def test_gram_block(srk, s, cplx):
    """FULL Y^H X and the trace; s > 16 runs on the FP64 tensor cores (DMMA)."""
    rng = np.random.default_rng(11)
    n = 10007
    X, Y = _rand(rng, n, s, cplx), _rand(rng, n, s, cplx)
    g = to_np(srk.gram_block(to_dev(X), to_dev(Y), "full"))
    assert rel(g, OL.gram(Y, X)) < 1e-12
    t = to_np(srk.gram_block(to_dev(X), to_dev(Y), "trace"))
    assert abs(t[0] - OL.trace_inner(X, Y)) <= 1e-12 * abs(OL.trace_inner(X, Y))


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("s", [1, 4, 7, 12, 16, 19, 32])
@pytest.mark.parametrize("kind", ["scalar", "diag", "full"])
def test_block_update(srk, s, cplx, kind):
    rng = np.random.default_rng(13)
    n = 4099
    Y, X = _rand(rng, n, s, cplx), _rand(rng, n, s, cplx)
    coef = {"scalar": _rand(rng, 1, 1, cplx)[0], "diag": _rand(rng, 1, s, cplx)[0], "full": _rand(rng, s, s, cplx)}[kind]
    out = to_np(srk.block_update(to_dev(Y), to_dev(X), to_dev(coef), kind, sign=-1))
    ref = Y - (X @ coef if kind == "full" else X * coef)
    assert np.max(np.abs(out - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("s", [1, 3, 8, 16, 19, 32])
def test_tsqr_matches_oracle(srk, s, cplx):
    rng = np.random.default_rng(17)
    Z = _rand(rng, 20011, s, cplx)
    Q, C, rank = srk.tsqr(to_dev(Z))
    Q, C = to_np(Q), to_np(C)
    Qo, Co = OL.thin_qr(Z)
    assert rank == s
    assert rel(C, Co) < 1e-12 and rel(Q, Qo) < 1e-12
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(s)) < 1e-12


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("s", [8, 12, 16, 17, 32, 64])
def test_gram_mma_edge_rows(srk, s, cplx):
    """DMMA Gram on row counts around the 16-row warp stage and the 32-row chunk (1, 15,
    16, 17, 31, 32, 33 rows, fewer stages than warps, a ragged multi-stage tail), with
    distinct operands and with X == Y (one staged copy serves both), against the
    oracle's Gram."""
    rng = np.random.default_rng(23)
    for n in (1, 15, 16, 17, 31, 32, 33, 4 * 32 * 148 + 5, 100003):
        X, Y = _rand(rng, n, s, cplx), _rand(rng, n, s, cplx)
        g = to_np(srk.gram_block(to_dev(X), to_dev(Y), "full"))
        assert rel(g, OL.gram(Y, X)) < 1e-12, n
        Xd = to_dev(X)
        g = to_np(srk.gram_block(Xd, Xd, "full"))
        assert rel(g, OL.gram(X, X)) < 1e-12, ("same", n)


def test_tsqr_rank_deficient(srk):
    rng = np.random.default_rng(19)
    w = rng.standard_normal((3000, 1))
    _, _, rank = srk.tsqr(to_dev(np.hstack([w, 2 * w, rng.standard_normal((3000, 1))])))
    assert rank < 3


def test_invalid_csr_rejected(srk):
    import torch
    rp = torch.tensor([0, 2, 3], dtype=torch.int64)
    ci = torch.tensor([1, 0, 1], dtype=torch.int32)  # row 0 unsorted
    va = torch.ones(3, dtype=torch.float64)
    with pytest.raises(srk.SrkError):
        srk.Matrix(rp, ci, va)
    with pytest.raises(srk.SrkError):
        srk.Matrix(rp, torch.tensor([0, 5, 1], dtype=torch.int32), va)  # column out of range


def test_limits_and_unsupported_combinations(srk):
    """The documented error paths (include/srk.h): nnz >= 2^31 (int32 indices) is
    refused before any allocation; s outside [1, 64]; block methods beyond s = 32;
    BSR widths outside {4, 8, 12, 16}; methods needing A^H on an operator without it."""
    import ctypes

    import torch
    ctx = srk.default_context()
    csr = srk._Csr(1 << 20, 1 << 31, 1, 1, 1, 0)  # header only: never dereferenced
    h = ctypes.c_void_p()
    assert srk._lib.srk_matrix_create(ctx.h, ctypes.byref(csr), 0, ctypes.byref(h)) == -3  # SRK_EUNSUPPORTED
    A = synth.conv_diff_2d(10)
    M = srk.Matrix.from_csr(A, need_adjoint=False)
    P = to_dev(synth.random_rhs(A.n, 65, 1))
    with pytest.raises(srk.SrkError):
        srk.spmm_block(M, P)
    with pytest.raises(srk.SrkError):  # Gl-BiCG needs A^H
        srk.Solver(M, 4, "gl_bicg")
    M2 = srk.Matrix.from_csr(A, need_adjoint=True)
    with pytest.raises(srk.SrkError):  # block methods: s <= 32
        srk.Solver(M2, 33, "bl_bicg")
    srk.Solver(M2, 32, "bl_bicg").close()
    brp, bcol, blocks = synth.lattice_4d_bsr(3)
    Mb = srk.Matrix.from_bsr(brp, bcol, blocks, unit_diag=True)
    with pytest.raises(srk.SrkError):  # BSR widths
        srk.Solver(Mb, 6, "gl_bicgstab")
    with pytest.raises(srk.SrkError):  # no A^H for BSR operators
        srk.Solver(Mb, 4, "gl_bicg")
    del torch


def test_full_size_config3_spmm_sampled(srk):
    """Config 3 at full size (n = 256^3, s = 16) in the bench launch configuration:
    sampled rows of A P against the oracle, and the fused trace against numpy."""
    import torch
    A, B = synth.make_config(3)
    M = srk.Matrix.from_csr(A, need_adjoint=False)
    Bd = to_dev(B)
    Rt = to_dev(synth.random_rhs(A.n, 16, 99))
    Q, tr = srk.spmm_block(M, Bd, gram="trace", Y=Rt)
    rows = np.random.default_rng(0).choice(A.n, 4096, replace=False)
    rows.sort()
    As = A.to_scipy()
    ref = As[rows] @ B
    Qs = to_np(Q[torch.from_numpy(rows).cuda()])
    assert np.max(np.abs(Qs - ref)) <= 1e-13 * np.max(np.abs(ref))
    Rtn = to_np(Rt)
    full = As @ B
    t_ref = np.vdot(Rtn.ravel(), full.ravel())
    assert abs(to_np(tr)[0] - t_ref) <= 1e-11 * np.linalg.norm(full) * np.linalg.norm(Rtn)


@pytest.mark.parametrize("s", [1, 2, 4, 8, 16, 32, 64])
def test_config5_spmm_gram_sweep(srk, s):
    """Config 5's SpMM+Gram sweep (power-law rows up to 512, uniform columns) at
    n = 2^16: the product and the reductions (trace, sum, norms and the full s x s
    Gram at every s) against the oracle."""
    A = synth.power_law(1 << 16, seed=4)
    As = A.to_scipy()
    M = srk.Matrix.from_csr(A, need_adjoint=False)
    P = synth.random_rhs(A.n, s, 4)
    Y = synth.random_rhs(A.n, s, 5)
    modes = ["trace", "norm2", "sumvec", "full"]  # FULL: fused for s <= 16, DMMA Gram after the SpMM above
    ref = As @ P
    for mode in modes:
        Yd = to_dev(Y[:, 0].copy()) if mode == "sumvec" else to_dev(Y)
        Q, g = srk.spmm_block(M, to_dev(P), gram=mode, Y=Yd)
        Q, g = to_np(Q), to_np(g)
        assert np.max(np.abs(Q - ref)) <= 1e-12 * np.max(np.abs(ref))
        expect = {"trace": lambda: np.array([OL.trace_inner(ref, Y)]), "norm2": lambda: np.array([OL.fro2(ref)]),
                  "sumvec": lambda: np.array([OL.sum_inner(Y[:, 0], ref)]), "full": lambda: OL.gram(Y, ref)}[mode]()
        assert rel(g.reshape(expect.shape), expect) < 1e-11, mode


def test_full_size_config5_sampled(srk):
    """Config 5 at full size (n = 2^22, ~67M nnz, s = 32) in the launch configuration
    of its sweep: 4096 sampled rows of A P against the oracle's products, and the
    fused sum(y^H Q) against numpy."""
    import torch
    A = synth.power_law(1 << 22, seed=4)
    M = srk.Matrix.from_csr(A, need_adjoint=False)
    B = synth.random_rhs(A.n, 32, 4)
    y = synth.random_rhs(A.n, 1, 6)[:, 0].copy()
    Q, sv = srk.spmm_block(M, to_dev(B), gram="sumvec", Y=to_dev(y))
    rows = np.sort(np.random.default_rng(1).choice(A.n, 4096, replace=False))
    As = A.to_scipy()
    ref = As[rows] @ B
    Qs = to_np(Q[torch.from_numpy(rows).cuda()])
    assert np.max(np.abs(Qs - ref)) <= 1e-12 * np.max(np.abs(ref))
    full = As @ B
    assert abs(to_np(sv)[0] - OL.sum_inner(y, full)) <= 1e-11 * np.linalg.norm(full) * np.linalg.norm(y) * np.sqrt(32)


def test_full_size_config2_sampled(srk):
    """Config 2 at full size (128^3 complex, s = 8): sampled rows of A P, of A^H P,
    and the fused s x s Gram P^H (A P) against numpy."""
    import torch
    A, B = synth.make_config(2)
    M = srk.Matrix.from_csr(A, need_adjoint=True)
    Bd = to_dev(B)
    Q, G = srk.spmm_block(M, Bd, gram="full", Y=Bd)
    QH = srk.spmm_block(M, Bd, adjoint=True)
    rows = np.sort(np.random.default_rng(2).choice(A.n, 4096, replace=False))
    As = A.to_scipy()
    sel = torch.from_numpy(rows).cuda()
    assert np.max(np.abs(to_np(Q[sel]) - As[rows] @ B)) <= 1e-12 * np.max(np.abs(B)) * 8
    AH = As.conj().T.tocsr()
    assert np.max(np.abs(to_np(QH[sel]) - AH[rows] @ B)) <= 1e-12 * np.max(np.abs(B)) * 8
    full = As @ B
    assert rel(to_np(G), OL.gram(B, full)) < 1e-11


def test_mid_size_config4_lattice_sampled(srk):
    """Config 4's operator at 16^4 sites (n = 786,432, 76M nnz, complex, s = 12):
    sampled rows of A P against the oracle's product."""
    import torch
    A, B = synth.make_config(4, m=16)
    M = srk.Matrix.from_csr(A, need_adjoint=False)
    Q = srk.spmm_block(M, to_dev(B))
    rows = np.sort(np.random.default_rng(3).choice(A.n, 4096, replace=False))
    As = A.to_scipy()
    ref = As[rows] @ B
    assert np.max(np.abs(to_np(Q[torch.from_numpy(rows).cuda()]) - ref)) <= 1e-12 * np.max(np.abs(ref))


def _bsr_from_csr(As, bs=12):
    """Explicit block form (diagonal blocks stored) of a CSR via scipy."""
    Bs = As.tobsr(blocksize=(bs, bs))
    Bs.sort_indices()
    return Bs.indptr.astype(np.int64), Bs.indices.astype(np.int32), np.ascontiguousarray(Bs.data)


@pytest.mark.parametrize("s", [4, 8, 12, 16])
@pytest.mark.parametrize("unit", [True, False])
def test_bsr_spmm_matches_oracle(srk, s, unit):
    """BSR-12 SpMM on the FP64 tensor cores (config 4's lattice at 4^4 sites: 256
    block rows, 8 blocks each, a ragged last CTA) against the oracle's product,
    with the identity diagonal implied (unit_diag) or stored as explicit blocks."""
    A = synth.lattice_4d(4)
    As = A.to_scipy()
    if unit:
        brp, bcol, blocks = synth.lattice_4d_bsr(4)
    else:
        brp, bcol, blocks = _bsr_from_csr(As)
    M = srk.Matrix.from_bsr(brp, bcol, blocks, unit_diag=unit)
    P = synth.random_rhs(A.n, s, 7, True)
    Q = to_np(srk.spmm_block(M, to_dev(P)))
    ref = As @ P
    assert np.max(np.abs(Q - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("mode", ["norm2", "diag", "trace", "sumvec", "full"])
def test_bsr_spmm_reductions(srk, mode):
    A = synth.lattice_4d(4)
    brp, bcol, blocks = synth.lattice_4d_bsr(4)
    M = srk.Matrix.from_bsr(brp, bcol, blocks, unit_diag=True)
    P = synth.random_rhs(A.n, 12, 8, True)
    Y = synth.random_rhs(A.n, 12, 9, True)
    y = Y[:, 0].copy()
    Q, g = srk.spmm_block(M, to_dev(P), gram=mode, Y=to_dev(y) if mode == "sumvec" else to_dev(Y))
    Q, g = to_np(Q), to_np(g)
    ref = {"norm2": lambda: np.array([OL.fro2(Q)]), "diag": lambda: OL.col_inner(Q, Y),
           "trace": lambda: np.array([OL.trace_inner(Q, Y)]), "sumvec": lambda: np.array([OL.sum_inner(y, Q)]),
           "full": lambda: OL.gram(Y, Q)}[mode]()
    assert rel(g.reshape(ref.shape), ref) < 1e-12


@pytest.mark.parametrize("L,w", [(4, 2), (8, 2), (8, 4)])
def test_bsr_row_order_hint(srk, L, w):
    """srk_matrix_set_row_order: a visiting order of the block rows changes the schedule only —
    Q is bitwise the natural-order product (and matches the oracle), the fused trace equals the
    oracle's to rounding; a non-permutation and a wrong length are rejected; None restores."""
    brp, bcol, blocks = synth.lattice_4d_bsr(L)
    M = srk.Matrix.from_bsr(brp, bcol, blocks, unit_diag=True)
    n = L ** 4 * 12
    P = synth.random_rhs(n, 12, 7, True)
    Y = synth.random_rhs(n, 12, 9, True)
    Q0, t0 = srk.spmm_block(M, to_dev(P), gram="trace", Y=to_dev(Y))
    Q0, t0 = to_np(Q0), to_np(t0)
    order = synth.lattice_tile_order(L, w)
    assert np.array_equal(np.sort(order), np.arange(L ** 4))
    M.set_row_order(order)
    Q1, t1 = srk.spmm_block(M, to_dev(P), gram="trace", Y=to_dev(Y))
    Q1, t1 = to_np(Q1), to_np(t1)
    assert np.array_equal(Q1, Q0)
    ref = OL.trace_inner(Q0, Y)
    assert abs(t1[0] - ref) <= 1e-12 * abs(ref) and abs(t0[0] - ref) <= 1e-12 * abs(ref)
    if L == 4:
        As = synth.lattice_4d(4).to_scipy()
        assert np.max(np.abs(Q1 - As @ P)) <= 1e-13 * np.max(np.abs(Q1))
    bad = order.copy()
    bad[0] = bad[1]
    with pytest.raises(srk.SrkError):
        M.set_row_order(bad)
    with pytest.raises(srk.SrkError):
        M.set_row_order(order[:-1])
    M.set_row_order(None)
    assert np.array_equal(to_np(srk.spmm_block(M, to_dev(P))), Q0)
    with pytest.raises(srk.SrkError):  # block-sparse operators only
        srk.Matrix.from_csr(synth.conv_diff_2d(8, (20.0, 20.0))).set_row_order(np.arange(64))


def test_bsr_rejects_invalid(srk):
    brp, bcol, blocks = synth.lattice_4d_bsr(3)
    bad = bcol.copy()
    bad[0], bad[1] = bcol[1], bcol[0]  # unsorted block columns
    with pytest.raises(srk.SrkError):
        srk.Matrix.from_bsr(brp, bad, blocks, unit_diag=True)
    with pytest.raises(srk.SrkError):  # 12 x 12 blocks only
        srk.Matrix.from_bsr(brp, bcol, np.ascontiguousarray(blocks[:, :6, :6]), unit_diag=True)


def test_mid_size_config4_bsr_sampled(srk):
    """Config 4's operator at 16^4 sites in BSR form (65,536 block rows, s = 12):
    sampled rows of A P against the oracle's (scalar CSR) product."""
    import torch
    A, B = synth.make_config(4, m=16)
    brp, bcol, blocks = synth.lattice_4d_bsr(16)
    M = srk.Matrix.from_bsr(brp, bcol, blocks, unit_diag=True)
    Q = srk.spmm_block(M, to_dev(B))
    rows = np.sort(np.random.default_rng(3).choice(A.n, 4096, replace=False))
    ref = A.to_scipy()[rows] @ B
    assert np.max(np.abs(to_np(Q[torch.from_numpy(rows).cuda()]) - ref)) <= 1e-12 * np.max(np.abs(ref))
