"""The banded-operator SpMM (band.cu, the SELL-C-σ slot for the
stencils): a0 detects <= 8 diagonals and the product runs on bulk-copied P windows. Parity
with the oracle's product (scipy CSR, to summation-order rounding) for every supported
width, real and complex, A and A^H, ragged and tiny n, boundary rows, every fused
non-FULL reduction; the config-3 operator at full size on sampled rows."""
import numpy as np
import pytest
import scipy.sparse as sp

import synth
from tests.gpu_util import rel, to_dev, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def srk():
    import paper_1504_04395_b200 as srk
    srk.load_library()
    return srk


def _ops():
    return {
        "2d": synth.conv_diff_2d(37, (20.0, 10.0)),                                   # 5 diagonals, ragged n
        "3d": synth.conv_diff_3d(21, (50.0, 30.0, 10.0)),                             # 7, far +-441
        "3dc": synth.conv_diff_3d(19, (50.0, 30.0, 10.0), np.complex128, -0.1j),      # complex
        "tiny": synth.conv_diff_2d(5),                                                # n = 25 < one tile
        "3dbig": synth.conv_diff_3d(70, (50.0, 30.0, 10.0)),                          # +-4900: far windows
    }


@pytest.mark.parametrize("name", ["2d", "3d", "3dc", "tiny", "3dbig"])
def test_band_detected(srk, name):
    A = _ops()[name]
    M = srk.Matrix.from_csr(A)
    fmt, nd = M.format()
    assert fmt == "band" and nd == (5 if name in ("2d", "tiny") else 7)
    assert M.format(adjoint=True)[0] == "band"


@pytest.mark.parametrize("adj", [False, True])
@pytest.mark.parametrize("name", ["2d", "3d", "3dc", "tiny", "3dbig"])
def test_band_spmm_matches_oracle_product(srk, name, adj):
    A = _ops()[name]
    cplx = A.dtype == np.complex128
    As = A.to_scipy()
    op = As.conj().T.tocsr() if adj else As
    M = srk.Matrix.from_csr(A)
    for s in ((1, 4, 8) if cplx else (1, 2, 4, 8, 16)):  # (real s = 1: band_vec_kernel, the economic variants' A^H p̂)
        P = synth.random_rhs(A.n, s, s + 3, cplx)
        Q = to_np(srk.spmm_block(M, to_dev(P), adjoint=adj))
        ref = op @ P
        assert rel(Q, ref) <= 1e-14, (name, adj, s, rel(Q, ref))


_RED_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import synth, paper_1504_04395_b200 as srk
from tests.gpu_util import rel, to_dev, to_np
srk.load_library()
for name, A in (("3d", synth.conv_diff_3d(21, (50.0, 30.0, 10.0))),
                ("3dc", synth.conv_diff_3d(19, (50.0, 30.0, 10.0), np.complex128, -0.1j))):
    cplx = A.dtype == np.complex128
    As = A.to_scipy()
    M = srk.Matrix.from_csr(A)
    s = 8 if cplx else 16
    for gram in ("norm2", "colnorm2", "diag", "trace", "sumvec"):
        P = synth.random_rhs(A.n, s, 1, cplx)
        Y = synth.random_rhs(A.n, 1 if gram == "sumvec" else s, 2, cplx)
        Yd = to_dev(Y[:, 0].copy() if gram == "sumvec" else Y)
        Q, g = srk.spmm_block(M, to_dev(P), gram=gram, Y=Yd)
        Q, g = to_np(Q), to_np(g)
        R = As @ P
        ref = {{"norm2": lambda: [np.vdot(R, R).real], "colnorm2": lambda: np.sum(np.abs(R) ** 2, axis=0),
               "diag": lambda: np.sum(Y.conj() * R, axis=0), "trace": lambda: [np.vdot(Y, R)],
               "sumvec": lambda: [np.sum(Y[:, 0].conj()[:, None] * R)]}}[gram]()
        assert rel(Q, R) <= 1e-14, (name, gram)
        assert rel(g, np.asarray(ref)) <= 1e-13, (name, gram, g, ref)
print("BAND_RED_OK")
"""


def test_band_fused_reductions():
    """Every fused non-FULL reduction in the banded kernel's epilogue, with the Y operand
    staged by the copy engine (SRK_BAND_ALL routes Y-operand products to the banded kernel;
    by default they keep the CSR kernel — equal speed measured), real and complex."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _RED_SCRIPT.format(root=root)], env={**os.environ, "SRK_BAND_ALL": "1"},
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert "BAND_RED_OK" in out.stdout, out.stderr[-2000:]


def test_band_full_size_config3_sampled(srk):
    """Config 3's operator (256^3, s = 16) in the banded form, the launch bench.py times
    (with the eGl vector-sum epilogue), on 4096 sampled rows plus the boundary planes."""
    import torch
    A = synth.make_config(3)[0]
    M = srk.Matrix.from_csr(A, need_adjoint=False)
    assert M.format() == ("band", 7)
    n, s = A.n, 16
    g = torch.Generator(device="cuda").manual_seed(5)
    P = torch.randn((n, s), dtype=torch.float64, device="cuda", generator=g)
    y = torch.randn((n,), dtype=torch.float64, device="cuda", generator=g)
    Q, sv = srk.spmm_block(M, P, gram="sumvec", Y=y)
    Q0 = srk.spmm_block(M, P)  # no epilogue operand: the banded kernel
    assert torch.equal(Q0, Q) or rel(Q0.cpu().numpy(), Q.cpu().numpy()) <= 1e-15
    rows = np.unique(np.concatenate([np.random.default_rng(0).integers(0, n, 4096),
                                     np.arange(0, 70000), np.arange(n - 70000, n)]))
    As = A.to_scipy()[rows]
    ref = As @ P.cpu().numpy()
    assert rel(Q[torch.from_numpy(rows).cuda()].cpu().numpy(), ref) <= 1e-14
    full = (y.double() @ Q).sum().item()
    assert abs(sv.item() - full) <= 1e-10 * abs(full) + 1e-6


def test_band_equals_csr_kernel_solver(srk):
    """A full eGl-QMR solve on the banded operator reproduces the oracle (lock-step over 20
    iterations at s = 16) — the solver path the bench times (see test_gpu_benchpath)."""
    import oracle
    A = synth.conv_diff_3d(30, (50.0, 30.0, 10.0))
    B = synth.random_rhs(A.n, 16, 2)
    M = srk.Matrix.from_csr(A)
    assert M.format()[0] == "band"
    a = oracle.solve("egl_qmr", A.to_scipy(), B, tol=1e-8, maxit=2000, record=20)
    sv = srk.Solver(M, 16, "egl_qmr", poll_every=1)
    sv.start(to_dev(B))
    for k in range(20):
        sv.iterate(1)
        assert rel(to_np(sv.x()), a.Xs[k]) <= 1e-10, k
    sv.close()


# ---------------------------------------------------------------- plane-marching kernel
def _seven_point(m, ny, nplanes_extra, seed, cplx=False):
    """A random matrix on exactly the diagonals {-F, -m, -1, 0, 1, m, F}, F = m ny, with
    n = F * nz + a ragged tail (n not a multiple of F) and nonzero values where a grid
    stencil would have none (row-index semantics across line / plane ends)."""
    F = m * ny
    n = F * nplanes_extra[0] + nplanes_extra[1]
    rng = np.random.default_rng(seed)
    offs = [-F, -m, -1, 0, 1, m, F]
    diags = []
    for d in offs:
        L = n - abs(d)
        v = rng.standard_normal(L)
        if cplx:
            v = v + 1j * rng.standard_normal(L)
        diags.append(v)
    A = sp.diags(diags, offs, shape=(n, n), format="csr", dtype=np.complex128 if cplx else np.float64)
    A.sort_indices()
    return A


def _plane_ops():
    return {
        "even": _seven_point(34, 10, (5, 17), 1),            # ragged x (34 = 32 + 2) and y (10 = 6 + 4) tiles, tail plane
        "odd": _seven_point(21, 7, (6, 0), 2),               # odd m: shifted value / vector copies
        "cplx": _seven_point(18, 13, (4, 101), 3, True),     # complex, m < tile width
        "cube": synth.conv_diff_3d(40, (50.0, 30.0, 10.0)),  # a grid stencil (zero values at the edges)
    }


@pytest.mark.parametrize("adj", [False, True])
@pytest.mark.parametrize("name", ["even", "odd", "cplx", "cube"])
def test_plane_spmm_matches_oracle_product(srk, name, adj):
    """The 7-point plane-marching kernel against the CSR product for every supported width,
    A and A^H, with the fused norm / column-norm / vector-sum epilogues."""
    A = _plane_ops()[name]
    As = A.to_scipy() if hasattr(A, "to_scipy") else A
    cplx = As.dtype == np.complex128
    op = As.conj().T.tocsr() if adj else As
    M = srk.Matrix.from_csr(A)
    assert M.format(adjoint=adj) == ("band", 7)
    n = As.shape[0]
    for s in ((1, 4, 8) if cplx else (2, 4, 8, 16)):
        P = synth.random_rhs(n, s, s + 3, cplx)
        R = op @ P
        Q = to_np(srk.spmm_block(M, to_dev(P), adjoint=adj))
        assert rel(Q, R) <= 1e-14, (name, adj, s, rel(Q, R))
        y = synth.random_rhs(n, 1, s + 7, cplx)[:, 0].copy()
        for gram, ref, mag in (("norm2", [np.vdot(R, R).real], np.vdot(R, R).real),
                               ("colnorm2", np.sum(np.abs(R) ** 2, axis=0), np.sum(np.abs(R) ** 2, axis=0)),
                               ("sumvec", [np.sum(y.conj()[:, None] * R)], np.sum(np.abs(y)[:, None] * np.abs(R)))):
            Q2, gv = srk.spmm_block(M, to_dev(P), adjoint=adj, gram=gram, Y=to_dev(y) if gram == "sumvec" else None)
            assert rel(to_np(Q2), R) <= 1e-14, (name, gram)
            # summation-order rounding: bounded by the sum of the terms' magnitudes (the vector
            # sum cancels, so a bound relative to the result alone would be order dependent)
            assert np.all(np.abs(to_np(gv).ravel() - np.asarray(ref).ravel()) <= 1e-13 * np.asarray(mag).ravel()), \
                (name, adj, s, gram)
        # row operands (Gl-BiCGStab's <A P, R~> and <A S, S>, Li's per-column forms): an external block
        # (rows requested ahead of each plane step) and the product's own input (rows already in registers)
        Yb = synth.random_rhs(n, s, s + 11, cplx)
        Pd = to_dev(P)
        for gram in ("trace", "diag"):
            for Yh, Yd in ((Yb, to_dev(Yb)), (P, Pd)):
                prod = Yh.conj() * R
                ref = [prod.sum()] if gram == "trace" else prod.sum(axis=0)
                mag = [np.abs(prod).sum()] if gram == "trace" else np.abs(prod).sum(axis=0)
                Q2, gv = srk.spmm_block(M, Pd, adjoint=adj, gram=gram, Y=Yd)
                assert rel(to_np(Q2), R) <= 1e-14, (name, gram)
                assert np.all(np.abs(to_np(gv).ravel() - np.asarray(ref).ravel()) <= 1e-13 * np.asarray(mag).ravel()), \
                    (name, adj, s, gram, Yh is P)


_PLANE_VS_RING = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import synth, paper_1504_04395_b200 as srk
from tests.gpu_util import to_dev, to_np
from tests.test_gpu_band import _plane_ops
srk.load_library()
out = {{}}
for name, A in _plane_ops().items():
    M = srk.Matrix.from_csr(A)
    n = M.n
    cplx = name == "cplx"
    for s in ((1, 4, 8) if cplx else (2, 4, 8, 16)):
        P = synth.random_rhs(n, s, s + 3, cplx)
        for adj in (False, True):
            out[f"{{name}}_{{s}}_{{int(adj)}}"] = to_np(srk.spmm_block(M, to_dev(P), adjoint=adj))
np.savez({path!r}, **out)
print("PLANE_DUMP_OK")
"""


def test_plane_kernel_bitwise_equals_ring_kernel(tmp_path):
    """Same summation order (ascending offset, FMA chain from zero) as the ring / far-window
    band kernel: the two products are bitwise equal (SRK_BAND_PLANE=0 selects the ring one)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("1", "0"):
        path = str(tmp_path / f"q{flag}.npz")
        out = subprocess.run([sys.executable, "-c", _PLANE_VS_RING.format(root=root, path=path)],
                             env={**os.environ, "SRK_BAND_PLANE": flag}, capture_output=True, text=True,
                             timeout=600, cwd=root)
        assert "PLANE_DUMP_OK" in out.stdout, out.stderr[-2000:]
        res[flag] = dict(np.load(path))
    assert res["1"].keys() == res["0"].keys()
    for k in res["1"]:
        assert np.array_equal(res["1"][k], res["0"][k]), k


def test_band_vector_product_with_reduction_falls_back(srk):
    """The banded vector kernel takes no fused reduction: a product with one runs on the CSR kernel
    and still matches the oracle's product and norm."""
    A = synth.conv_diff_3d(21, (50.0, 30.0, 10.0))
    M = srk.Matrix.from_csr(A)
    p = synth.random_rhs(A.n, 1, 5)
    Q, g = srk.spmm_block(M, to_dev(p), gram="norm2")
    ref = A.to_scipy() @ p
    assert rel(to_np(Q), ref) <= 1e-14 and abs(to_np(g)[0] - np.vdot(ref, ref).real) <= 1e-12 * np.vdot(ref, ref).real
