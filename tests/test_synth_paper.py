"""Pins of the paper's Ex. 1-3 generators (synth.paper_ex1 / paper_ex2, PAPER.md
P:695-750) against exact discrete solutions: central differences are exact on
polynomials of degree <= 1 per coordinate, so boundary data taken from such a
function must give a right-hand side whose solution is that function on the grid."""
import numpy as np
import scipy.sparse.linalg as spla

import synth


def _grid2(m):
    h = 1.0 / (m + 1)
    idx = np.arange(m * m)
    return (idx % m + 1) * h, (idx // m + 1) * h


def test_ex1_corner_data_are_the_bilinear_hats():
    """Corner (cx, cy)'s boundary data is the restriction of the bilinear hat
    (1 - |x - cx|)(1 - |y - cy|), which the 5-point Laplacian (a = 0) reproduces
    exactly: A(0) @ hat = b_corner."""
    m = 17
    A, B = synth.paper_ex1(m, alpha=(0.0, 0.0, 0.0))
    x, y = _grid2(m)
    As = A.to_scipy()
    for k, (cx, cy) in enumerate(((0, 0), (1, 0), (0, 1), (1, 1))):
        hat = (1 - np.abs(x - cx)) * (1 - np.abs(y - cy))
        assert np.max(np.abs(As @ hat - B[:, k])) < 1e-13


def test_ex1_sizes_and_convection():
    """Paper size: 200^2 unknowns, s = 4 (Table 1); with a != 0 the four
    solutions still add up to the solution for boundary data 1 (superposition)."""
    A, B = synth.paper_ex1(200)
    assert A.n == 40000 and B.shape == (40000, 4)
    A, B = synth.paper_ex1(15)
    As = A.to_scipy()
    one = spla.spsolve(As.tocsc(), B.sum(axis=1))
    parts = sum(spla.spsolve(As.tocsc(), B[:, k]) for k in range(4))
    assert np.max(np.abs(one - parts)) < 1e-12
    assert 0.0 < one.min() and one.max() < 10  # a bounded, positive field (maximum principle-ish)


def _col(axis, side, which):
    return 1 + (axis * 2 + side) * 3 + which


def test_ex2_face_data_reproduce_affine_solutions():
    """u = 1, u = y and u = z solve u_xx + u_yy + u_zz + nu u_x = 0 exactly (also
    discretely): the matching combinations of the 18 face right-hand sides are
    A @ u."""
    m = 9
    for nu in (10.0, 1000.0):
        A, B = synth.paper_ex2(m, nu)
        assert B.shape == (m ** 3, 19)
        h = 1.0 / (m + 1)
        idx = np.arange(m ** 3)
        y = ((idx // m) % m + 1) * h
        z = (idx // (m * m) + 1) * h
        As = A.to_scipy()
        ones = sum(B[:, _col(a, s, 2)] for a in range(3) for s in range(2))
        assert np.max(np.abs(As @ np.ones(m ** 3) - ones)) < 1e-10
        # u = y: faces x=0/1 (first free coordinate y), z=0/1 (second free coordinate y), y=1 (constant)
        by = B[:, _col(0, 0, 0)] + B[:, _col(0, 1, 0)] + B[:, _col(2, 0, 1)] + B[:, _col(2, 1, 1)] + B[:, _col(1, 1, 2)]
        assert np.max(np.abs(As @ y - by)) < 1e-10
        # u = z: faces x=0/1 (second free coordinate), y=0/1 (second free coordinate), z=1 (constant)
        bz = B[:, _col(0, 0, 1)] + B[:, _col(0, 1, 1)] + B[:, _col(1, 0, 1)] + B[:, _col(1, 1, 1)] + B[:, _col(2, 1, 2)]
        assert np.max(np.abs(As @ z - bz)) < 1e-10


def test_ex2_manufactured_solution_second_order():
    """RHS 1 is f for u = exp(xyz) sin(pi x) sin(pi y) sin(pi z): the discrete
    solution converges to u at second order (nu = 10, Ex. 3's value)."""
    errs = []
    for m in (8, 16):
        A, B = synth.paper_ex2(m, 10.0)
        h = 1.0 / (m + 1)
        idx = np.arange(m ** 3)
        x, y, z = [((idx // m ** d) % m + 1) * h for d in range(3)]
        u = np.exp(x * y * z) * np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
        sol = spla.spsolve(A.to_scipy().tocsc(), B[:, 0])
        errs.append(np.max(np.abs(sol - u)))
    assert errs[1] < errs[0] / 3.0 and errs[1] < 5e-3


def test_lattice_tile_order_is_a_tiled_permutation():
    """synth.lattice_tile_order (the traversal hint of srk_matrix_set_row_order): a permutation of
    the L^4 sites in which a site's +-t neighbours lie w planes apart and whole (x, y) planes stay
    contiguous (index arithmetic only)."""
    import numpy as np
    import synth
    L, w = 8, 2
    o = synth.lattice_tile_order(L, w)
    assert o.dtype == np.int32 and np.array_equal(np.sort(o), np.arange(L ** 4))
    pos = np.empty(L ** 4, dtype=np.int64)
    pos[o] = np.arange(L ** 4)
    site = np.arange(L ** 4)
    t = site // L ** 3
    inner = t < L - 1
    assert np.all(pos[site[inner] + L ** 3] - pos[site[inner]] == w * L * L)       # +t: w planes later
    plane = o.reshape(-1, L * L)
    assert np.all(plane - plane[:, :1] == np.arange(L * L))                         # planes contiguous
    with __import__("pytest").raises(ValueError):
        synth.lattice_tile_order(8, 3)
