"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the solvers (no products, inner products,
coefficients or factorisations of the method). It only builds the operators A
(CSR arrays) and right-hand sides B of SURVEY.md §8(d).1, which stand in for
the paper's examples (§5.1), whose matrices are not
available (Ex. 4 gauge field and Ex. 5 graphene matrix are missing).

Conventions:
  * grid unknown index i + m*j (+ m^2*k), x fastest; h = 1/(m+1);
  * operator h^2 * (-Laplace u + c . grad u), central differences: diagonal 2d,
    neighbour at +e_d gets -1 + c_d*h/2, at -e_d gets -1 - c_d*h/2;
    off-grid neighbours dropped (homogeneous Dirichlet); CSR columns ascending;
  * RHS: numpy default_rng(seed); real B = standard_normal((n, s));
    complex B = (standard_normal((n,s)) + 1j*standard_normal((n,s)))/sqrt(2).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np


@dataclass
class CSR:
    """Plain CSR arrays (0-based, sorted unique columns per row)."""
    n: int
    row_ptr: np.ndarray  # int64, n+1
    col_idx: np.ndarray  # int32, nnz
    values: np.ndarray   # float64 or complex128, nnz
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def dtype(self):
        return self.values.dtype

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.col_idx, self.row_ptr), shape=(self.n, self.n))


def _stencil_csr(dims: tuple, diag: complex, coup: list, dtype) -> CSR:
    """Assemble a structured-grid CSR matrix.

    dims: grid extents (x fastest). coup: list of (axis, direction, value) for
    the neighbour couplings. Columns come out ascending because neighbours are
    visited in order of their linear offset."""
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    strides = [1]
    for d in dims[:-1]:
        strides.append(strides[-1] * d)
    # entries: (offset, value, axis, direction); diagonal offset 0
    ents = [(0, diag, None, 0)]
    for axis, direction, val in coup:
        ents.append((direction * strides[axis], val, axis, direction))
    ents.sort(key=lambda e: e[0])
    idx = np.arange(n, dtype=np.int64)
    coords = []
    rem = idx
    for d in dims:
        coords.append((rem % d).astype(np.int32))
        rem = rem // d
    k = len(ents)
    valid = np.empty((n, k), dtype=bool)
    cols = np.empty((n, k), dtype=np.int32)
    vals = np.empty((n, k), dtype=dtype)
    for j, (off, val, axis, direction) in enumerate(ents):
        if axis is None:
            valid[:, j] = True
        elif direction > 0:
            valid[:, j] = coords[axis] < dims[axis] - 1
        else:
            valid[:, j] = coords[axis] > 0
        cols[:, j] = (idx + off).astype(np.int32)
        vals[:, j] = val
    counts = valid.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    m = valid.ravel()
    col_idx = cols.ravel()[m]
    values = vals.ravel()[m]
    return CSR(n, row_ptr, np.ascontiguousarray(col_idx), np.ascontiguousarray(values))


def conv_diff_2d(m: int, c=(20.0, 20.0), dtype=np.float64, shift=0.0) -> CSR:
    """2D 5-point h^2-scaled -Laplace u + c.grad u (config 1; stands in for Ex. 1)."""
    h = 1.0 / (m + 1)
    coup = []
    for axis in range(2):
        coup.append((axis, +1, -1.0 + c[axis] * h / 2))
        coup.append((axis, -1, -1.0 - c[axis] * h / 2))
    A = _stencil_csr((m, m), 4.0 + shift, coup, dtype)
    A.meta = dict(kind="conv_diff_2d", m=m, c=tuple(c), shift=shift)
    return A


def conv_diff_3d(m: int, c=(50.0, 30.0, 10.0), dtype=np.float64, shift=0.0) -> CSR:
    """3D 7-point h^2-scaled -Laplace u + c.grad u (+ shift on the diagonal);
    configs 2-3 (stand in for Ex. 2/3)."""
    h = 1.0 / (m + 1)
    coup = []
    for axis in range(3):
        coup.append((axis, +1, -1.0 + c[axis] * h / 2))
        coup.append((axis, -1, -1.0 - c[axis] * h / 2))
    A = _stencil_csr((m, m, m), 6.0 + shift, coup, dtype)
    A.meta = dict(kind="conv_diff_3d", m=m, c=tuple(c), shift=shift)
    return A


def _boundary_rhs(m: int, dims: int, coup_vals: dict, g) -> np.ndarray:
    """b = -sum over boundary neighbours of (coupling * g(boundary point)) for the
    h^2-scaled stencil on the m^dims interior grid (unknown index x fastest).
    coup_vals[(axis, direction)] is the neighbour coupling; g(points) evaluates the
    Dirichlet data at an (N, dims) array of boundary points."""
    h = 1.0 / (m + 1)
    n = m ** dims
    idx = np.arange(n, dtype=np.int64)
    co = [(idx // m ** d) % m + 1 for d in range(dims)]  # 1-based grid coordinates
    b = np.zeros(n)
    for (axis, direction), val in coup_vals.items():
        edge = m if direction > 0 else 1
        sel = co[axis] == edge
        pts = np.stack([c[sel] * h for c in co], axis=1)
        pts[:, axis] = 1.0 if direction > 0 else 0.0
        b[sel] -= val * g(pts)
    return b


def paper_ex1(m: int = 200, alpha=(5.0, 5.0, 5.0)):
    """Ex. 1 of the paper: -u_xx - u_yy + 2 a1 u_x + 2 a2 u_y - 2 a3 u = 0 on
    the unit square, Dirichlet data, a = (5, 5, 5), central differences on the m x m
    interior grid (h^2-scaled). Four right-hand sides, one per corner: the boundary
    data is continuous and piecewise linear along the boundary, 1 at that corner and
    0 at the other three. Returns (A, B) with B of shape (m^2, 4); corners in the order
    (0,0), (1,0), (0,1), (1,1)."""
    h = 1.0 / (m + 1)
    a1, a2, a3 = alpha
    A = conv_diff_2d(m, c=(2 * a1, 2 * a2), shift=-2 * a3 * h * h)
    coup = {(0, +1): -1.0 + a1 * h, (0, -1): -1.0 - a1 * h, (1, +1): -1.0 + a2 * h, (1, -1): -1.0 - a2 * h}

    def corner(cx, cy):
        # piecewise linear hat along the boundary: on the two edges through the corner
        # it falls linearly from 1 to 0, elsewhere it is 0
        def g(pts):
            x, y = pts[:, 0], pts[:, 1]
            on_vx = np.isclose(x, cx)  # edge x = cx: linear in y
            on_hy = np.isclose(y, cy)  # edge y = cy: linear in x
            return np.where(on_vx, 1.0 - np.abs(y - cy), 0.0) + np.where(on_hy & ~on_vx, 1.0 - np.abs(x - cx), 0.0)
        return g

    B = np.stack([_boundary_rhs(m, 2, coup, corner(cx, cy)) for cx, cy in ((0, 0), (1, 0), (0, 1), (1, 1))], axis=1)
    A.meta = dict(kind="paper_ex1", m=m, alpha=tuple(alpha))
    return A, B


def paper_ex2(m: int = 50, nu: float = 1000.0):
    """Ex. 2 of the paper (Ex. 3 = nu 10): u_xx + u_yy + u_zz +
    nu u_x = f on the unit cube, central differences on the m^3 interior grid, written
    as the h^2-scaled -Delta u - nu u_x = -f (conv_diff_3d with c = (-nu, 0, 0)).
    19 right-hand sides: (1) f such that u = exp(xyz) sin(pi x) sin(pi y) sin(pi z) with
    zero boundary data; (2-19) f = 0 with, for each face in the order x=0, x=1, y=0,
    y=1, z=0, z=1, the boundary data equal to its first free coordinate, its second
    free coordinate and 1 on that face (0 on the others)."""
    h = 1.0 / (m + 1)
    A = conv_diff_3d(m, c=(-nu, 0.0, 0.0))
    coup = {}
    for axis in range(3):
        cval = -nu if axis == 0 else 0.0
        coup[(axis, +1)] = -1.0 + cval * h / 2
        coup[(axis, -1)] = -1.0 - cval * h / 2
    n = m ** 3
    idx = np.arange(n, dtype=np.int64)
    x, y, z = [((idx // m ** d) % m + 1) * h for d in range(3)]
    E = np.exp(x * y * z)
    sx, sy, sz = np.sin(np.pi * x), np.sin(np.pi * y), np.sin(np.pi * z)
    cx, cy, cz = np.cos(np.pi * x), np.cos(np.pi * y), np.cos(np.pi * z)
    S = sx * sy * sz
    pi = np.pi
    uxx = E * ((y * z) ** 2 * S + 2 * y * z * pi * cx * sy * sz - pi * pi * S)
    uyy = E * ((x * z) ** 2 * S + 2 * x * z * pi * sx * cy * sz - pi * pi * S)
    uzz = E * ((x * y) ** 2 * S + 2 * x * y * pi * sx * sy * cz - pi * pi * S)
    ux = E * (y * z * S + pi * cx * sy * sz)
    f = uxx + uyy + uzz + nu * ux
    cols = [-h * h * f]
    for axis in range(3):
        for side in (0.0, 1.0):
            free = [d for d in range(3) if d != axis]

            def face(which, axis=axis, side=side, free=free):
                def g(pts):
                    on = np.isclose(pts[:, axis], side)
                    val = np.ones(len(pts)) if which == 2 else pts[:, free[which]]
                    return np.where(on, val, 0.0)
                return g
            for which in range(3):
                cols.append(_boundary_rhs(m, 3, coup, face(which)))
    B = np.stack(cols, axis=1)
    A.meta = dict(kind="paper_ex2", m=m, nu=nu)
    return A, B


def random_rhs(n: int, s: int, seed: int, complex_: bool = False) -> np.ndarray:
    """Gaussian right-hand sides, row-major draw order."""
    rng = np.random.default_rng(seed)
    if not complex_:
        return rng.standard_normal((n, s))
    re = rng.standard_normal((n, s))
    im = rng.standard_normal((n, s))
    return (re + 1j * im) / np.sqrt(2.0)


def random_sparse(n: int, nnz_per_row: int, seed: int, dtype=np.float64, dominance: float = 0.0) -> CSR:
    """Small random nonsymmetric sparse test matrix (tests only): nnz_per_row
    uniform random off-diagonal columns per row (duplicates merged) plus a
    diagonal equal to `dominance` x off-diagonal absolute row sum (+1)."""
    rng = np.random.default_rng(seed + 1000)
    rows = np.repeat(np.arange(n), nnz_per_row)
    cols = rng.integers(0, n, n * nnz_per_row)
    v = rng.standard_normal(n * nnz_per_row)
    if np.dtype(dtype).kind == "c":
        v = v + 1j * rng.standard_normal(n * nnz_per_row)
    import scipy.sparse as sp
    M = sp.coo_matrix((v, (rows, cols)), shape=(n, n)).tocsr()
    M.setdiag(0)
    M.eliminate_zeros()
    rs = np.asarray(abs(M).sum(axis=1)).ravel()
    M = M + sp.diags(dominance * rs + 1.0)
    M = M.tocsr()
    M.sort_indices()
    return CSR(n, M.indptr.astype(np.int64), M.indices.astype(np.int32),
               M.data.astype(dtype), dict(kind="random_sparse", seed=seed))


def power_law(n: int, seed: int, a: float = 1.19794, lmax: int = 512, lmin_scale: float = 4.0) -> CSR:
    """Config 5 (reading G24): row lengths L_i (counting
    the diagonal) = min(lmax, floor(4 U^(-1/a))), columns uniform over the other
    rows, values N(0,1), duplicates summed, diagonal 1.1 x off-diagonal abs sum."""
    rng = np.random.default_rng(seed + 1000)
    U = 1.0 - rng.random(n)
    L = np.minimum(lmax, np.floor(lmin_scale * U ** (-1.0 / a))).astype(np.int64)
    noff = L - 1
    tot = int(noff.sum())
    c = rng.integers(0, n - 1, tot)
    rows = np.repeat(np.arange(n, dtype=np.int64), noff)
    c = c + (c >= rows)
    v = rng.standard_normal(tot)
    import scipy.sparse as sp
    M = sp.coo_matrix((v, (rows, c)), shape=(n, n)).tocsr()  # duplicates summed
    M.sum_duplicates()
    rs = np.asarray(abs(M).sum(axis=1)).ravel()
    M = (M + sp.diags(1.1 * rs)).tocsr()
    M.sort_indices()
    return CSR(n, M.indptr.astype(np.int64), M.indices.astype(np.int32), M.data.astype(np.float64),
               dict(kind="power_law", seed=seed, a=a, lmax=lmax))


def _lattice_blocks(L: int, kappa: float, seed: int, dof: int, chunk: int):
    """Neighbour table (nsites, 8) and the stored blocks -kappa*H (nsites, 8, dof, dof)
    of config 4, in the draw order of SURVEY §8d.1 item 4 (shared by the CSR and
    the BSR forms, so both describe the same matrix)."""
    if L < 3:
        raise ValueError("L >= 3 keeps the 8 neighbours of a site distinct")
    rng = np.random.default_rng(seed + 1000)
    nsites = L ** 4
    site = np.arange(nsites, dtype=np.int64)
    co = [(site // L ** d) % L for d in range(4)]
    nbr = np.empty((nsites, 8), dtype=np.int64)
    for d in range(4):
        for k, step in enumerate((+1, -1)):
            c2 = list(co)
            c2[d] = (co[d] + step) % L
            nbr[:, 2 * d + k] = c2[0] + L * c2[1] + L ** 2 * c2[2] + L ** 3 * c2[3]
    vals = np.empty((nsites, 8, dof, dof), dtype=np.complex128)
    for start in range(0, nsites, chunk):
        c = min(chunk, nsites - start)
        re = rng.standard_normal((c, 8, dof, dof))
        im = rng.standard_normal((c, 8, dof, dof))
        vals[start:start + c] = (re + 1j * im) * np.sqrt(1.0 / 12.0)
    vals *= -kappa
    return nbr, vals


def lattice_4d(L: int, kappa: float = 0.12, seed: int = 3, dof: int = 12, chunk: int = 4096) -> CSR:
    """Config 4 (reading G23): periodic L^4 lattice, `dof`
    complex unknowns per site, A = I - kappa*H with H a nearest-neighbour coupling
    whose 8 blocks per site (order +x, -x, +y, -y, +z, -z, +t, -t; site index
    x + L y + L^2 z + L^3 t, row = dof*site + a) have entries CN(0, 1/6).
    Stands in for the paper's Wilson-Dirac Ex. 4, whose gauge field is
    not available. Matrix RNG default_rng(seed + 1000), drawn in chunks of `chunk`
    sites: re = standard_normal((c, 8, dof, dof)), then im of the same shape."""
    nbr, vals = _lattice_blocks(L, kappa, seed, dof, chunk)
    nsites = L ** 4
    n = nsites * dof
    site = np.arange(nsites, dtype=np.int64)
    # row (site, a): the 8 neighbour blocks (dof columns each) and the identity's
    # diagonal entry, in ascending column order -> 8*dof + 1 entries per row
    cols_site = np.concatenate([nbr, site[:, None]], axis=1)              # (nsites, 9) block columns
    order = np.argsort(cols_site, axis=1, kind="stable")
    cols_site = np.take_along_axis(cols_site, order, axis=1)
    full = np.zeros((nsites, 9, dof, dof), dtype=np.complex128)
    full[:, :8] = vals
    full[:, 8] = np.eye(dof)
    full = np.take_along_axis(full, order[:, :, None, None], axis=1)
    own = (order == 8)                                                     # (nsites, 9): the identity block
    col = cols_site[:, None, :, None] * dof + np.arange(dof)[None, None, None, :]   # (nsites, 1, 9, dof)
    col = np.broadcast_to(col, (nsites, dof, 9, dof))
    val = np.transpose(full, (0, 2, 1, 3))                                 # [site, a, blk, b]
    a_idx = np.arange(dof)[None, :, None, None]
    b_idx = np.arange(dof)[None, None, None, :]
    keep = ~own[:, None, :, None] | (a_idx == b_idx)                       # identity block: diagonal only
    keep = np.broadcast_to(keep, (nsites, dof, 9, dof))
    col = col[keep].reshape(n, 8 * dof + 1)
    val = val[keep].reshape(n, 8 * dof + 1)
    row_ptr = np.arange(0, n * (8 * dof + 1) + 1, 8 * dof + 1, dtype=np.int64)
    A = CSR(n, row_ptr, np.ascontiguousarray(col.reshape(-1).astype(np.int32)),
            np.ascontiguousarray(val.reshape(-1)))
    A.meta = dict(kind="lattice_4d", L=L, kappa=kappa, seed=seed, dof=dof)
    return A


def lattice_4d_bsr(L: int, kappa: float = 0.12, seed: int = 3, dof: int = 12, chunk: int = 4096):
    """The same operator as lattice_4d in block-sparse form with an implied unit
    diagonal: A = I + sum of the 8 stored neighbour blocks per block row.
    Returns (block_row_ptr int64 (nsites+1), block_col int32 (8 nsites, ascending
    within a block row), blocks complex128 (8 nsites, dof, dof) row-major).
    Generated chunk by chunk (same draws and arithmetic as _lattice_blocks), so the
    only full-size array is the output (19.3 GB at L = 32)."""
    if L < 3:
        raise ValueError("L >= 3 keeps the 8 neighbours of a site distinct")
    rng = np.random.default_rng(seed + 1000)
    nsites = L ** 4
    blocks = np.empty((nsites * 8, dof, dof), dtype=np.complex128)
    bcol = np.empty(nsites * 8, dtype=np.int32)
    for start in range(0, nsites, chunk):
        c = min(chunk, nsites - start)
        site = np.arange(start, start + c, dtype=np.int64)
        co = [(site // L ** d) % L for d in range(4)]
        nbr = np.empty((c, 8), dtype=np.int64)
        for d in range(4):
            for k, step in enumerate((+1, -1)):
                c2 = list(co)
                c2[d] = (co[d] + step) % L
                nbr[:, 2 * d + k] = c2[0] + L * c2[1] + L ** 2 * c2[2] + L ** 3 * c2[3]
        re = rng.standard_normal((c, 8, dof, dof))
        im = rng.standard_normal((c, 8, dof, dof))
        vals = (re + 1j * im) * np.sqrt(1.0 / 12.0)
        vals *= -kappa
        order = np.argsort(nbr, axis=1, kind="stable")
        bcol[8 * start:8 * (start + c)] = np.take_along_axis(nbr, order, axis=1).reshape(-1)
        blocks[8 * start:8 * (start + c)] = np.take_along_axis(vals, order[:, :, None, None], axis=1).reshape(c * 8, dof, dof)
    brp = np.arange(0, 8 * nsites + 1, 8, dtype=np.int64)
    return brp, bcol, blocks


def lattice_tile_order(L: int, w: int) -> np.ndarray:
    """Visiting order of the L^4 lattice sites (site = x + L y + L^2 z + L^3 t) that walks one
    tile of w z-planes through every t before the next tile: the +-t neighbours of a site are
    then w planes (w L^2 sites) apart in the order instead of L planes (index arithmetic only;
    the traversal hint of srk_matrix_set_row_order)."""
    if L % w:
        raise ValueError("w must divide L")
    zt, t, zi, yx = np.meshgrid(np.arange(L // w), np.arange(L), np.arange(w), np.arange(L * L), indexing="ij")
    return (yx + L * L * (zt * w + zi) + L ** 3 * t).reshape(-1).astype(np.int32)


def input_hash(A: CSR, B: np.ndarray) -> str:
    h = hashlib.sha256()
    for arr in (A.row_ptr, A.col_idx, A.values, B):
        h.update(np.ascontiguousarray(arr).view(np.uint8).data)
    return h.hexdigest()[:16]


# ---------------------------------------------------------------------------
# BASELINE.json configs (SURVEY §8 "Config geometry")
# ---------------------------------------------------------------------------

CONFIGS = {
    1: dict(name="cfg1_conv_diff_2d_32", dims=2, m=32, c=(20.0, 20.0), dtype="f64", s=4, seed=0,
            methods=("egl_bicg", "bl_bicgstab_rq")),
    2: dict(name="cfg2_conv_diff_3d_128_c128", dims=3, m=128, c=(50.0, 30.0, 10.0), dtype="c128",
            shift=-0.1j, s=8, seed=1, methods=("bl_bicg_rq", "bl_qmr", "bl_bicgstab_rq")),
    3: dict(name="cfg3_conv_diff_3d_256", dims=3, m=256, c=(50.0, 30.0, 10.0), dtype="f64", s=16, seed=2,
            methods=("egl_qmr", "gl_bicgstab")),
    4: dict(name="cfg4_lattice_32^4_c128", L=32, dtype="c128", s=12, seed=3, kappa=0.12,
            methods=("li_bicgstab", "gl_bicgstab", "bl_bicgstab", "bl_bicgstab_rq")),
    5: dict(name="cfg5_power_law_4M", n=1 << 22, dtype="f64", s=32, seed=4, methods=("egl_bicg",)),
}


def make_config(cfg: int, m: int | None = None, s: int | None = None, n: int | None = None):
    """Build (A, B) for a BASELINE config; m / s / n override sizes for scaled-down tests."""
    c = CONFIGS[cfg]
    s = c["s"] if s is None else s
    cplx = c["dtype"] == "c128"
    dt = np.complex128 if cplx else np.float64
    if cfg in (1, 2, 3):
        mm = c["m"] if m is None else m
        if c["dims"] == 2:
            A = conv_diff_2d(mm, c["c"], dt, c.get("shift", 0.0))
        else:
            A = conv_diff_3d(mm, c["c"], dt, c.get("shift", 0.0))
    elif cfg == 4:
        A = lattice_4d(c["L"] if m is None else m, c["kappa"], c["seed"])
    elif cfg == 5:
        nn = c["n"] if n is None else n
        A = power_law(nn, c["seed"])
    else:
        raise ValueError(cfg)
    B = random_rhs(A.n, s, c["seed"], cplx)
    return A, B
