"""Oracle primitives — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package. The product path (the CUDA library and
its Python binding) never imports it.

Plain, slow, obviously-correct numpy/scipy versions of the block operations of
PAPER.md §2 and §4, in float64 / complex128. Every function names the passage
it follows (P:n = /root/reference/PAPER.md line n).

Conventions: <x, y> = y^H x and <X, Y> = tr(Y^H X).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

EPS_BRK = 1e-14   # reading G12: LU pivot |u_kk| <= EPS_BRK * max|G| is a singular Gram
EPS_DEFL = 1e-12  # reading G11: thin-QR diagonal <= EPS_DEFL * ||Z||_F is rank deficiency


class Breakdown(Exception):
    """Numerical breakdown: data, not an error."""

    def __init__(self, kind: str, col: int = -1):
        super().__init__(kind)
        self.kind = kind
        self.col = col


class Counter:
    """Vector-operation counter with Proposition 1's convention: an
    inner product or a SAXPY of length n is one vector operation."""

    def __init__(self):
        self.vector_ops = 0
        self.matvec_cols_A = 0
        self.matvec_cols_AH = 0


def H(X):
    return X.conj().T


def _sum_rows(prod: np.ndarray, order: str) -> np.ndarray:
    """Sum an (n, ...) array of elementwise products over its rows in a stated order.
    'seq'  : plain left-to-right accumulation over chunks of 64 rows,
    'rev'  : the same chunks accumulated right-to-left.
    Two orders exist only to measure the method's own rounding spread."""
    n = prod.shape[0]
    chunks = [prod[i:i + 64].sum(axis=0) for i in range(0, n, 64)] or [np.zeros(prod.shape[1:], prod.dtype)]
    if order == "rev":
        chunks = chunks[::-1]
    acc = np.zeros_like(chunks[0])
    for c in chunks:
        acc = acc + c
    return acc


def gram(Y: np.ndarray, X: np.ndarray, ctr: Counter | None = None, order: str = "blas") -> np.ndarray:
    """Block inner product Y^H X (sy x sx) — Alg. 3 Grams, e.g. (R̂^(k))^H R^(k)."""
    if ctr is not None:
        ctr.vector_ops += Y.shape[1] * X.shape[1]
    if order == "blas":
        return H(Y) @ X
    return _sum_rows(Y.conj()[:, :, None] * X[:, None, :], order)


def col_inner(X: np.ndarray, Y: np.ndarray, ctr: Counter | None = None, order: str = "blas") -> np.ndarray:
    """Per-column <x_i, y_i> = y_i^H x_i (Alg. 1)."""
    if ctr is not None:
        ctr.vector_ops += X.shape[1]
    if order == "blas":
        return np.einsum("ij,ij->j", Y.conj(), X)
    return _sum_rows(Y.conj() * X, order)


def trace_inner(X: np.ndarray, Y: np.ndarray, ctr: Counter | None = None, order: str = "blas"):
    """<X, Y> = tr(Y^H X) (Alg. 2)."""
    if ctr is not None:
        ctr.vector_ops += X.shape[1]
    if order == "blas":
        return np.vdot(Y.ravel(), X.ravel())
    return _sum_rows(Y.conj() * X, order).sum()


def sum_inner(y: np.ndarray, X: np.ndarray, ctr: Counter | None = None, order: str = "blas"):
    """sum(y^H X), the sum of the entries of the row vector y^H X (Alg. 4)."""
    if ctr is not None:
        ctr.vector_ops += X.shape[1]
    if order == "blas":
        return (y.conj() @ X).sum()
    return _sum_rows(y.conj()[:, None] * X, order).sum()


def fro2(X: np.ndarray, order: str = "blas") -> float:
    """||X||_F^2 (stopping criterion)."""
    if order == "blas":
        return float(np.vdot(X.ravel(), X.ravel()).real)
    return float(_sum_rows((X.conj() * X).real, order).sum())


def saxpy_count(ctr: Counter | None, n_ops: int):
    if ctr is not None:
        ctr.vector_ops += n_ops


def small_solve(G: np.ndarray, M: np.ndarray) -> np.ndarray:
    """G^{-1} M by LU with partial pivoting (SPEC small_solve S:106-114; reading G29).
    Singular Gram -> Breakdown('gram') (reading G12)."""
    G = np.atleast_2d(G)
    if not np.all(np.isfinite(G)) or not np.all(np.isfinite(M)):
        raise Breakdown("nonfinite")
    lu, piv = sla.lu_factor(G, check_finite=False)
    gmax = np.abs(G).max()
    if gmax == 0 or np.abs(np.diag(lu)).min() <= EPS_BRK * gmax:
        raise Breakdown("gram")
    return sla.lu_solve((lu, piv), M, check_finite=False)


def small_solve_h(G: np.ndarray, M: np.ndarray) -> np.ndarray:
    """G^{-H} M (adjoint reuse of Prop. 1's proof)."""
    return small_solve(H(G), M)


DEFL_SEED = 0x5EED1504  # seed of the rank-deficiency replacement vectors (f4)


def _splitmix64(x):
    """SplitMix64 finaliser on uint64 (wrapping) — the counter-based generator both
    sides implement for the replacement vectors (no shared code, same definition)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def counter_uniform(n: int, key: int, cplx: bool, seed: int = DEFL_SEED, row0: int = 0) -> np.ndarray:
    """Replacement vector number `key` (event * 64 + column): entry i (global row
    row0 + i) is 2u - 1, u = (splitmix64(h + 2i + part) >> 11) * 2^-53, with the stream
    h = splitmix64(seed ^ (key * 0x9E3779B97F4A7C15)); part 0 real, 1 imaginary."""
    with np.errstate(over="ignore"):
        h = _splitmix64(np.uint64(seed) ^ (np.uint64(key) * np.uint64(0x9E3779B97F4A7C15)))
        i = np.arange(row0, row0 + n, dtype=np.uint64)

        def part(p):
            v = _splitmix64(h + np.uint64(2) * i + np.uint64(p))
            return (v >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 2.0 - 1.0
    return part(0) + 1j * part(1) if cplx else part(0)


def thin_qr(Z: np.ndarray, ctr: Counter | None = None, order: str = "blas", fill=None):
    """Thin QR Z = Q C by modified Gram-Schmidt with one full re-orthogonalisation
    pass (Eq. (3); cost remark "3ns^2 ... modified Gram-Schmidt" P:598-603;
    SPEC thin_qr S:97-105). C is upper triangular with real non-negative diagonal.
    A diagonal <= EPS_DEFL*||Z||_F raises Breakdown('rank') (reading G11) — unless
    `fill` is given (rank-deficiency continuation; S:101, S:141;
    the implicit deflation of [Oleary80, Dub01]): then column j of Q is
    fill(j) orthogonalised (two passes) against q_0..q_{j-1} and normalised, C[j, j] = 0,
    and the later columns are orthogonalised against it as usual, so Z = Q C still
    holds with Q orthonormal (reading R8)."""
    n, s = Z.shape
    if order == "cholqr":
        return _cholqr2(Z, ctr)
    Q = np.array(Z, dtype=np.result_type(Z.dtype, np.float64), copy=True)
    C = np.zeros((s, s), dtype=Q.dtype)
    zn = np.sqrt(fro2(Z))
    for j in range(s):
        for _pass in range(2):
            for i in range(j):
                if order == "blas":
                    r = np.vdot(Q[:, i], Q[:, j])
                else:
                    r = _sum_rows(Q[:, i].conj() * Q[:, j], order)
                Q[:, j] -= r * Q[:, i]
                C[i, j] += r
        d = np.sqrt(fro2(Q[:, j:j + 1], order))
        if not np.isfinite(d) or d <= EPS_DEFL * zn or zn == 0:
            if fill is None or not np.isfinite(d):
                raise Breakdown("rank", j)
            Q[:, j] = fill(j)
            for _pass in range(2):
                for i in range(j):
                    r = np.vdot(Q[:, i], Q[:, j]) if order == "blas" else _sum_rows(Q[:, i].conj() * Q[:, j], order)
                    Q[:, j] -= r * Q[:, i]
            Q[:, j] /= np.sqrt(fro2(Q[:, j:j + 1], order))
            continue
        C[j, j] = d
        Q[:, j] /= d
    if ctr is not None:
        ctr.vector_ops += 3 * s * s  # "at least a cost of 3ns^2", counted as vector ops
    return Q, C


def _cholqr2(Z: np.ndarray, ctr: Counter | None = None):
    """The second thin-QR algorithm of reading G10 ("e.g. MGS", P:603 leaves it open):
    Cholesky QR applied twice, G = Z^H Z = R1^H R1, Z1 = Z R1^{-1}, Z1^H Z1 = R2^H R2,
    Q = Z1 R2^{-1}, C = R2 R1 (real positive diagonal). Used only as the oracle's
    alternative order (order="cholqr") to measure the method's rounding spread under the
    QR algorithm; a pivot <= 1e-14 tr(G) is rank deficiency (reading R5)."""
    s = Z.shape[1]
    Q = np.array(Z, dtype=np.result_type(Z.dtype, np.float64), copy=True)
    C = np.eye(s, dtype=Q.dtype)
    for _pass in range(2):
        G = H(Q) @ Q
        tr = float(np.trace(G).real)
        try:
            L = np.linalg.cholesky(G)
        except np.linalg.LinAlgError:
            raise Breakdown("rank")
        if tr <= 0 or np.min(np.abs(np.diag(L))) ** 2 <= 1e-14 * tr:
            raise Breakdown("rank")
        R = H(L)
        Q = sla.solve_triangular(R, Q.T, trans="T", lower=False).T if not np.iscomplexobj(Q) else \
            H(sla.solve_triangular(R, H(Q), trans="C", lower=False))
        C = R @ C
    if ctr is not None:
        ctr.vector_ops += 3 * s * s
    return Q, C


def unitary_qr_stack(M: np.ndarray):
    """Full QR of a (2s x s) stack, M = Omega [R; 0], Omega unitary 2s x 2s, R upper
    triangular with real non-negative diagonal (Householder via LAPACK; block QMR
    quasi-minimisation, SURVEY App. A.3 reading G19)."""
    k = M.shape[1]
    Om, R = np.linalg.qr(M, mode="complete")
    d = np.diag(R[:k, :k])
    ph = np.ones(k, dtype=np.result_type(M.dtype, np.float64))
    nz = np.abs(d) > 0
    ph[nz] = d[nz] / np.abs(d[nz])
    Om = Om.astype(ph.dtype, copy=True)
    R = R.astype(ph.dtype, copy=True)
    Om[:, :k] = Om[:, :k] * ph[None, :]
    R[:k, :] = R[:k, :] * ph.conj()[:, None]
    return Om, R[:k, :]
