"""Oracle (test infrastructure only): right ILU(0) preconditioning, the paper's
preconditioned experiments (Table 2 lower half
P:833-848). Plain and slow by design.

ilu0(A): the incomplete LU factorisation without fill-in ("no-fill ILU", the Matlab
`ilu` the paper uses): L unit lower and U upper triangular with the
sparsity pattern of A, computed row by row in the IKJ order of the textbook
algorithm (Saad, Iterative Methods for Sparse Linear Systems, Alg. 10.4):
    for i = 1..n:  for k < i in row i:  a_ik /= u_kk;
                                       for j > k in row i (and in row k): a_ij -= a_ik u_kj
Its defining property (L U)_ij = A_ij on the pattern of A is what the tests check,
together with ILU(0) = LU when the factorisation has no fill.

ilutp(A, droptol, thresh): the incomplete LU "with threshold and pivoting with a drop
tolerance of 5e-2" the paper uses for Ex. 4 (Matlab's `ilu` type 'ilutp'). The
paper gives nothing beyond that phrase; reading R14 fixes the algorithm as the
left-looking (column) ILU with partial pivoting: for column j, x = A(:, j); the pivoted
rows are eliminated in step order k (x -= L(:, k) x_r, r the row pivoted at step k), a
multiplier with |x_r| < droptol ||A(:, j)||_2 is dropped instead of used; the pivot is the
largest |x_r| over the rows not yet pivoted (the original row j when |x_j| >= thresh
max |x_r|); the other entries below tol are dropped, the rest divided by the pivot form
L(:, j). Result: Pi A ~ L U, Pi the row permutation (perm[k] = row pivoted at step k),
L unit lower and U upper triangular in the permuted order, and Pi A - L U = exactly the
dropped entries (each below its column's tolerance) — the property the pins check.

Right preconditioning: the methods run on A M^-1 Y = B with M = L U (ILUTP:
M = Pi^T L U, M^-1 = U^-1 L^-1 Pi) and return X = M^-1 Y; the A^H products become (A M^-1)^H = M^-H A^H. `RightPrec` wraps A
so that the unchanged solvers of oracle/solvers.py see the preconditioned operator.
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import solvers


def ilu0(A):
    """(L, U) as CSR: L strictly lower + unit diagonal, U upper with the diagonal,
    both on the pattern of A (sorted columns). Raises ZeroDivisionError on a zero pivot."""
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    ip, ix, vals = A.indptr, A.indices, A.data.astype(np.result_type(A.data, np.float64)).copy()
    diag_pos = np.full(n, -1)
    for i in range(n):
        for p in range(ip[i], ip[i + 1]):
            if ix[p] == i:
                diag_pos[i] = p
    for i in range(n):
        pos = {int(ix[p]): p for p in range(ip[i], ip[i + 1])}
        for p in range(ip[i], ip[i + 1]):
            k = int(ix[p])
            if k >= i:
                break
            if diag_pos[k] < 0 or vals[diag_pos[k]] == 0:
                raise ZeroDivisionError(f"ILU(0): zero pivot in row {k}")
            vals[p] = vals[p] / vals[diag_pos[k]]
            lik = vals[p]
            for q in range(diag_pos[k] + 1, ip[k + 1]):  # u_kj, j > k
                j = int(ix[q])
                if j in pos:
                    vals[pos[j]] -= lik * vals[q]
        if diag_pos[i] < 0 or vals[diag_pos[i]] == 0:
            raise ZeroDivisionError(f"ILU(0): zero pivot in row {i}")
    F = sp.csr_matrix((vals, ix.copy(), ip.copy()), shape=A.shape)
    L = sp.tril(F, k=-1, format="csr") + sp.identity(n, dtype=vals.dtype, format="csr")
    U = sp.triu(F, k=0, format="csr")
    L.sort_indices()
    U.sort_indices()
    return L, U


def ilutp(A, droptol=5e-2, thresh=1.0):
    """(L, U, perm) of the threshold ILU with partial pivoting (reading R14):
    A[perm] ~ L @ U, L unit lower, U upper (CSR, sorted columns). Raises
    ZeroDivisionError when a column has no nonzero pivot candidate."""
    import heapq
    Ac = sp.csc_matrix(A)
    Ac.sort_indices()
    n = Ac.shape[0]
    dt = np.result_type(Ac.data, np.float64)
    perm = [-1] * n       # perm[k]: original row pivoted at step k
    step = {}             # original row -> its pivot step
    Lcol = []             # Lcol[k]: {original row: l_rk} (rows not pivoted before step k + 1)
    Ucol = []             # Ucol[j]: {k: u_kj}, the diagonal u_jj included
    for j in range(n):
        x = {int(r): dt.type(v) for r, v in zip(Ac.indices[Ac.indptr[j]:Ac.indptr[j + 1]],
                                                 Ac.data[Ac.indptr[j]:Ac.indptr[j + 1]])}
        tol = droptol * np.linalg.norm(Ac.data[Ac.indptr[j]:Ac.indptr[j + 1]])
        heap = [step[r] for r in x if r in step]
        heapq.heapify(heap)
        seen = set()
        u = {}
        while heap:  # pivoted rows in increasing step order
            k = heapq.heappop(heap)
            if k in seen:
                continue
            seen.add(k)
            ukj = x.pop(perm[k])
            if ukj == 0 or abs(ukj) < tol:
                continue  # dropped multiplier (not used, not stored)
            u[k] = ukj
            for r, l in Lcol[k].items():
                x[r] = x.get(r, 0) - l * ukj
                if r in step and step[r] not in seen:
                    heapq.heappush(heap, step[r])
        # x now holds only rows not yet pivoted
        cand = [(r, v) for r, v in x.items() if v != 0]
        if not cand:
            raise ZeroDivisionError(f"ILUTP: no pivot in column {j}")
        big = max(abs(v) for _, v in cand)
        imax = min(r for r, v in cand if abs(v) == big)
        piv = j if (j in x and j not in step and x[j] != 0 and abs(x[j]) >= thresh * big) else imax
        d = x.pop(piv)
        perm[j] = piv
        step[piv] = j
        u[j] = d
        Ucol.append(u)
        Lcol.append({r: v / d for r, v in x.items() if v != 0 and abs(v) >= tol})
    dtc = dt
    rows, cols, vals = [], [], []
    for k in range(n):
        for r, v in Lcol[k].items():
            rows.append(step[r]); cols.append(k); vals.append(v)
    L = sp.csr_matrix((np.asarray(vals, dtype=dtc), (rows, cols)), shape=(n, n)) + sp.identity(n, dtype=dtc, format="csr")
    rows, cols, vals = [], [], []
    for j in range(n):
        for k, v in Ucol[j].items():
            rows.append(k); cols.append(j); vals.append(v)
    U = sp.csr_matrix((np.asarray(vals, dtype=dtc), (rows, cols)), shape=(n, n))
    L.sort_indices()
    U.sort_indices()
    return L, U, np.asarray(perm, dtype=np.int64)


def apply_inv(L, U, P, perm=None):
    """M^-1 P = U^-1 (L^-1 P)  (with a row permutation: U^-1 L^-1 (Pi P), (Pi P)_k = P_perm[k])."""
    P = np.asarray(P)
    if perm is not None:
        P = P[perm]
    Y = spla.spsolve_triangular(L, P, lower=True, unit_diagonal=True)
    return spla.spsolve_triangular(U, Y, lower=False)


def apply_inv_adj(L, U, P, perm=None):
    """M^-H P = L^-H (U^-H P)  (with a row permutation: Pi^T L^-H U^-H P)."""
    P = np.asarray(P)
    UH = U.conj().T.tocsr()
    LH = L.conj().T.tocsr()
    Y = spla.spsolve_triangular(UH, P, lower=True)
    Z = spla.spsolve_triangular(LH, Y, lower=False, unit_diagonal=True)
    if perm is None:
        return Z
    out = np.empty_like(Z)
    out[perm] = Z
    return out


class _Adj:
    def __init__(self, op):
        self.op = op

    def __matmul__(self, P):  # (A M^-1)^H P = M^-H (A^H P)
        return apply_inv_adj(self.op.L, self.op.U, self.op.AH @ P, self.op.perm)

    def tocsr(self):
        return self

    @property
    def T(self):
        return self


class RightPrec:
    """The operator A M^-1 with M = L U, in the interface the oracle solvers use."""

    def __init__(self, A, L, U, perm=None):
        self.A, self.L, self.U, self.perm = sp.csr_matrix(A), L, U, perm
        self.AH = self.A.conj().T.tocsr()
        self.data = self.A.data
        self.shape = self.A.shape

    def __matmul__(self, P):
        return self.A @ apply_inv(self.L, self.U, P, self.perm)

    def conj(self):
        return _Conj(self)


class _Conj:
    def __init__(self, op):
        self.op = op

    @property
    def T(self):
        return _Adj(self.op)


def solve_right(method, A, B, L=None, U=None, perm=None, **kw):
    """oracle.solve on A M^-1 Y = B (M = ILU(0) of A unless L, U (and the ILUTP row
    permutation perm) are given); the result's X and recorded iterates are mapped back:
    X = M^-1 Y."""
    if L is None:
        L, U = ilu0(A)
    r = solvers.solve(method, RightPrec(A, L, U, perm), B, **kw)
    r.X = apply_inv(L, U, r.X, perm)
    r.Xs = [apply_inv(L, U, X, perm) for X in r.Xs]
    return r
