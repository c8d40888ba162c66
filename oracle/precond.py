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

Right preconditioning: the methods run on A M^-1 Y = B with M = L U and
return X = M^-1 Y; the A^H products become (A M^-1)^H = M^-H A^H. `RightPrec` wraps A
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


def apply_inv(L, U, P):
    """M^-1 P = U^-1 (L^-1 P)."""
    P = np.asarray(P)
    Y = spla.spsolve_triangular(L, P, lower=True, unit_diagonal=True)
    return spla.spsolve_triangular(U, Y, lower=False)


def apply_inv_adj(L, U, P):
    """M^-H P = L^-H (U^-H P)."""
    P = np.asarray(P)
    UH = U.conj().T.tocsr()
    LH = L.conj().T.tocsr()
    Y = spla.spsolve_triangular(UH, P, lower=True)
    return spla.spsolve_triangular(LH, Y, lower=False, unit_diagonal=True)


class _Adj:
    def __init__(self, op):
        self.op = op

    def __matmul__(self, P):  # (A M^-1)^H P = M^-H (A^H P)
        return apply_inv_adj(self.op.L, self.op.U, self.op.AH @ P)

    def tocsr(self):
        return self

    @property
    def T(self):
        return self


class RightPrec:
    """The operator A M^-1 with M = L U, in the interface the oracle solvers use."""

    def __init__(self, A, L, U):
        self.A, self.L, self.U = sp.csr_matrix(A), L, U
        self.AH = self.A.conj().T.tocsr()
        self.data = self.A.data
        self.shape = self.A.shape

    def __matmul__(self, P):
        return self.A @ apply_inv(self.L, self.U, P)

    def conj(self):
        return _Conj(self)


class _Conj:
    def __init__(self, op):
        self.op = op

    @property
    def T(self):
        return _Adj(self.op)


def solve_right(method, A, B, L=None, U=None, **kw):
    """oracle.solve on A M^-1 Y = B (M = ILU(0) of A unless L, U are given); the
    result's X and recorded iterates are mapped back: X = M^-1 Y."""
    if L is None:
        L, U = ilu0(A)
    r = solvers.solve(method, RightPrec(A, L, U), B, **kw)
    r.X = apply_inv(L, U, r.X)
    r.Xs = [apply_inv(L, U, X) for X in r.Xs]
    return r
