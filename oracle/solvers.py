"""Oracle solvers — TEST INFRASTRUCTURE ONLY (see oracle/linalg.py header).

Plain numpy/scipy implementations of the 13 simultaneous short-recurrence
methods, written step by step in the paper's order and notation:

  BiCG family   : Alg. 1 Li-BiCG, Alg. 2 Gl-BiCG,
                  Alg. 3 Bl-BiCG (with the adjoint reuse of
                  Prop. 1's proof P:279-285), Alg. 4 eGl-BiCG,
                  Alg. 5 Bl-BiCG-rQ (Eqs. (4)-(7) P:541-560).
  QMR family    : Li/Gl/eGl-QMR (named P:300-301; not printed),
                  Bl-QMR (characterised P:300-305) — step lists SURVEY App. A.2/A.3.
  BiCGStab      : Li/Gl/Bl-BiCGStab ([ELg03] delegated) and
                  Bl-BiCGStab-rQ (not printed) — SURVEY App. A.4/A.5.

Readings of the paper: X0 = 0 default, shadow
R̂0 = R0, economic shadow = column mean, stop when the recursive
‖R‖_F (‖C‖_F for rQ) <= tol·‖R0‖_F confirmed by the true
residual (G26), breakdown rules G11/G12, Li per-column freeze G13.

Parity status: every solver here is pinned by tests/test_oracle_*.py against
scipy's single-RHS bicg/qmr/bicgstab (s=1 and per column), the Kronecker lift
(P:165-184), the rank-1 shadow equivalence, the rQ exact-arithmetic
equivalences (Eqs. (4)-(7)), Petrov-Galerkin conditions, brute-force
quasi-minimisation (QMR), finite termination and dense direct solves.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .linalg import (Breakdown, Counter, H, col_inner, counter_uniform, fro2, gram, saxpy_count, small_solve,
                     small_solve_h, sum_inner, thin_qr, trace_inner, unitary_qr_stack)

METHODS = ("li_bicg", "gl_bicg", "egl_bicg", "bl_bicg", "bl_bicg_rq",
           "li_qmr", "gl_qmr", "egl_qmr", "bl_qmr",
           "li_bicgstab", "gl_bicgstab", "bl_bicgstab", "bl_bicgstab_rq")


@dataclass
class Result:
    X: np.ndarray
    outcome: str = "maxit"          # converged | maxit | breakdown | diverged
    iterations: int = 0
    half_step: bool = False
    breakdown_kind: str = ""
    breakdown_iter: int = -1
    breakdown_cols: list = field(default_factory=list)
    history: list = field(default_factory=list)      # recursive relative residual per iteration
    Xs: list = field(default_factory=list)           # X_k, k = 1..record
    Rs: list = field(default_factory=list)           # R_k (or C_k for rQ), k = 1..record
    coefs: list = field(default_factory=list)        # per-iteration scalars / s x s coefficients
    matvec_cols_A: int = 0
    matvec_cols_AH: int = 0
    vector_ops: int = 0
    final_true_rel_residual: float = float("nan")


class _Run:
    """Shared bookkeeping: counters, recording, and the stopping rule of P:643
    with the true-residual confirmation (reading G26)."""

    def __init__(self, A, B, X0, tol, maxit, record, order):
        self.A = A
        self.B = np.asarray(B)
        cplx = np.iscomplexobj(B) or np.iscomplexobj(A.data)
        self.dt = np.complex128 if cplx else np.float64
        self.B = self.B.astype(self.dt)
        self.X = np.zeros_like(self.B) if X0 is None else np.array(X0, dtype=self.dt)
        self.tol, self.maxit, self.record, self.order = tol, maxit, record, order
        self.ctr = Counter()
        self.res = Result(self.X)
        self.R0 = self.B - A @ self.X
        self.r0norm = np.sqrt(fro2(self.R0))
        self._AH = None

    @property
    def AH(self):
        if self._AH is None:
            self._AH = self.A.conj().T.tocsr()
        return self._AH

    def matA(self, P):
        self.ctr.matvec_cols_A += P.shape[1] if P.ndim == 2 else 1
        return self.A @ P

    def matAH(self, P):
        self.ctr.matvec_cols_AH += P.shape[1] if P.ndim == 2 else 1
        return self.AH @ P

    def true_rel(self, X):
        if self.r0norm == 0:
            return 0.0
        return float(np.sqrt(fro2(self.B - self.A @ X)) / self.r0norm)

    def step_done(self, k, X, resnorm, Rrec=None, coef=None):
        """Record iteration k (1-based) and decide whether to stop."""
        self.res.iterations = k
        rel = resnorm / self.r0norm if self.r0norm > 0 else 0.0
        self.res.history.append(float(rel))
        if k <= self.record:
            self.res.Xs.append(X.copy())
            if Rrec is not None:
                self.res.Rs.append(Rrec.copy())
            self.res.coefs.append(coef)
        if not np.isfinite(rel):
            raise Breakdown("nonfinite")
        if rel <= self.tol:
            if self.true_rel(X) <= self.tol:
                self.res.outcome = "converged"
                return True
        return False

    def finish(self, X):
        r = self.res
        r.X = X
        r.matvec_cols_A = self.ctr.matvec_cols_A
        r.matvec_cols_AH = self.ctr.matvec_cols_AH
        r.vector_ops = self.ctr.vector_ops
        r.final_true_rel_residual = self.true_rel(X)
        if r.outcome == "maxit" and r.final_true_rel_residual > 1:
            r.outcome = "diverged"
        return r

    def breakdown(self, X, e: Breakdown, k: int):
        # A breakdown at an iterate that already meets the stopping rule is a
        # "lucky" breakdown (e.g. a thin QR of an exactly zero residual): converged.
        if k > 0 and self.true_rel(X) <= self.tol:
            self.res.iterations = k
            self.res.outcome = "converged"
            return self.finish(X)
        self.res.outcome = "breakdown"
        self.res.breakdown_kind = e.kind
        self.res.breakdown_iter = k
        return self.finish(X)


def _shadow_block(run: _Run, shadow):
    """R̂0 choice: 'r0' (default), 'conj', or a given block."""
    if shadow is None or (isinstance(shadow, str) and shadow == "r0"):
        return run.R0.copy()
    if isinstance(shadow, str) and shadow == "conj":
        return run.R0.conj().copy()
    if isinstance(shadow, str) and shadow == "mean":
        r = run.R0.mean(axis=1)
        return np.repeat(r[:, None], run.R0.shape[1], axis=1)
    return np.array(shadow, dtype=run.dt)


def _shadow_vector(run: _Run, shadow):
    """Economic r̂0: arithmetic mean of the initial residuals; 'conj' its
    complex conjugate (the economic analogue of R̂0 = conj(R0)), or a given vector."""
    if shadow is None or (isinstance(shadow, str) and shadow == "mean"):
        return run.R0.mean(axis=1)
    if isinstance(shadow, str) and shadow == "conj":
        return run.R0.mean(axis=1).conj()
    return np.array(shadow, dtype=run.dt).reshape(-1)


def _safe_div(num, den, frozen):
    """Per-column division with the Li freeze policy (reading G13): a zero
    denominator or a non-finite quotient freezes that column (coefficient 0)."""
    out = np.zeros(np.broadcast(num, den).shape, dtype=np.result_type(num, den))
    ok = (den != 0) & ~frozen
    with np.errstate(all="ignore"):
        q = np.where(ok, num / np.where(den == 0, 1, den), 0)
    bad = ok & ~np.isfinite(q)
    newly = (~ok & ~frozen) | bad
    q = np.where(newly | frozen, 0, q)
    return q, newly


def _deflation_fill(run: _Run, deflate: bool):
    """fill(event) -> the thin-QR replacement callable of QR number `event` (init 0;
    iteration k: 2k for the residual factor, 2k + 1 for the shadow's), or None
    (BREAKDOWN(rank) policy, reading G11)."""
    n, cplx = run.B.shape[0], run.dt == np.complex128
    if not deflate:
        return lambda event: None
    return lambda event: (lambda j: counter_uniform(n, event * 64 + j, cplx))


def _quiet(fn):
    """Run a solver with numpy FP warnings silenced: breakdowns are detected
    explicitly (non-finite coefficients), not through warnings."""
    import functools

    @functools.wraps(fn)
    def wrapper(*a, **kw):
        with np.errstate(all="ignore"):
            return fn(*a, **kw)
    return wrapper


def _scalar_div(num, den, kind):
    """Scalar coefficient with breakdown on a zero denominator."""
    if den == 0 or not np.isfinite(num) or not np.isfinite(den):
        raise Breakdown(kind)
    q = num / den
    if not np.isfinite(q):
        raise Breakdown(kind)
    return q


# =============================================================================
# BiCG family
# =============================================================================

@_quiet
def li_bicg(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Alg. 1 Li-BiCG: s BiCGs in lockstep, per-column α_i, β_i."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    Rh = _shadow_block(run, shadow)
    P, Ph = R.copy(), Rh.copy()
    frozen = np.zeros(s, dtype=bool)
    rho = col_inner(R, Rh, None, order)          # <r_i, r̂_i>, saved for re-use
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    for k in range(1, maxit + 1):
        Q = run.matA(P)                              # Q = A P
        Qh = run.matAH(Ph)                           # A^H P̂
        den = col_inner(Q, Ph, ctr, order)           # <q_i, p̂_i>
        alpha, newly = _safe_div(rho, den, frozen)
        frozen |= newly
        X = X + P * alpha[None, :]
        R = R - Q * alpha[None, :]
        Rh = Rh - Qh * alpha.conj()[None, :]
        saxpy_count(ctr, 3 * s)
        rho_new = col_inner(R, Rh, ctr, order)
        beta, newly = _safe_div(rho_new, rho, frozen)
        frozen |= newly
        P = R + P * beta[None, :]
        Ph = Rh + Ph * beta.conj()[None, :]
        saxpy_count(ctr, 2 * s)
        rho = rho_new
        run.res.breakdown_cols = [int(i) for i in np.nonzero(frozen)[0]]
        if frozen.all():
            return run.breakdown(X, Breakdown("lanczos"), k)
        if run.step_done(k, X, np.sqrt(fro2(R, order)), R, dict(alpha=alpha.copy(), beta=beta.copy())):
            break
    return run.finish(X)


@_quiet
def gl_bicg(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Alg. 2 Gl-BiCG: BiCG on (I⊗A)x = b with traces."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    Rh = _shadow_block(run, shadow)
    P, Ph = R.copy(), Rh.copy()
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    rho = trace_inner(R, Rh, None, order)        # tr(R̂^H R)
    k = 0
    try:
        for k in range(1, maxit + 1):
            Q = run.matA(P)
            Qh = run.matAH(Ph)
            alpha = _scalar_div(rho, trace_inner(Q, Ph, ctr, order), "lanczos")
            X = X + alpha * P
            R = R - alpha * Q
            Rh = Rh - np.conj(alpha) * Qh
            saxpy_count(ctr, 3 * s)
            rho_new = trace_inner(R, Rh, ctr, order)
            beta = _scalar_div(rho_new, rho, "lanczos")
            P = R + beta * P
            Ph = Rh + np.conj(beta) * Ph
            saxpy_count(ctr, 2 * s)
            rho = rho_new
            if run.step_done(k, X, np.sqrt(fro2(R, order)), R, dict(alpha=alpha, beta=beta)):
                break
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


@_quiet
def egl_bicg(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Alg. 4 eGl-BiCG: Gl-BiCG with R̂0 = r̂0 1^T kept as one vector;
    one A^H-vector product per iteration."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    rh = _shadow_vector(run, shadow)
    P, ph = R.copy(), rh.copy()
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    rho = sum_inner(rh, R, None, order)          # sum(r̂^H R)
    k = 0
    try:
        for k in range(1, maxit + 1):
            Q = run.matA(P)
            qh = run.matAH(ph)                       # A^H p̂ (one vector)
            alpha = _scalar_div(rho, sum_inner(ph, Q, ctr, order), "lanczos")
            X = X + alpha * P
            R = R - alpha * Q
            rh = rh - np.conj(alpha) * qh
            saxpy_count(ctr, 2 * s + 1)
            rho_new = sum_inner(rh, R, ctr, order)
            beta = _scalar_div(rho_new, rho, "lanczos")
            P = R + beta * P
            ph = rh + np.conj(beta) * ph
            saxpy_count(ctr, s + 1)
            rho = rho_new
            if run.step_done(k, X, np.sqrt(fro2(R, order)), R, dict(alpha=alpha, beta=beta)):
                break
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


@_quiet
def bl_bicg(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Alg. 3 Bl-BiCG with the adjoint reuse of Prop. 1's proof
    (P:279-285): α̂ = G^{-H} M^H, β̂ = M^{-H} M₊^H (reading G5)."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    Rh = _shadow_block(run, shadow)
    P, Ph = R.copy(), Rh.copy()
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    M = gram(Rh, R, None, order)                 # (R̂^(k))^H R^(k)
    k = 0
    try:
        for k in range(1, maxit + 1):
            Q = run.matA(P)
            Qh = run.matAH(Ph)
            G = gram(Ph, Q, ctr, order)              # (P̂^(k))^H Q^(k)
            alpha = small_solve(G, M)
            alpha_h = small_solve_h(G, H(M))
            X = X + P @ alpha
            R = R - Q @ alpha
            Rh = Rh - Qh @ alpha_h
            saxpy_count(ctr, 3 * s * s)
            M_new = gram(Rh, R, ctr, order)
            beta = small_solve(M, M_new)
            beta_h = small_solve_h(M, H(M_new))
            P = R + P @ beta
            Ph = Rh + Ph @ beta_h
            saxpy_count(ctr, 2 * s * s)
            M = M_new
            if run.step_done(k, X, np.sqrt(fro2(R, order)), R, dict(alpha=alpha, beta=beta)):
                break
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


@_quiet
def bl_bicg_rq(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas", deflate=False):
    """Alg. 5 Bl-BiCG-rQ, loop from k = 0 (reading G1), α̂/β̂ by
    adjoint reuse (G5), Ŝ^H in β and S^H in β̂ as printed (G4), stopping on
    ‖C^(k)‖_F. Names: Qr = orthonormal residual factor, Sig = S.
    deflate=True: rank-deficiency continuation (f4) instead of BREAKDOWN(rank) —
    no C or Σ is ever inverted, so a zero diagonal of C just "hides" the deflated
    direction."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    fill = _deflation_fill(run, deflate)
    k = 0
    try:
        Qr, C = thin_qr(run.R0, None, order, fill(0))          # Q^(0) C^(0) = R^(0)
        Qh, Ch = thin_qr(_shadow_block(run, shadow), None, order, fill(0))
        V, Vh = Qr.copy(), Qh.copy()
        G2 = gram(Qh, Qr, None, order)                         # (Q̂^(k))^H Q^(k)
        for k in range(1, maxit + 1):
            W = run.matA(V)
            Wh = run.matAH(Vh)
            G1 = gram(Vh, W, ctr, order)                       # (V̂^(k))^H W^(k)
            alpha = small_solve(G1, G2)                        # Eq. (4)
            alpha_h = small_solve_h(G1, H(G2))                 # Eq. (5)
            X = X + V @ (alpha @ C)
            Qr_new, Sig = thin_qr(Qr - W @ alpha, ctr, order, fill(2 * k))
            C = Sig @ C
            Qh_new, Sig_h = thin_qr(Qh - Wh @ alpha_h, ctr, order, fill(2 * k + 1))
            Ch = Sig_h @ Ch
            saxpy_count(ctr, 3 * s * s)
            G2_new = gram(Qh_new, Qr_new, ctr, order)
            beta = small_solve(G2, H(Sig_h) @ G2_new)          # Eq. (6)
            beta_h = small_solve_h(G2, H(Sig) @ H(G2_new))     # Eq. (7)
            V = Qr_new + V @ beta
            Vh = Qh_new + Vh @ beta_h
            saxpy_count(ctr, 2 * s * s)
            Qr, Qh, G2 = Qr_new, Qh_new, G2_new
            if run.step_done(k, X, np.sqrt(fro2(C)), C, dict(alpha=alpha, beta=beta, C=C.copy())):
                break
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


@_quiet
def bl_bicg_sq(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Bl-BiCG with QR-factorised search directions — the stabilisation of [Oleary80]
    that the paper names and rejects in favour of the residual QR ("use a QR
    factorization of the search direction block vectors P^(k) and P̂^(k)").
    The paper prints no recurrences; derived here (reading R9): P and P̂ are
    kept orthonormal, so α, β come from the defining conditions instead of M = R̂^H R:
      Galerkin      P̂^H R₊ = 0            ->  α = G^{-1} P̂^H R,   G = P̂^H A P
      biconjugacy   P̂^H A (R₊ + P β) = 0   ->  β = -G^{-1} (A^H P̂)^H R₊
    and the shadow side with G^H (α̂ = G^{-H} P^H R̂, β̂ = -G^{-H} (A P)^H R̂₊). Any basis
    of the Bl-BiCG search space gives the same X_k (the s x s coefficients absorb it),
    so in exact arithmetic the iterates are Alg. 3's."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    Rh = _shadow_block(run, shadow)
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    k = 0
    try:
        P = thin_qr(R, None, order)[0]               # orthonormal basis of span(R0)
        Ph = thin_qr(Rh, None, order)[0]
        for k in range(1, maxit + 1):
            Q = run.matA(P)
            Qh = run.matAH(Ph)
            G = gram(Ph, Q, ctr, order)              # P̂^H A P
            alpha = small_solve(G, gram(Ph, R, ctr, order))
            alpha_h = small_solve_h(G, gram(P, Rh, ctr, order))
            X = X + P @ alpha
            R = R - Q @ alpha
            Rh = Rh - Qh @ alpha_h
            saxpy_count(ctr, 3 * s * s)
            beta = -small_solve(G, gram(Qh, R, ctr, order))
            beta_h = -small_solve_h(G, gram(Q, Rh, ctr, order))
            P = thin_qr(R + P @ beta, ctr, order)[0]
            Ph = thin_qr(Rh + Ph @ beta_h, ctr, order)[0]
            saxpy_count(ctr, 2 * s * s)
            if run.step_done(k, X, np.sqrt(fro2(R, order)), R, dict(alpha=alpha, beta=beta)):
                break
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


@_quiet
def bl_bicgstab_sq(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Bl-BiCGStab with QR-factorised search directions ("a corresponding variant
    based on QR factorization of the search directions"). SURVEY App. A.4
    with P kept orthonormal: α = G^{-1} R̃^H R and β = -G^{-1} R̃^H T are basis
    covariant (P -> P γ gives α -> γ^{-1} α, β -> γ^{-1} β), so P₊ = qr(R + (P - ω U) β)
    changes no iterate in exact arithmetic (reading R9)."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    Rt = _shadow_block(run, shadow)
    k = 0
    try:
        P = thin_qr(R, None, order)[0]
        for k in range(1, maxit + 1):
            U = run.matA(P)
            G = gram(Rt, U, ctr, order)                  # R̃^H U
            alpha = small_solve(G, gram(Rt, R, ctr, order))
            S = R - U @ alpha
            saxpy_count(ctr, s * s)
            snorm = np.sqrt(fro2(S, order))
            if snorm / run.r0norm <= tol:
                Xh = X + P @ alpha
                if run.true_rel(Xh) <= tol:
                    X = Xh
                    run.res.half_step = True
                    run.res.outcome = "converged"
                    run.step_done(k, X, snorm, S, dict(alpha=alpha))
                    break
            T = run.matA(S)
            omega = _scalar_div(trace_inner(S, T, ctr, order), trace_inner(T, T, ctr, order), "omega")
            X = X + P @ alpha + omega * S
            R = S - omega * T
            saxpy_count(ctr, s * s + 2 * s)
            beta = -small_solve(G, gram(Rt, T, ctr, order))
            P = thin_qr(R + (P - omega * U) @ beta, ctr, order)[0]
            saxpy_count(ctr, s * s + s)
            if run.step_done(k, X, np.sqrt(fro2(R, order)), R, dict(alpha=alpha, omega=omega, beta=beta)):
                break
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


# =============================================================================
# QMR family (coupled two-term, no look-ahead, unit
# weights — reading G17; [FrNa92] cited at P:94-95)
# =============================================================================

@_quiet
def _qmr_li_gl(A, B, tol, maxit, X0, shadow, record, order, mode):
    """Li-QMR (mode 'li': every scalar an s-vector, column norms), Gl-QMR
    (mode 'gl': traces and Frobenius norms), eGl-QMR (mode 'egl': the left
    Lanczos block W̃ = w̃ 1^T kept as one vector, ξ = √s‖w̃‖, reading G18)."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    li = mode == "li"
    egl = mode == "egl"

    def nrm(Y):
        if li:
            return np.sqrt(np.real(col_inner(Y, Y, None, order)))
        if egl and Y.ndim == 1:
            return np.sqrt(s) * np.sqrt(fro2(Y[:, None], order))
        return np.sqrt(fro2(Y, order))

    def inner(Xb, Yb):   # <X, Y> in the variant's sense
        if li:
            return col_inner(Xb, Yb, ctr, order)
        if egl:
            return sum_inner(Yb, Xb, ctr, order)
        return trace_inner(Xb, Yb, ctr, order)

    frozen = np.zeros(s, dtype=bool)

    def div(num, den):
        nonlocal frozen
        if li:
            q, newly = _safe_div(num, den, frozen)
            frozen |= newly
            return q
        return _scalar_div(num, den, "lanczos")

    Vt = R.copy()
    rho = nrm(Vt)
    Wt = _shadow_vector(run, shadow) if egl else _shadow_block(run, shadow)
    xi = nrm(Wt)
    shp = (s,) if li else ()
    gam_prev = np.ones(shp)
    eta = -np.ones(shp, dtype=run.dt)
    theta_prev = np.zeros(shp)
    eps = None
    P = Q = D = S = None
    k = 0
    try:
        for k in range(1, maxit + 1):
            V = Vt * div(1.0, rho)
            W = Wt * div(1.0, xi)
            delta = inner(V, W)
            if k == 1:
                P, Q = V.copy(), W.copy()
            else:
                P = V - P * div(xi * delta, eps)
                Q = W - Q * np.conj(div(rho * delta, eps))
                saxpy_count(ctr, s + (1 if egl else s))
            Pt = run.matA(P)
            eps = inner(Pt, Q)
            beta = div(eps, delta)
            Vt = Pt - V * beta
            rho_new = nrm(Vt)
            Wt = run.matAH(Q) - W * np.conj(beta)
            xi = nrm(Wt)
            saxpy_count(ctr, s + (1 if egl else s))
            theta = rho_new / (gam_prev * np.abs(beta))
            gam = 1.0 / np.sqrt(1.0 + theta ** 2)
            eta = -eta * rho * gam ** 2 / (beta * gam_prev ** 2)
            if li:
                theta = np.where(frozen, 0.0, theta)
                gam = np.where(frozen, 1.0, gam)
                eta = np.where(frozen, 0.0, eta)
            if not li and (gam == 0 or not np.isfinite(eta)):
                raise Breakdown("lanczos")
            if k == 1:
                D = P * eta
                S = Pt * eta
            else:
                f = (theta_prev * gam) ** 2
                D = P * eta + D * f
                S = Pt * eta + S * f
            X = X + D
            R = R - S
            saxpy_count(ctr, 4 * s)
            rho, gam_prev, theta_prev = rho_new, gam, theta
            if li:
                run.res.breakdown_cols = [int(i) for i in np.nonzero(frozen)[0]]
                if frozen.all():
                    return run.breakdown(X, Breakdown("lanczos"), k)
            if run.step_done(k, X, np.sqrt(fro2(R, order)), R,
                             dict(beta=np.copy(beta), eta=np.copy(eta), theta=np.copy(theta))):
                break
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


def li_qmr(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Li-QMR: s QMRs in lockstep."""
    return _qmr_li_gl(A, B, tol, maxit, X0, shadow, record, order, "li")


def gl_qmr(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Gl-QMR: QMR on (I⊗A)x = b with traces/Frobenius norms."""
    return _qmr_li_gl(A, B, tol, maxit, X0, shadow, record, order, "gl")


def egl_qmr(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """eGl-QMR: Gl-QMR with a rank-1 left Lanczos block, one A^H-vector product
    per iteration."""
    return _qmr_li_gl(A, B, tol, maxit, X0, shadow, record, order, "egl")


@_quiet
def bl_qmr(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas", trace=None):
    """Block QMR built on matrix-block products (P:300-305 characterisation;
    SURVEY App. A.3, reading G19): QR-normalised two-sided block Lanczos
    (coupled two-term, no look-ahead) and a quasi-minimal residual over the
    nested bi-orthogonal basis via a 2s x 2s unitary per iteration."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    k = 0
    try:
        V, rho = thin_qr(R, None, order)
        W, xi = thin_qr(_shadow_block(run, shadow), None, order)
        tau_t = rho.copy()
        Om_prev = None
        P = Q = D = F = eps = None
        for k in range(1, maxit + 1):
            delta = gram(W, V, ctr, order)                       # W^H V
            if k == 1:
                P, Q = V.copy(), W.copy()
            else:
                P = V - P @ small_solve(eps, H(xi) @ delta)
                Q = W - Q @ small_solve_h(eps, H(rho) @ H(delta))
                saxpy_count(ctr, 2 * s * s)
            AP = run.matA(P)
            eps = gram(Q, AP, ctr, order)                        # Q^H A P
            beta = small_solve(delta, eps)
            gam_h = small_solve_h(delta, H(eps))
            pending = None
            try:
                V_new, rho_new = thin_qr(AP - V @ beta, ctr, order)
            except Breakdown as e:       # deferred: the quasi-minimisation still uses ρ₊ (exactly 0 if AP ∈ span V)
                pending, V_new = e, None
                rho_new = np.linalg.qr(AP - V @ beta, mode="r")
                rho_new = rho_new * np.where(np.diag(rho_new) == 0, 1, np.conj(np.sign(np.diag(rho_new))))[:, None]
            AHQ = run.matAH(Q)
            try:
                W_new, xi_new = thin_qr(AHQ - W @ gam_h, ctr, order)
            except Breakdown as e:
                pending, W_new, xi_new = e, None, None
            saxpy_count(ctr, 2 * s * s)
            if k == 1:
                top = np.zeros((s, s), dtype=run.dt)
                c = beta.copy()
            else:
                tc = H(Om_prev) @ np.vstack([np.zeros((s, s), dtype=run.dt), beta])
                top, c = tc[:s], tc[s:]
            Om, Rii = unitary_qr_stack(np.vstack([c, rho_new]))
            tt = H(Om) @ np.vstack([tau_t, np.zeros((s, s), dtype=run.dt)])
            tau, tau_t = tt[:s], tt[s:]
            Rinv_rhs = np.eye(s, dtype=run.dt)
            Rii_inv = small_solve(Rii, Rinv_rhs)
            if k == 1:
                D = P @ Rii_inv
                F = AP @ Rii_inv
            else:
                D = (P - D @ top) @ Rii_inv
                F = (AP - F @ top) @ Rii_inv
            X = X + D @ tau
            R = R - F @ tau
            saxpy_count(ctr, 4 * s * s)
            if trace is not None:   # Lanczos blocks for the brute-force quasi-minimisation pin
                trace.append(dict(V=V, W=W, P=P, beta=beta, rho_next=rho_new, rho0=None, X=X.copy()))
            V, W, rho, xi, Om_prev = V_new, W_new, rho_new, xi_new, Om
            if run.step_done(k, X, np.sqrt(fro2(R, order)), R,
                             dict(beta=beta, rho=rho_new.copy(), tau_t=np.sqrt(fro2(tau_t)))):
                break
            if pending is not None:
                raise pending
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


# =============================================================================
# BiCGStab family (van der Vorst two-stage form, shadow
# R̃ = R0 fixed, half-step exit on ‖S‖_F)
# =============================================================================

@_quiet
def li_bicgstab(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Li-BiCGStab: s BiCGStabs in lockstep, per-column α_i, ω_i, β_i."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    Rt = _shadow_block(run, shadow)
    P = R.copy()
    frozen = np.zeros(s, dtype=bool)
    rho = col_inner(R, Rt, None, order)
    for k in range(1, maxit + 1):
        V = run.matA(P)
        alpha, newly = _safe_div(rho, col_inner(V, Rt, ctr, order), frozen)
        frozen |= newly
        S = R - V * alpha[None, :]
        saxpy_count(ctr, s)
        snorm = np.sqrt(fro2(S, order))
        if run.r0norm > 0 and snorm / run.r0norm <= tol:
            Xh = X + P * alpha[None, :]
            if run.true_rel(Xh) <= tol:
                X = Xh
                run.res.half_step = True
                run.res.outcome = "converged"
                run.step_done(k, X, snorm, S, dict(alpha=alpha.copy()))
                break
        T = run.matA(S)
        omega, newly = _safe_div(col_inner(S, T, ctr, order), col_inner(T, T, ctr, order), frozen)
        frozen |= newly
        X = X + P * alpha[None, :] + S * omega[None, :]
        R = S - T * omega[None, :]
        saxpy_count(ctr, 3 * s)
        rho_new = col_inner(R, Rt, ctr, order)
        beta, newly = _safe_div(rho_new * alpha, rho * omega, frozen)
        frozen |= newly
        P = R + (P - V * omega[None, :]) * beta[None, :]
        saxpy_count(ctr, 2 * s)
        rho = rho_new
        run.res.breakdown_cols = [int(i) for i in np.nonzero(frozen)[0]]
        if frozen.all():
            return run.breakdown(X, Breakdown("lanczos"), k)
        if run.step_done(k, X, np.sqrt(fro2(R, order)), R,
                         dict(alpha=alpha.copy(), omega=omega.copy(), beta=beta.copy())):
            break
    return run.finish(X)


@_quiet
def gl_bicgstab(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Gl-BiCGStab [Jbilou05]: BiCGStab on (I⊗A) with traces."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    Rt = _shadow_block(run, shadow)
    P = R.copy()
    rho = trace_inner(R, Rt, None, order)        # tr(R̃^H R)
    k = 0
    try:
        for k in range(1, maxit + 1):
            V = run.matA(P)
            alpha = _scalar_div(rho, trace_inner(V, Rt, ctr, order), "lanczos")
            S = R - alpha * V
            saxpy_count(ctr, s)
            snorm = np.sqrt(fro2(S, order))
            if snorm / run.r0norm <= tol:
                Xh = X + alpha * P
                if run.true_rel(Xh) <= tol:
                    X = Xh
                    run.res.half_step = True
                    run.res.outcome = "converged"
                    run.step_done(k, X, snorm, S, dict(alpha=alpha))
                    break
            T = run.matA(S)
            omega = _scalar_div(trace_inner(S, T, ctr, order), trace_inner(T, T, ctr, order), "omega")
            X = X + alpha * P + omega * S
            R = S - omega * T
            saxpy_count(ctr, 3 * s)
            rho_new = trace_inner(R, Rt, ctr, order)
            beta = _scalar_div(rho_new * alpha, rho * omega, "lanczos")
            P = R + beta * (P - omega * V)
            saxpy_count(ctr, 2 * s)
            rho = rho_new
            if run.step_done(k, X, np.sqrt(fro2(R, order)), R, dict(alpha=alpha, omega=omega, beta=beta)):
                break
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


@_quiet
def bl_bicgstab(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas"):
    """Bl-BiCGStab [ELg03]: s x s α, β and a scalar ω, the "global
    steepest descent" step. Step list SURVEY App. A.4 (reading G14)."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    R = run.R0.copy()
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    Rt = _shadow_block(run, shadow)
    P = R.copy()
    k = 0
    try:
        for k in range(1, maxit + 1):
            U = run.matA(P)
            G = gram(Rt, U, ctr, order)                  # R̃^H U
            alpha = small_solve(G, gram(Rt, R, ctr, order))
            S = R - U @ alpha
            saxpy_count(ctr, s * s)
            snorm = np.sqrt(fro2(S, order))
            if snorm / run.r0norm <= tol:
                Xh = X + P @ alpha
                if run.true_rel(Xh) <= tol:
                    X = Xh
                    run.res.half_step = True
                    run.res.outcome = "converged"
                    run.step_done(k, X, snorm, S, dict(alpha=alpha))
                    break
            T = run.matA(S)
            omega = _scalar_div(trace_inner(S, T, ctr, order), trace_inner(T, T, ctr, order), "omega")
            X = X + P @ alpha + omega * S
            R = S - omega * T
            saxpy_count(ctr, s * s + 2 * s)
            beta = -small_solve(G, gram(Rt, T, ctr, order))
            P = R + (P - omega * U) @ beta
            saxpy_count(ctr, s * s + s)
            if run.step_done(k, X, np.sqrt(fro2(R, order)), R, dict(alpha=alpha, omega=omega, beta=beta)):
                break
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


@_quiet
def bl_bicgstab_rq(A, B, tol=1e-8, maxit=2000, X0=None, shadow=None, record=20, order="blas", deflate=False):
    """Bl-BiCGStab-rQ ("we do not write down the resulting algorithm"):
    SURVEY App. A.5 (reading G16): R = Qr C kept factored, P = V C, one thin QR
    per iteration, ω through M = C C^H, residual monitored by ‖C‖_F.
    deflate=True: rank-deficiency continuation (f4), as in bl_bicg_rq."""
    run = _Run(A, B, X0, tol, maxit, record, order)
    ctr, s = run.ctr, run.B.shape[1]
    X = run.X
    if run.r0norm == 0:
        run.res.outcome = "converged"
        return run.finish(X)
    fill = _deflation_fill(run, deflate)
    k = 0
    try:
        Qr, C = thin_qr(run.R0, None, order, fill(0))
        Rt = _shadow_block(run, shadow)
        Q0h = Qr.copy() if (shadow is None or (isinstance(shadow, str) and shadow == "r0")) \
            else thin_qr(Rt, None, order, fill(1))[0]
        V = Qr.copy()
        GQ = gram(Q0h, Qr, None, order)
        c0 = np.sqrt(fro2(C))
        for k in range(1, maxit + 1):
            W = run.matA(V)
            G = gram(Q0h, W, ctr, order)
            alpha = small_solve(G, GQ)
            Z = Qr - W @ alpha
            saxpy_count(ctr, s * s)
            ZZ = gram(Z, Z, ctr, order)
            s2 = np.real(np.trace(H(C) @ ZZ @ C))
            if np.sqrt(max(s2, 0.0)) <= tol * c0:
                Xh = X + V @ (alpha @ C)
                if run.true_rel(Xh) <= tol:
                    X = Xh
                    run.res.half_step = True
                    run.res.outcome = "converged"
                    run.step_done(k, X, np.sqrt(max(s2, 0.0)), C, dict(alpha=alpha))
                    break
            Y = run.matA(Z)
            M = C @ H(C)
            YZ = gram(Y, Z, ctr, order)
            YY = gram(Y, Y, ctr, order)
            omega = _scalar_div(np.trace(YZ @ M), np.trace(YY @ M), "omega")
            X = X + (V @ alpha + omega * Z) @ C
            Qr_new, Sig = thin_qr(Z - omega * Y, ctr, order, fill(2 * k))
            C = Sig @ C
            GQ_new = gram(Q0h, Qr_new, ctr, order)
            beta = small_solve(G, GQ_new) / omega
            V = Qr_new + (V - omega * W) @ beta
            saxpy_count(ctr, 3 * s * s + s)
            Qr, GQ = Qr_new, GQ_new
            if run.step_done(k, X, np.sqrt(fro2(C)), C, dict(alpha=alpha, omega=omega, beta=beta, C=C.copy())):
                break
    except Breakdown as e:
        return run.breakdown(X, e, k)
    return run.finish(X)


# QR of the search directions: the comparison variants the paper rejects
SQ_METHODS = ("bl_bicg_sq", "bl_bicgstab_sq")
SOLVERS = {name: globals()[name] for name in METHODS + SQ_METHODS}


def solve(method: str, A, B, **kw) -> Result:
    """Dispatch: oracle.solve('egl_bicg', A_scipy_csr, B, tol=..., maxit=...)."""
    return SOLVERS[method](A, B, **kw)
