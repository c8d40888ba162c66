"""paper_1504_04395_b200 — B200-native simultaneous short-recurrence Krylov
solvers for AX = B with s right-hand sides (arXiv:1504.04395).

Thin Python binding over the C-ABI library libsrk.so (include/srk.h): argument
marshalling only. Every step of the path runs in the library's CUDA kernels;
PyTorch provides device memory and streams. There is no CPU fallback: if the
library or a CUDA device is missing, every call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_HERE, "libsrk.so")

METHODS = ("li_bicg", "gl_bicg", "egl_bicg", "bl_bicg", "bl_bicg_rq",
           "li_qmr", "gl_qmr", "egl_qmr", "bl_qmr",
           "li_bicgstab", "gl_bicgstab", "bl_bicgstab", "bl_bicgstab_rq",
           "bl_bicg_sq", "bl_bicgstab_sq")  # the last two: QR of the search directions (f3)
METHOD_ID = {m: i for i, m in enumerate(METHODS)}
NEEDS_ADJOINT = {m: ("bicgstab" not in m) for m in METHODS}
GRAM = {"none": 0, "norm2": 1, "diag": 2, "trace": 3, "sumvec": 4, "full": 5, "colnorm2": 6}
COEF = {"scalar": 1, "diag": 2, "full": 3}
OUTCOME = {0: "converged", 1: "maxit", 2: "breakdown", 3: "diverged"}
BREAKDOWN = {0: "", 1: "lanczos", 2: "gram", 3: "rank", 4: "nonfinite", 5: "omega"}
SRK_F64, SRK_C128 = 0, 1

EXPORTS = ("srk_create", "srk_destroy", "srk_last_error", "srk_version", "srk_matrix_create",
           "srk_matrix_destroy", "srk_matrix_adjoint", "srk_spmm_block", "srk_gram_block",
           "srk_block_update", "srk_tsqr", "srk_solve", "srk_solve_host", "srk_solver_create",
           "srk_solver_destroy", "srk_solver_start", "srk_solver_iterate", "srk_solver_get_x",
           "srk_solver_get_residual", "srk_solver_report", "srk_solver_history", "srk_solver_profile",
           "srk_solver_profile_read", "srk_solver_profile_launches", "srk_partition_rows", "srk_plan_create", "srk_plan_sizes", "srk_plan_arrays",
           "srk_plan_destroy", "srk_nccl_unique_id", "srk_comm_init", "srk_matrix_create_dist",
           "srk_vgroup_create", "srk_vgroup_destroy", "srk_comm_init_virtual", "srk_csr_adjoint_host",
           "srk_matrix_format", "srk_matrix_sell_info", "srk_matrix_set_row_order", "srk_matrix_create_bsr_dist",
           "srk_matrix_create_bsr", "srk_matrix_ilu0", "srk_matrix_ilu0_factor", "srk_precond_apply",
           "srk_matrix_ilutp", "srk_matrix_prec_info", "srk_matrix_ilutp_factor")


class SrkError(RuntimeError):
    pass


class _Csr(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col_idx", ctypes.c_void_p), ("values", ctypes.c_void_p), ("dtype", ctypes.c_int)]


class _Opts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("maxit", ctypes.c_int), ("poll_every", ctypes.c_int),
                ("record_history", ctypes.c_int), ("check_true_residual", ctypes.c_int),
                ("use_graph", ctypes.c_int), ("x0_zero", ctypes.c_int), ("shadow", ctypes.c_int),
                ("shadow_given", ctypes.c_void_p), ("preprocess_rhs", ctypes.c_int), ("eps_brk", ctypes.c_double),
                ("eps_defl", ctypes.c_double), ("rank_policy", ctypes.c_int), ("trace_iterates", ctypes.c_int),
                ("on_iter", ctypes.c_void_p), ("user", ctypes.c_void_p)]


# void on_iter(int k, const void* X_k, const void* R_or_C_k, int64_t r_rows, const double* scalars, void* user)
ON_ITER = ctypes.CFUNCTYPE(None, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                           ctypes.POINTER(ctypes.c_double), ctypes.c_void_p)


class _Halo(ctypes.Structure):
    _fields_ = [("recv_counts", ctypes.c_void_p), ("send_counts", ctypes.c_void_p), ("send_local", ctypes.c_void_p),
                ("n_send", ctypes.c_int64)]


class _Report(ctypes.Structure):
    _fields_ = [("outcome", ctypes.c_int), ("iterations", ctypes.c_int), ("half_step", ctypes.c_int),
                ("breakdown_kind", ctypes.c_int), ("breakdown_iter", ctypes.c_int), ("frozen_cols", ctypes.c_int),
                ("matvec_cols_A", ctypes.c_int64), ("matvec_cols_AH", ctypes.c_int64),
                ("final_true_rel_residual", ctypes.c_double), ("final_recursive_rel_residual", ctypes.c_double),
                ("seconds", ctypes.c_double), ("kernel_launches", ctypes.c_int64), ("vector_ops", ctypes.c_int64),
                ("breakdown_col", ctypes.c_int), ("deflated_cols", ctypes.c_int)]


_lib = None


def load_library(path: str | None = None):
    """Load libsrk.so (built in-tree by paper_1504_04395_b200.build). Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or _LIBPATH
    if not os.path.exists(p):
        raise SrkError(f"{p} not found: build it with `python -m paper_1504_04395_b200.build` "
                       "(there is no CPU fallback)")
    lib = ctypes.CDLL(p)
    vp, i, i64, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    sig = {
        "srk_create": ([ctypes.POINTER(vp), i, vp], i),
        "srk_destroy": ([vp], i),
        "srk_last_error": ([], ctypes.c_char_p),
        "srk_version": ([], i),
        "srk_matrix_create": ([vp, ctypes.POINTER(_Csr), i, ctypes.POINTER(vp)], i),
        "srk_matrix_create_bsr": ([vp, i64, i, i64, vp, vp, vp, i, i, ctypes.POINTER(vp)], i),
        "srk_matrix_destroy": ([vp], i),
        "srk_matrix_ilu0": ([vp], i),
        "srk_matrix_ilu0_factor": ([vp, vp], i),
        "srk_matrix_ilutp": ([vp, d, d], i),
        "srk_matrix_prec_info": ([vp, ctypes.POINTER(i), ctypes.POINTER(i64), ctypes.POINTER(i)], i),
        "srk_matrix_ilutp_factor": ([vp, vp, vp, vp, vp], i),
        "srk_precond_apply": ([vp, vp, i, vp, vp, i], i),
        "srk_matrix_adjoint": ([vp, vp, vp, vp], i),
        "srk_spmm_block": ([vp, vp, i, vp, vp, i, i, vp, vp], i),
        "srk_gram_block": ([vp, vp, vp, i64, i, i, i, vp], i),
        "srk_block_update": ([vp, vp, vp, vp, vp, i, i, i64, i, i], i),
        "srk_tsqr": ([vp, vp, vp, vp, i64, i, i, ctypes.POINTER(i)], i),
        "srk_solve": ([vp, vp, vp, vp, i, i, ctypes.POINTER(_Opts), ctypes.POINTER(_Report)], i),
        "srk_solve_host": ([vp, vp, vp, vp, i, i, ctypes.POINTER(_Opts), ctypes.POINTER(_Report)], i),
        "srk_solver_create": ([vp, vp, i, i, ctypes.POINTER(_Opts), ctypes.POINTER(vp)], i),
        "srk_solver_destroy": ([vp], i),
        "srk_solver_start": ([vp, vp, vp], i),
        "srk_solver_iterate": ([vp, i, ctypes.POINTER(i)], i),
        "srk_solver_get_x": ([vp, vp], i),
        "srk_solver_get_residual": ([vp, vp, ctypes.POINTER(i64)], i),
        "srk_solver_report": ([vp, ctypes.POINTER(_Report)], i),
        "srk_solver_history": ([vp, ctypes.POINTER(d), i], i),
        "srk_solver_profile": ([vp, i], i),
        "srk_solver_profile_read": ([vp, ctypes.POINTER(d), ctypes.POINTER(i64), i], i),
        "srk_solver_profile_launches": ([vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                         ctypes.POINTER(d), ctypes.POINTER(d), i], i),
        "srk_partition_rows": ([i64, vp, i, vp], i),
        "srk_plan_create": ([i64, vp, vp, i, vp, i, ctypes.POINTER(vp)], i),
        "srk_plan_sizes": ([vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)], i),
        "srk_plan_arrays": ([vp, vp, vp, vp, vp, vp, vp], i),
        "srk_plan_destroy": ([vp], i),
        "srk_nccl_unique_id": ([vp], i),
        "srk_comm_init": ([vp, vp, i, i], i),
        "srk_vgroup_create": ([i, ctypes.POINTER(vp)], i),
        "srk_matrix_format": ([vp, i, ctypes.POINTER(i)], i),
        "srk_matrix_sell_info": ([vp, i, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i)], i),
        "srk_matrix_set_row_order": ([vp, vp, i64], i),
        "srk_matrix_create_bsr_dist": ([vp, i64, i, i64, vp, vp, vp, i, i, i64, ctypes.POINTER(_Halo),
                                        ctypes.POINTER(vp)], i),
        "srk_vgroup_destroy": ([vp], i),
        "srk_comm_init_virtual": ([vp, vp, i], i),
        "srk_csr_adjoint_host": ([i64, vp, vp, vp, i, vp, vp, vp], i),
        "srk_matrix_create_dist": ([vp, ctypes.POINTER(_Csr), i64, ctypes.POINTER(_Halo), ctypes.POINTER(_Csr), i64,
                                    ctypes.POINTER(_Halo)], i),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = _lib.srk_last_error().decode() if _lib else ""
        raise SrkError(f"{what} failed ({rc}): {msg}")


def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float64:
        return SRK_F64
    if t.dtype == torch.complex128:
        return SRK_C128
    raise SrkError(f"unsupported dtype {t.dtype}: float64 or complex128 required")


def _dev(t, name):
    if not t.is_cuda:
        raise SrkError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise SrkError(f"{name} must be contiguous (row-major n x s)")
    return ctypes.c_void_p(t.data_ptr())


class Context:
    """srk_ctx bound to the current CUDA device and torch's current stream."""

    def __init__(self, device: int | None = None, stream=None):
        torch = _torch()
        lib = load_library()
        if not torch.cuda.is_available():
            raise SrkError("CUDA is not available: the srk path has no CPU fallback")
        dev = torch.cuda.current_device() if device is None else device
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        self.stream = st
        self.device = dev
        h = ctypes.c_void_p()
        _check(lib.srk_create(ctypes.byref(h), dev, ctypes.c_void_p(st.cuda_stream)), "srk_create")
        self.h = h

    def close(self):
        if self.h:
            _lib.srk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context()
    return _default_ctx


class Matrix:
    """srk_matrix (a0): validated device CSR copy (+ explicit A^H when needed)."""

    def __init__(self, row_ptr, col_idx, values, need_adjoint: bool = True, ctx: Context | None = None):
        torch = _torch()
        self.ctx = ctx or default_context()
        dev = torch.device("cuda", self.ctx.device)
        rp = torch.as_tensor(row_ptr).to(dev, torch.int64).contiguous()
        ci = torch.as_tensor(col_idx).to(dev, torch.int32).contiguous()
        va = torch.as_tensor(values).to(dev).contiguous()
        if va.dtype not in (torch.float64, torch.complex128):
            va = va.to(torch.float64)
        self.n = rp.numel() - 1
        self.nnz = ci.numel()
        self.dtype = va.dtype
        csr = _Csr(self.n, self.nnz, rp.data_ptr(), ci.data_ptr(), va.data_ptr(), _dtype_code(va))
        h = ctypes.c_void_p()
        _check(_lib.srk_matrix_create(self.ctx.h, ctypes.byref(csr), int(need_adjoint), ctypes.byref(h)),
               "srk_matrix_create")
        self.h = h
        self.has_adjoint = need_adjoint

    @classmethod
    def from_csr(cls, A, need_adjoint=True, ctx=None):
        """From a synth.CSR / scipy.sparse.csr_matrix / (row_ptr, col_idx, values) triple."""
        if isinstance(A, tuple):
            return cls(*A, need_adjoint=need_adjoint, ctx=ctx)
        if hasattr(A, "indptr"):
            return cls(A.indptr, A.indices, A.data, need_adjoint=need_adjoint, ctx=ctx)
        return cls(A.row_ptr, A.col_idx, A.values, need_adjoint=need_adjoint, ctx=ctx)

    @classmethod
    def from_bsr(cls, block_row_ptr, block_col, blocks, unit_diag: bool = False, ctx=None):
        """Block-sparse operator (srk_matrix_create_bsr): blocks (nnzb, 12, 12) complex
        row-major; unit_diag: identity diagonal blocks implied, not stored."""
        torch = _torch()
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        dev = torch.device("cuda", self.ctx.device)
        rp = torch.as_tensor(np.asarray(block_row_ptr)).to(dev, torch.int64).contiguous()
        ci = torch.as_tensor(np.asarray(block_col)).to(dev, torch.int32).contiguous()
        va = blocks if isinstance(blocks, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(blocks))
        va = va.to(dev, torch.complex128).contiguous()
        nb = rp.numel() - 1
        bs = int(va.shape[-1]) if va.dim() == 3 else 12
        self.n = nb * bs
        self.nnz = ci.numel() * bs * bs + (self.n if unit_diag else 0)
        self.dtype = torch.complex128
        h = ctypes.c_void_p()
        _check(_lib.srk_matrix_create_bsr(self.ctx.h, nb, bs, ci.numel(), ctypes.c_void_p(rp.data_ptr()),
                                          ctypes.c_void_p(ci.data_ptr()), ctypes.c_void_p(va.data_ptr()),
                                          _dtype_code(va), int(unit_diag), ctypes.byref(h)), "srk_matrix_create_bsr")
        self.h = h
        self.has_adjoint = False
        return self

    FORMATS = ("csr", "csr_sorted", "band", "bsr")

    def format(self, adjoint: bool = False):
        """(storage, diagonals) the SpMM of A (or A^H) uses (srk_matrix_format)."""
        nd = ctypes.c_int(0)
        f = _lib.srk_matrix_format(self.h, int(adjoint), ctypes.byref(nd))
        _check(min(f, 0), "srk_matrix_format")
        return self.FORMATS[f], nd.value

    def set_row_order(self, order=None):
        """Visiting order of a block-sparse operator's block rows (srk_matrix_set_row_order):
        a host int32 permutation, or None for the natural order; returns self."""
        if order is None:
            _check(_lib.srk_matrix_set_row_order(self.h, None, 0), "srk_matrix_set_row_order")
            return self
        o = np.ascontiguousarray(order, dtype=np.int32)
        _check(_lib.srk_matrix_set_row_order(self.h, o.ctypes.data_as(ctypes.c_void_p), o.size), "srk_matrix_set_row_order")
        return self

    def sell_info(self, adjoint: bool = False):
        """None, or (chunks, stored entries incl. padding, sigma) of the SELL-32-sigma form
        narrow products of A (or A^H) use (srk_matrix_sell_info)."""
        nc, ne, sg = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int(0)
        f = _lib.srk_matrix_sell_info(self.h, int(adjoint), ctypes.byref(nc), ctypes.byref(ne), ctypes.byref(sg))
        _check(min(f, 0), "srk_matrix_sell_info")
        return (nc.value, ne.value, sg.value) if f == 1 else None

    def ilu0(self):
        """Attach the right ILU(0) preconditioner (srk_matrix_ilu0); returns self."""
        _check(_lib.srk_matrix_ilu0(self.h), "srk_matrix_ilu0")
        self.preconditioned = True
        return self

    def ilutp(self, droptol: float = 5e-2, thresh: float = 1.0):
        """Attach the right ILUTP preconditioner (srk_matrix_ilutp, reading R14):
        threshold ILU with partial pivoting, M = Pi^T L U; returns self."""
        _check(_lib.srk_matrix_ilutp(self.h, float(droptol), float(thresh)), "srk_matrix_ilutp")
        self.preconditioned = True
        return self

    def prec_info(self):
        """(kind: 'ilu0' | 'ilutp', nnz of the factor, pivoted)"""
        k, nz, pv = ctypes.c_int(0), ctypes.c_int64(0), ctypes.c_int(0)
        _check(_lib.srk_matrix_prec_info(self.h, ctypes.byref(k), ctypes.byref(nz), ctypes.byref(pv)),
               "srk_matrix_prec_info")
        return ("ilu0", "ilutp")[k.value], nz.value, bool(pv.value)

    def ilutp_factor(self):
        """(L, U, perm) of the attached ILUTP as scipy CSR (pivot order; host copy):
        A[perm] ~ L @ U."""
        import scipy.sparse as sp
        torch = _torch()
        cplx = self.dtype == torch.complex128
        _, nz, _ = self.prec_info()
        rp = np.empty(self.n + 1, dtype=np.int64)
        ci = np.empty(max(nz, 1), dtype=np.int32)
        va = np.empty(max(nz, 1), dtype=np.complex128 if cplx else np.float64)
        perm = np.empty(self.n, dtype=np.int64)
        _check(_lib.srk_matrix_ilutp_factor(self.h, rp.ctypes.data_as(ctypes.c_void_p), ci.ctypes.data_as(ctypes.c_void_p),
                                            va.ctypes.data_as(ctypes.c_void_p), perm.ctypes.data_as(ctypes.c_void_p)),
               "srk_matrix_ilutp_factor")
        F = sp.csr_matrix((va[:nz], ci[:nz], rp), shape=(self.n, self.n))
        L = sp.tril(F, k=-1, format="csr") + sp.identity(self.n, dtype=va.dtype, format="csr")
        U = sp.triu(F, k=0, format="csr")
        L.sort_indices()
        U.sort_indices()
        return L, U, perm

    def ilu0_factor(self) -> np.ndarray:
        """The ILU(0) factor values on the operator's pattern (host copy)."""
        torch = _torch()
        cplx = self.dtype == torch.complex128
        out = np.empty(self.nnz, dtype=np.complex128 if cplx else np.float64)
        _check(_lib.srk_matrix_ilu0_factor(self.h, out.ctypes.data_as(ctypes.c_void_p)), "srk_matrix_ilu0_factor")
        return out

    def adjoint_csr(self):
        torch = _torch()
        dev = torch.device("cuda", self.ctx.device)
        rp = torch.empty(self.n + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(self.nnz, dtype=torch.int32, device=dev)
        va = torch.empty(self.nnz, dtype=self.dtype, device=dev)
        _check(_lib.srk_matrix_adjoint(self.h, ctypes.c_void_p(rp.data_ptr()), ctypes.c_void_p(ci.data_ptr()),
                                       ctypes.c_void_p(va.data_ptr())), "srk_matrix_adjoint")
        return rp, ci, va

    def close(self):
        if getattr(self, "h", None):
            _lib.srk_matrix_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ multi-GPU
def _np_ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def partition_rows(row_ptr, nranks: int) -> np.ndarray:
    """Contiguous row ranges balanced by nnz (host; srk_partition_rows)."""
    lib = load_library()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    off = np.zeros(nranks + 1, dtype=np.int64)
    _check(lib.srk_partition_rows(rp.size - 1, _np_ptr(rp), nranks, _np_ptr(off)), "srk_partition_rows")
    return off


@dataclass
class Plan:
    """Halo plan of one rank (srk_plan_*): local CSR pattern, ghosts, send lists."""
    n_local: int
    row_ptr: np.ndarray
    col: np.ndarray
    ghosts: np.ndarray
    recv_counts: np.ndarray
    send_counts: np.ndarray
    send_local: np.ndarray
    off0: int
    off1: int


def make_plan(row_ptr, col_idx, offsets, rank: int) -> Plan:
    lib = load_library()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    nr = off.size - 1
    h = ctypes.c_void_p()
    _check(lib.srk_plan_create(rp.size - 1, _np_ptr(rp), _np_ptr(ci), nr, _np_ptr(off), rank, ctypes.byref(h)),
           "srk_plan_create")
    try:
        nl, nz, ng, ns = (ctypes.c_int64() for _ in range(4))
        _check(lib.srk_plan_sizes(h, ctypes.byref(nl), ctypes.byref(nz), ctypes.byref(ng), ctypes.byref(ns)),
               "srk_plan_sizes")
        prl = np.zeros(nl.value + 1, np.int64)
        col = np.zeros(max(nz.value, 1), np.int32)
        gh = np.zeros(max(ng.value, 1), np.int64)
        rc = np.zeros(nr, np.int32)
        sc = np.zeros(nr, np.int32)
        sl = np.zeros(max(ns.value, 1), np.int32)
        _check(lib.srk_plan_arrays(h, _np_ptr(prl), _np_ptr(col), _np_ptr(gh), _np_ptr(rc), _np_ptr(sc), _np_ptr(sl)),
               "srk_plan_arrays")
    finally:
        lib.srk_plan_destroy(h)
    return Plan(nl.value, prl, col[:nz.value], gh[:ng.value], rc, sc, sl[:ns.value], int(off[rank]),
                int(off[rank + 1]))


def init_distributed(ctx: "Context | None" = None):
    """Create the context's NCCL communicator over the torch.distributed world
    (one process per GPU): rank 0 draws the unique id, broadcast as bytes."""
    import torch.distributed as dist
    ctx = ctx or default_context()
    world, rank = dist.get_world_size(), dist.get_rank()
    buf = (ctypes.c_char * 128)()
    if rank == 0:
        _check(_lib.srk_nccl_unique_id(buf), "srk_nccl_unique_id")
    obj = [bytes(buf)]
    dist.broadcast_object_list(obj, src=0)
    ctypes.memmove(buf, obj[0], 128)
    _check(_lib.srk_comm_init(ctx.h, buf, world, rank), "srk_comm_init")
    return ctx


class VirtualGroup:
    """srk_vgroup: k virtual ranks of a row-partitioned operator on ONE GPU.
    Each rank gets its own Context (own stream) attached with `attach`, and its own host
    thread that makes the same sequence of library calls as the others (collectives are
    rendezvous points); the transport is device-to-device, reductions in rank order."""

    def __init__(self, k: int):
        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.srk_vgroup_create(k, ctypes.byref(h)), "srk_vgroup_create")
        self.h = h
        self.k = k

    def attach(self, ctx: "Context", rank: int) -> "Context":
        _check(_lib.srk_comm_init_virtual(ctx.h, self.h, rank), "srk_comm_init_virtual")
        return ctx

    def close(self):
        if getattr(self, "h", None):
            _lib.srk_vgroup_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def csr_adjoint_host(row_ptr, col_idx, values):
    """A^H = conj(A)^T of a host CSR, computed by the library (srk_csr_adjoint_host)."""
    lib = load_library()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    va = np.ascontiguousarray(values)
    if va.dtype not in (np.float64, np.complex128):
        raise SrkError("values must be float64 or complex128")
    n = rp.size - 1
    rpT = np.zeros(n + 1, np.int64)
    ciT = np.zeros(max(ci.size, 1), np.int32)
    vaT = np.zeros(max(va.size, 1), va.dtype)
    dt = SRK_C128 if va.dtype == np.complex128 else SRK_F64
    _check(lib.srk_csr_adjoint_host(n, _np_ptr(rp), _np_ptr(ci), _np_ptr(va), dt, _np_ptr(rpT), _np_ptr(ciT),
                                    _np_ptr(vaT)), "srk_csr_adjoint_host")
    return rpT, ciT[:ci.size], vaT[:va.size]


class DistMatrix:
    """srk_matrix_create_dist: this rank's rows of A (and of A^H) with halo plans."""

    def __init__(self, A, offsets, rank: int, need_adjoint: bool = True, ctx: "Context | None" = None):
        torch = _torch()
        self.ctx = ctx or default_context()
        dev = torch.device("cuda", self.ctx.device)
        if hasattr(A, "indptr"):
            rp, ci, va, n = A.indptr, A.indices, A.data, A.shape[0]
        else:
            rp, ci, va, n = A.row_ptr, A.col_idx, A.values, A.n
        self.offsets = np.asarray(offsets, np.int64)
        self.rank = rank
        self.plan = make_plan(rp, ci, self.offsets, rank)
        self.n_local = self.plan.n_local
        self.n_ghost = self.plan.ghosts.size
        self.dtype = torch.from_numpy(np.asarray(va[:1])).dtype
        keep = []

        def csr_struct(plan, vals):
            t_rp = torch.from_numpy(plan.row_ptr).to(dev)
            t_ci = torch.from_numpy(plan.col).to(dev)
            t_va = torch.from_numpy(np.ascontiguousarray(vals)).to(dev)
            keep.extend([t_rp, t_ci, t_va])
            return _Csr(plan.n_local, plan.col.size, t_rp.data_ptr(), t_ci.data_ptr(), t_va.data_ptr(),
                        _dtype_code(t_va))

        def halo_struct(plan):
            keep.extend([plan.recv_counts, plan.send_counts, plan.send_local])
            return _Halo(plan.recv_counts.ctypes.data, plan.send_counts.ctypes.data,
                         plan.send_local.ctypes.data if plan.send_local.size else None, plan.send_local.size)

        lo, hi = int(rp[self.plan.off0]), int(rp[self.plan.off1])
        csrA = csr_struct(self.plan, va[lo:hi])
        haloA = halo_struct(self.plan)
        csrH = haloH = None
        ngH = 0
        if need_adjoint:
            rpH, ciH, vaH = csr_adjoint_host(rp, ci, va)   # a0 inside the library
            self.planH = make_plan(rpH, ciH, self.offsets, rank)
            lo, hi = int(rpH[self.planH.off0]), int(rpH[self.planH.off1])
            csrH = csr_struct(self.planH, vaH[lo:hi])
            haloH = halo_struct(self.planH)
            ngH = self.planH.ghosts.size
        h = ctypes.c_void_p()
        _check(_lib.srk_matrix_create_dist(self.ctx.h, ctypes.byref(csrA), self.n_ghost, ctypes.byref(haloA),
                                           ctypes.byref(csrH) if csrH else None, ngH,
                                           ctypes.byref(haloH) if haloH else None, ctypes.byref(h)),
               "srk_matrix_create_dist")
        torch.cuda.synchronize()
        self.h = h
        self.n = self.n_local
        self.has_adjoint = need_adjoint

    @classmethod
    def from_bsr(cls, block_row_ptr, block_col, blocks, offsets_blocks, rank: int, unit_diag: bool = True,
                 ctx: "Context | None" = None):
        """srk_matrix_create_bsr_dist: this rank's block rows of a BSR-12 operator (config 4's
        lattice as t-slabs when the offsets split the lexicographic site order), planned on the
        block-row CSR pattern by the library's planner; the halo moves 12 rows per ghost block."""
        torch = _torch()
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        dev = torch.device("cuda", self.ctx.device)
        brp = np.ascontiguousarray(block_row_ptr, np.int64)
        bci = np.ascontiguousarray(block_col, np.int32)
        self.offsets = np.asarray(offsets_blocks, np.int64)
        self.rank = rank
        self.plan = make_plan(brp, bci, self.offsets, rank)
        nb_local, bs = self.plan.n_local, 12
        lo, hi = int(brp[self.plan.off0]), int(brp[self.plan.off1])
        t_rp = torch.from_numpy(self.plan.row_ptr).to(dev)
        t_ci = torch.from_numpy(self.plan.col).to(dev)
        t_bv = torch.from_numpy(np.ascontiguousarray(blocks[lo:hi])).to(dev)
        keep = [self.plan.recv_counts, self.plan.send_counts, self.plan.send_local]
        halo = _Halo(self.plan.recv_counts.ctypes.data, self.plan.send_counts.ctypes.data,
                     self.plan.send_local.ctypes.data if self.plan.send_local.size else None, self.plan.send_local.size)
        h = ctypes.c_void_p()
        _check(_lib.srk_matrix_create_bsr_dist(self.ctx.h, nb_local, bs, hi - lo, ctypes.c_void_p(t_rp.data_ptr()),
                                               ctypes.c_void_p(t_ci.data_ptr()), ctypes.c_void_p(t_bv.data_ptr()),
                                               SRK_C128, int(unit_diag), self.plan.ghosts.size, ctypes.byref(halo),
                                               ctypes.byref(h)), "srk_matrix_create_bsr_dist")
        torch.cuda.synchronize()
        del keep
        self.h = h
        self.n_local = nb_local * bs
        self.n = self.n_local
        self.n_ghost = self.plan.ghosts.size * bs
        self.has_adjoint = False
        return self

    def close(self):
        if getattr(self, "h", None):
            _lib.srk_matrix_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _gram_shape(mode: str, s: int, cplx: bool):
    torch = _torch()
    dt = torch.complex128 if cplx else torch.float64
    if mode == "norm2":
        return (1,), torch.float64
    if mode == "colnorm2":
        return (s,), torch.float64
    if mode == "diag":
        return (s,), dt
    if mode in ("trace", "sumvec"):
        return (1,), dt
    if mode == "full":
        return (s, s), dt
    raise SrkError(mode)


def spmm_block(A: Matrix, P, adjoint: bool = False, gram: str = "none", Y=None, Q=None):
    """Q = op(A) P (+ fused reduction between Q and Y). Returns Q or (Q, gram)."""
    torch = _torch()
    n, s = P.shape if P.dim() == 2 else (P.shape[0], 1)
    if Q is None:
        Q = torch.empty_like(P)
    out = None
    if gram != "none":
        shp, dt = _gram_shape(gram, s, P.is_complex())
        out = torch.empty(shp, dtype=dt, device=P.device)
    _check(_lib.srk_spmm_block(A.ctx.h, A.h, int(adjoint), _dev(P, "P"), _dev(Q, "Q"), s, GRAM[gram],
                               _dev(Y, "Y") if Y is not None else None,
                               ctypes.c_void_p(out.data_ptr()) if out is not None else None), "srk_spmm_block")
    return Q if out is None else (Q, out)


def precond_apply(A: Matrix, P, adjoint: bool = False):
    """Z = M^-1 P (or M^-H P) with the operator's ILU(0) (srk_precond_apply)."""
    torch = _torch()
    Z = torch.empty_like(P)
    s = P.shape[1] if P.dim() == 2 else 1
    _check(_lib.srk_precond_apply(A.ctx.h, A.h, int(adjoint), _dev(P, "P"), _dev(Z, "Z"), s), "srk_precond_apply")
    return Z


def gram_block(X, Y=None, mode: str = "full", ctx: Context | None = None):
    """Reduction between blocks X and Y (FULL: Y^H X)."""
    torch = _torch()
    ctx = ctx or default_context()
    n = X.shape[0]
    s = X.shape[1] if X.dim() == 2 else 1
    shp, dt = _gram_shape(mode, s, X.is_complex())
    out = torch.empty(shp, dtype=dt, device=X.device)
    _check(_lib.srk_gram_block(ctx.h, _dev(X, "X"), _dev(Y, "Y") if Y is not None else None, n, s,
                               _dtype_code(X), GRAM[mode], ctypes.c_void_p(out.data_ptr())), "srk_gram_block")
    return out


def block_update(Yin, X, coef, kind: str = "full", sign: int = 1, Yout=None, ctx: Context | None = None):
    """Yout = Yin + sign * X * coef (coef scalar / s-vector / s x s, device tensor)."""
    torch = _torch()
    ctx = ctx or default_context()
    if Yout is None:
        Yout = torch.empty_like(Yin)
    coef = torch.as_tensor(coef, device=Yin.device, dtype=Yin.dtype).contiguous()
    n, s = Yin.shape
    _check(_lib.srk_block_update(ctx.h, _dev(Yout, "Yout"), _dev(Yin, "Yin"), _dev(X, "X"), _dev(coef, "coef"),
                                 COEF[kind], int(sign), n, s, _dtype_code(Yin)), "srk_block_update")
    return Yout


def tsqr(Z, ctx: Context | None = None):
    """Thin QR Z = Q C (CholQR2). Returns (Q, C, rank)."""
    torch = _torch()
    ctx = ctx or default_context()
    n, s = Z.shape
    Q = torch.empty_like(Z)
    C = torch.empty((s, s), dtype=Z.dtype, device=Z.device)
    rank = ctypes.c_int(0)
    _check(_lib.srk_tsqr(ctx.h, _dev(Z, "Z"), _dev(Q, "Q"), ctypes.c_void_p(C.data_ptr()), n, s, _dtype_code(Z),
                         ctypes.byref(rank)), "srk_tsqr")
    return Q, C, rank.value


@dataclass
class Report:
    outcome: str
    iterations: int
    half_step: bool
    breakdown_kind: str
    breakdown_iter: int
    frozen_cols: int
    matvec_cols_A: int
    matvec_cols_AH: int
    final_true_rel_residual: float
    final_recursive_rel_residual: float
    seconds: float
    kernel_launches: int
    vector_ops: int = 0
    breakdown_col: int = -1
    deflated_cols: int = 0


def _report(r: _Report) -> Report:
    return Report(OUTCOME.get(r.outcome, str(r.outcome)), r.iterations, bool(r.half_step),
                  BREAKDOWN.get(r.breakdown_kind, str(r.breakdown_kind)), r.breakdown_iter, r.frozen_cols,
                  r.matvec_cols_A, r.matvec_cols_AH, r.final_true_rel_residual, r.final_recursive_rel_residual,
                  r.seconds, r.kernel_launches, r.vector_ops, r.breakdown_col, r.deflated_cols)


SHADOW = {"default": 0, "conj": 1, "mean": 2, "given": 3}


class _DevView:
    """A raw device pointer as a CUDA array (torch.as_tensor reads __cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2, "strides": None}


def _opts(tol, maxit, poll_every=8, check_true_residual=True, use_graph=True, x0_zero=False, shadow="default",
          shadow_given=None, preprocess_rhs=False, eps_brk=0.0, eps_defl=0.0, rank_policy="breakdown"):
    """srk_opts. rank_policy: "breakdown" (reading G11) or "continue" (f4, the rQ variants)."""
    if rank_policy not in ("breakdown", "continue"):
        raise SrkError(f"rank_policy must be 'breakdown' or 'continue', not {rank_policy!r}")
    if shadow not in SHADOW:
        raise SrkError(f"shadow must be one of {sorted(SHADOW)}")
    if (shadow == "given") != (shadow_given is not None):
        raise SrkError("shadow='given' needs shadow_given (and only then)")
    sg = _dev(shadow_given, "shadow_given") if shadow_given is not None else None
    return _Opts(float(tol), int(maxit), int(poll_every), 1, int(check_true_residual), int(use_graph), int(x0_zero),
                 SHADOW[shadow], sg, int(preprocess_rhs), float(eps_brk), float(eps_defl),
                 1 if rank_policy == "continue" else 0)


class Solver:
    """Stepping interface (srk_solver_*): lock-step parity and benchmarking."""

    def __init__(self, A: Matrix, s: int, method: str, tol: float = 1e-8, maxit: int = 2000, poll_every: int = 8,
                 check_true_residual: bool = True, use_graph: bool = True, **opts):
        if method not in METHOD_ID:
            raise SrkError(f"unknown method {method}")
        self.A, self.s, self.method = A, s, method
        o = _opts(tol, maxit, poll_every, check_true_residual, use_graph, **opts)
        self._shadow = opts.get("shadow_given")
        h = ctypes.c_void_p()
        _check(_lib.srk_solver_create(A.ctx.h, A.h, s, METHOD_ID[method], ctypes.byref(o), ctypes.byref(h)),
               "srk_solver_create")
        self.h = h

    def start(self, B, X0=None):
        self._B = B
        _check(_lib.srk_solver_start(self.h, _dev(B, "B"), _dev(X0, "X0") if X0 is not None else None),
               "srk_solver_start")

    def iterate(self, k: int) -> int:
        st = ctypes.c_int(0)
        _check(_lib.srk_solver_iterate(self.h, int(k), ctypes.byref(st)), "srk_solver_iterate")
        return st.value

    def x(self):
        X = _torch().empty_like(self._B)
        _check(_lib.srk_solver_get_x(self.h, _dev(X, "X")), "srk_solver_get_x")
        return X

    def residual(self):
        torch = _torch()
        n = self._B.shape[0]
        buf = torch.empty((max(n, self.s), self.s), dtype=self._B.dtype, device=self._B.device)
        rows = ctypes.c_int64(0)
        _check(_lib.srk_solver_get_residual(self.h, _dev(buf, "out"), ctypes.byref(rows)), "srk_solver_get_residual")
        return buf[: rows.value].clone()

    def report(self) -> Report:
        r = _Report()
        _check(_lib.srk_solver_report(self.h, ctypes.byref(r)), "srk_solver_report")
        return _report(r)

    def history(self, k: int) -> np.ndarray:
        buf = (ctypes.c_double * max(k, 1))()
        _check(_lib.srk_solver_history(self.h, buf, k), "srk_solver_history")
        return np.array(buf[:k])

    PROFILE_TAGS = ("spmm", "spmm_adj", "update", "finalize", "coef")

    def profile(self, enable: bool = True):
        _check(_lib.srk_solver_profile(self.h, int(enable)), "srk_solver_profile")

    def profile_read(self) -> dict:
        n = len(self.PROFILE_TAGS)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        _check(_lib.srk_solver_profile_read(self.h, ms, cnt, n), "srk_solver_profile_read")
        return {t: (ms[i], cnt[i]) for i, t in enumerate(self.PROFILE_TAGS)}

    def profile_launches(self, max_records: int = 1 << 16) -> list:
        """Per-launch records [(tag, signature, ms, algorithmic_bytes)] since the last read."""
        t = (ctypes.c_int32 * max_records)()
        g = (ctypes.c_int32 * max_records)()
        ms = (ctypes.c_double * max_records)()
        nb = (ctypes.c_double * max_records)()
        k = _lib.srk_solver_profile_launches(self.h, t, g, ms, nb, max_records)
        _check(min(k, 0), "srk_solver_profile_launches")
        return [(self.PROFILE_TAGS[t[i]] if t[i] < len(self.PROFILE_TAGS) else "other", g[i], ms[i], nb[i])
                for i in range(k)]

    def close(self):
        if getattr(self, "h", None):
            _lib.srk_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve(A: Matrix, B, method: str = "egl_bicg", tol: float = 1e-8, maxit: int = 2000, X0=None,
          poll_every: int = 8, trace_iterates: int = 0, on_iter=None, **opts):
    """X, report = solve(A, B, method, tol, maxit, **opts) — srk_solve on device tensors
    (B: contiguous (n, s) float64/complex128 CUDA tensor). opts: shadow ("default",
    "conj", "mean", "given" + shadow_given), preprocess_rhs, eps_brk, eps_defl,
    rank_policy ("breakdown" / "continue"). trace_iterates = K with on_iter(k, X_k, R_or_C_k,
    rel_residual, state): the library's iteration callback (srk_opts.on_iter) for the first K
    iterations; X_k / R_or_C_k are CUDA tensors (copies made here, valid after the call)."""
    torch = _torch()
    n, s = B.shape
    X = torch.empty_like(B) if X0 is None else X0.clone()
    o = _opts(tol, maxit, poll_every, x0_zero=X0 is None, **opts)
    cb = None
    if trace_iterates > 0 and on_iter is not None:
        typestr = "<c16" if B.is_complex() else "<f8"

        def _cb(k, xp, rp, rows, sc, _user):
            # tensors over the library's device copies, cloned before the callback returns
            xk = torch.as_tensor(_DevView(xp, (n, s), typestr), device=B.device).clone()
            rk = torch.as_tensor(_DevView(rp, (int(rows), s), typestr), device=B.device).clone()
            on_iter(int(k), xk, rk, float(sc[0]), int(sc[1]))
        cb = ON_ITER(_cb)
        o.trace_iterates = int(trace_iterates)
        o.on_iter = ctypes.cast(cb, ctypes.c_void_p)
    r = _Report()
    _check(_lib.srk_solve(A.ctx.h, A.h, _dev(B, "B"), _dev(X, "X"), s, METHOD_ID[method], ctypes.byref(o),
                          ctypes.byref(r)), "srk_solve")
    return X, _report(r)


def solve_host(A: Matrix, B: np.ndarray, method: str = "egl_bicg", tol: float = 1e-8, maxit: int = 2000,
               X0: np.ndarray | None = None, poll_every: int = 8, inplace: bool = False, x0_zero: bool = False):
    """srk_solve_host: B, X in host memory (numpy, C-contiguous (n, s)). inplace=True
    overwrites X0 with the solution (keeps a pinned X0 buffer pinned: no staging copy);
    x0_zero=True (or X0=None) starts from X0 = 0 without copying X0 in."""
    B = np.ascontiguousarray(B)
    if X0 is None:
        X = np.zeros_like(B)
    elif inplace:
        if not (X0.flags.c_contiguous and X0.flags.writeable and X0.dtype == B.dtype and X0.shape == B.shape):
            raise SrkError("solve_host(inplace=True): X0 must be a writable C-contiguous array like B")
        X = X0
    else:
        X = np.ascontiguousarray(X0).copy()
    n, s = B.shape
    o = _opts(tol, maxit, poll_every, x0_zero=x0_zero or X0 is None)
    r = _Report()
    _check(_lib.srk_solve_host(A.ctx.h, A.h, B.ctypes.data_as(ctypes.c_void_p), X.ctypes.data_as(ctypes.c_void_p),
                               s, METHOD_ID[method], ctypes.byref(o), ctypes.byref(r)), "srk_solve_host")
    return X, _report(r)
