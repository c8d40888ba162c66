/* srk.h — C-ABI of the B200-native hot path for simultaneous short-recurrence
 * Krylov solvers, AX = B with s right-hand sides (Rashedi, Birk, Frommer,
 * Ebadi, arXiv:1504.04395; PAPER.md = /root/reference/PAPER.md, cited P:line).
 *
 * Problem (Eq. (1)): A in C^{n x n} sparse, X, B in C^{n x s}.
 *
 * CONVENTIONS (all entry points)
 *  - Block vectors (n x s; "block vector denoting a matrix of size n x s",
 *    P:131-132) are ROW-MAJOR ("row-interleaved"): element (i, j) at i*s + j,
 *    so one nonzero of A is applied to s contiguous values.
 *    SRK_C128 values are interleaved (re, im) doubles. Base addresses must be
 *    16-byte aligned (cudaMalloc / torch allocations are).
 *  - s x s results are row-major; scalars are one value of the dtype.
 *  - Inner products: <x, y> = y^H x and <X, Y> = tr(Y^H X).
 *  - Pointers are DEVICE pointers unless a name ends in _host.
 *  - Ownership: the caller owns every array it passes; srk_matrix_create copies
 *    the CSR arrays (the caller may free them afterwards); the library owns the
 *    workspace inside srk_ctx / srk_matrix / srk_solver.
 *  - Errors: every function returns SRK_OK (0) or a negative code; the message
 *    for the last error of the calling thread is srk_last_error(). Numerical
 *    breakdown is NOT an error: it is reported in srk_report.outcome.
 *  - Synchronisation: kernel-level calls (srk_spmm_block, srk_gram_block,
 *    srk_block_update, srk_tsqr) are asynchronous on the context's stream;
 *    srk_solve / srk_solver_* return after the device work they describe.
 *  - Determinism: no floating-point atomics; for a fixed input and launch
 *    configuration results are bitwise reproducible.
 *  - There is no CPU fallback: without a CUDA device every compute call fails
 *    with SRK_ECUDA.
 */
#ifndef SRK_H
#define SRK_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { SRK_F64 = 0, SRK_C128 = 1 } srk_dtype;

/* The 13 simultaneous methods (§2, §4):
 *  Li  = loop interchanged (Alg. 1), Gl = global (Alg. 2),
 *  eGl = economic global (Alg. 4; eGl-QMR P:464-465),
 *  Bl  = block (Alg. 3), rQ = QR of the block residual (Alg. 5,
 *  P:565-583; Bl-BiCGStab-rQ P:625-631). */
typedef enum {
  SRK_LI_BICG = 0, SRK_GL_BICG = 1, SRK_EGL_BICG = 2, SRK_BL_BICG = 3, SRK_BL_BICG_RQ = 4,
  SRK_LI_QMR = 5, SRK_GL_QMR = 6, SRK_EGL_QMR = 7, SRK_BL_QMR = 8,
  SRK_LI_BICGSTAB = 9, SRK_GL_BICGSTAB = 10, SRK_BL_BICGSTAB = 11, SRK_BL_BICGSTAB_RQ = 12,
  /* QR of the search directions [O'Leary]: the
   * stabilisation the paper compares with and rejects; iterates equal Bl-BiCG /
   * Bl-BiCGStab in exact arithmetic (reading R9) */
  SRK_BL_BICG_SQ = 13, SRK_BL_BICGSTAB_SQ = 14
} srk_method;

enum { SRK_OK = 0, SRK_EINVAL = -1, SRK_EDIM = -2, SRK_EUNSUPPORTED = -3, SRK_ECUDA = -4,
       SRK_ENCCL = -5, SRK_ENOMEM = -6 };

/* outcome of a solve ("div." = final true residual > 1) */
typedef enum { SRK_CONVERGED = 0, SRK_MAXIT = 1, SRK_BREAKDOWN = 2, SRK_DIVERGED = 3 } srk_outcome;
/* breakdown kinds: zero Lanczos denominator, singular s x s Gram
 * (P:232-234), rank-deficient thin QR (reading G11), non-finite value */
enum { SRK_BK_NONE = 0, SRK_BK_LANCZOS = 1, SRK_BK_GRAM = 2, SRK_BK_RANK = 3, SRK_BK_NONFINITE = 4,
       SRK_BK_OMEGA = 5 };

/* fused reductions */
typedef enum {
  SRK_GRAM_NONE = 0, SRK_GRAM_NORM2 = 1, SRK_GRAM_DIAG = 2, SRK_GRAM_TRACE = 3,
  SRK_GRAM_SUMVEC = 4, SRK_GRAM_FULL = 5, SRK_GRAM_COLNORM2 = 6
} srk_gram;
typedef enum { SRK_COEF_SCALAR = 1, SRK_COEF_DIAG = 2, SRK_COEF_FULL = 3 } srk_coef;

typedef struct srk_ctx srk_ctx;
typedef struct srk_matrix srk_matrix;
typedef struct srk_solver srk_solver;

/* CSR operator (0-based, sorted unique column indices per row).
 * row_ptr: n+1 int64 (values must fit int32: nnz < 2^31), col_idx: nnz int32,
 * values: nnz of dtype. All DEVICE pointers. */
typedef struct {
  int64_t n;
  int64_t nnz;
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const void* values;
  int dtype; /* srk_dtype */
} srk_csr;

typedef struct {
  int outcome;          /* srk_outcome */
  int iterations;       /* completed iterations (a BiCGStab half-step counts as one) */
  int half_step;        /* 1 if a BiCGStab variant stopped after its first half */
  int breakdown_kind;   /* SRK_BK_* */
  int breakdown_iter;   /* iteration (1-based) in which the breakdown occurred, else -1 */
  int frozen_cols;      /* Li variants: number of columns frozen by breakdown (reading G13) */
  int64_t matvec_cols_A;   /* columns multiplied by A (Prop. 1 counters) */
  int64_t matvec_cols_AH;  /* columns multiplied by A^H */
  double final_true_rel_residual;      /* ||B - A X||_F / ||R0||_F recomputed at exit */
  double final_recursive_rel_residual; /* ||R||_F (or ||C||_F for rQ) / ||R0||_F */
  double seconds;                      /* wall time of the iteration loop */
  int64_t kernel_launches;             /* kernels launched by the loop */
  int64_t vector_ops;   /* Prop. 1's count: inner products and SAXPYs of length n, per
                           iteration 7s (Li / Gl) or 7s^2 (Bl) for BiCG, summed over the solve */
  int breakdown_col;    /* Li variants: first frozen column (reading G13); thin QR: first
                           deficient column; else -1 */
  int deflated_cols;    /* rank_policy 1: columns replaced by the continuation so far */
} srk_report;

/* ------------------------------------------------------------------ context */
/* Create a context on `device` using CUDA stream `cuda_stream` (NULL = default
 * stream). Errors: SRK_ECUDA if no device. */
int srk_create(srk_ctx** ctx, int device, void* cuda_stream);
int srk_destroy(srk_ctx* ctx);
const char* srk_last_error(void);
int srk_version(void);

/* --------------------------------------------------------- a0: the operator */
/* Validate and copy a CSR operator to the device; if need_adjoint, also build
 * A^H = conj(A)^T explicitly ("A^H P̂"). Errors: SRK_EINVAL for an
 * invalid CSR (unsorted / out-of-range columns, bad row_ptr), SRK_ENOMEM. */
int srk_matrix_create(srk_ctx* ctx, const srk_csr* A, int need_adjoint, srk_matrix** out);
/* Block-sparse operator (a0, "BSR-12 (lattice)" of SURVEY §8(a); PAPER.md Ex. 4,
 * P:752-778): nb block rows of bs x bs blocks, block_row_ptr (nb+1, int64),
 * block_col (nnzb, int32, sorted unique per block row, < nb) and values (nnzb
 * blocks, each bs x bs row-major, complex interleaved), all DEVICE pointers, copied.
 * unit_diag = 1: the diagonal blocks are the identity and are NOT stored
 * (A = I + sum of the stored blocks, the A = I - kappa H form). Supported: bs = 12,
 * dtype SRK_C128, block widths s in {4, 8, 12, 16}, methods without A^H (the
 * BiCGStab family). Errors: SRK_EINVAL (invalid blocks), SRK_EUNSUPPORTED. */
int srk_matrix_create_bsr(srk_ctx* ctx, int64_t nb, int bs, int64_t nnzb, const int64_t* block_row_ptr,
                          const int32_t* block_col, const void* values, int dtype, int unit_diag,
                          srk_matrix** out);
/* Traversal hint for a block-sparse operator (a1; the read-A-once product of P:66-74 reads
 * every P row once only if its readers run close together in time): order_host (HOST array,
 * n = nb entries, a permutation of the block rows) is the order in which the product's warps
 * visit the block rows; null restores the natural order. Only the schedule changes: every entry
 * of Q is the same sum in the same order, so Q is bitwise independent of the hint (fused
 * reductions are summed in visiting order: deterministic, equal to rounding). For the
 * lexicographic 4D lattice of config 4 (site = x + L y + L^2 z + L^3 t) an order that walks
 * z-tiles of w planes through all t before the next tile brings the +-t neighbours within w
 * planes of each other (synth.lattice_tile_order). Not supported on distributed operators'
 * ghost rows (local rows only). Errors: SRK_EINVAL (not a permutation), SRK_EDIM (n != nb),
 * SRK_EUNSUPPORTED (not block-sparse), SRK_ENOMEM. */
int srk_matrix_set_row_order(srk_matrix* A, const int32_t* order_host, int64_t n);
/* Right ILU(0) preconditioning (the
 * no-fill incomplete LU of A, M = L U, computed once on the host from the operator's
 * CSR and attached to it). Every later solve with this operator iterates on
 * A M^-1 Y = B (A^H products as M^-H A^H) and returns X = M^-1 Y; X0 enters as Y0 = M X0.
 * The triangular solves run level-scheduled on the device. Scalar single-GPU CSR
 * operators only. Errors: SRK_EINVAL (zero pivot), SRK_EUNSUPPORTED, SRK_ENOMEM. */
int srk_matrix_ilu0(srk_matrix* A);
/* the factor values on A's pattern (L strictly below, U on and above the diagonal),
 * nnz values (complex interleaved) into a HOST buffer — for tests */
int srk_matrix_ilu0_factor(const srk_matrix* A, void* values_host);
/* Right ILUTP preconditioning: the incomplete LU "with threshold and pivoting with a drop
 * tolerance of 5e-2" of Ex. 4. The paper names only
 * Matlab's ilu; reading R14 fixes the algorithm: left-looking column ILU with
 * partial pivoting, a multiplier or L entry of column j dropped when its magnitude is below
 * droptol * ||A(:, j)||_2 (the pivot never), pivot = the largest candidate of the rows not yet
 * pivoted unless the original diagonal row's candidate reaches thresh times that (thresh = 1:
 * partial pivoting, 0: no pivoting while the diagonal is nonzero). Pi A ~ L U; solves then
 * iterate on A M^-1 Y = B with M = Pi^T L U (A^H products as M^-H A^H = Pi^T L^-H U^-H A^H),
 * the row permutation applied on the device around the level-scheduled triangular solves.
 * Computed once on the HOST from the operator's CSR (a0 work). Scalar single-GPU CSR
 * operators only. Errors: SRK_EINVAL (droptol < 0, thresh outside [0, 1], a column with no
 * nonzero pivot candidate), SRK_EUNSUPPORTED, SRK_ENOMEM. */
int srk_matrix_ilutp(srk_matrix* A, double droptol, double thresh);
/* kind 0 = ILU(0), 1 = ILUTP; nnz of the factor (L strictly lower + U); pivoted = a row moved */
int srk_matrix_prec_info(const srk_matrix* A, int* kind, int64_t* nnz_factor, int* pivoted);
/* the ILUTP factor F = (L - I) + U in the pivot order as a CSR (row_ptr n+1, col_idx /
 * values nnz_factor, complex interleaved) and perm (n: row of A pivoted at step k), all
 * HOST buffers — for tests */
int srk_matrix_ilutp_factor(const srk_matrix* A, int64_t* row_ptr, int32_t* col_idx, void* values, int64_t* perm);
/* Z = M^-1 P (adjoint: M^-H P), n x s device blocks, stream-ordered */
int srk_precond_apply(srk_ctx* ctx, const srk_matrix* A, int adjoint, const void* P, void* Z, int s);
int srk_matrix_destroy(srk_matrix* A);
/* copy A^H back (CSR arrays of size n+1 / nnz, device pointers) — for tests */
int srk_matrix_adjoint(const srk_matrix* A, int64_t* row_ptr, int32_t* col_idx, void* values);

/* -------------------------------------------- a8: multi-GPU (one process per GPU) */
/* Row partitioning and halo planning; HOST code, no GPU needed.
 * srk_partition_rows: contiguous row ranges balanced by nnz, offsets[nranks+1].
 * srk_plan_create: from the GLOBAL CSR (host arrays) the plan of `rank`: local CSR
 * (rows offsets[rank]..offsets[rank+1]-1, owned columns renumbered to [0, n_local),
 * ghost columns to n_local + position in the sorted ghost list, entries kept in the
 * global order so values[row_ptr[off0] : row_ptr[off1]] apply unchanged), the ghost
 * rows received per peer, and the owned rows sent to each peer. */
typedef struct srk_plan srk_plan;
int srk_partition_rows(int64_t n, const int64_t* row_ptr_host, int nranks, int64_t* offsets_host);
int srk_plan_create(int64_t n, const int64_t* row_ptr_host, const int32_t* col_idx_host, int nranks,
                    const int64_t* offsets_host, int rank, srk_plan** out);
int srk_plan_sizes(const srk_plan* p, int64_t* n_local, int64_t* nnz_local, int64_t* n_ghost, int64_t* n_send);
int srk_plan_arrays(const srk_plan* p, int64_t* row_ptr_local, int32_t* col_local, int64_t* ghost_global,
                    int32_t* recv_counts, int32_t* send_counts, int32_t* send_local);
int srk_plan_destroy(srk_plan* p);

/* NCCL communicator of the context (NCCL resolved at run time): rank 0 calls
 * srk_nccl_unique_id, broadcasts the 128 bytes (e.g. torch.distributed), every
 * rank calls srk_comm_init. With a communicator every reduction of the solver is
 * followed by an FP64 ncclAllReduce (the solver's: out of place, from a staging copy
 * of its workspace, so a reduction skipped after the stop flag cannot rescale a
 * carried value; kernel-level calls: in place) and every SpMM by a halo exchange. */
int srk_nccl_unique_id(void* id128_host);
int srk_comm_init(srk_ctx* ctx, const void* id128_host, int nranks, int rank);

/* Single-GPU virtual partition (SURVEY §4 "Multi-GPU without a cluster"): k virtual
 * ranks of one row-partitioned operator on ONE GPU, each driven by its own host thread
 * with its own srk_ctx (and stream) attached by srk_comm_init_virtual. Every solver and
 * kernel-level call then runs the distributed code path (halo exchange before each
 * SpMM, one allreduce per reduction point) with a device-to-device transport: halo rows
 * are copied out of the peers' send buffers, partial sums are reduced in rank order.
 * Collectives are rendezvous points: all k threads must make the same sequence of calls
 * (a thread that stops calling blocks the others). The group must outlive the contexts
 * attached to it. Errors: SRK_EINVAL (k < 1 or k > 16, bad rank). */
typedef struct srk_vgroup srk_vgroup;
int srk_vgroup_create(int k, srk_vgroup** out);
int srk_vgroup_destroy(srk_vgroup* g);
int srk_comm_init_virtual(srk_ctx* ctx, srk_vgroup* g, int rank);

/* A^H = conj(A)^T of a HOST CSR (a0), for building the adjoint operator of a
 * distributed matrix on every rank's host before srk_plan_create: row_ptr_out (n+1),
 * col_out (nnz, ascending within each row), values_out (nnz, dtype). Caller-owned
 * arrays. Errors: SRK_EINVAL (null pointers, n <= 0, bad dtype, column out of range). */
int srk_csr_adjoint_host(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const void* values, int dtype,
                         int64_t* row_ptr_out, int32_t* col_out, void* values_out);

/* halo of one local operator (host arrays): rows received from / sent to each peer */
typedef struct {
  const int32_t* recv_counts; /* nranks: ghost rows from each peer (sum = n_ghost) */
  const int32_t* send_counts; /* nranks */
  const int32_t* send_local;  /* n_send local row indices, grouped by peer */
  int64_t n_send;
} srk_halo;
/* Distributed operator: local rows of A (columns < n_local + n_ghost, device CSR)
 * and optionally of A^H with its own halo. Every n x s block passed to this
 * operator's SpMM must hold n_local + n_ghost rows (the ghost tail is written by
 * the halo exchange); the solver allocates its blocks that way. */
int srk_matrix_create_dist(srk_ctx* ctx, const srk_csr* A_local, int64_t n_ghost, const srk_halo* halo,
                           const srk_csr* AH_local, int64_t n_ghost_adj, const srk_halo* halo_adj,
                           srk_matrix** out);

/* Storage the SpMM of op(A) uses (a0): 0 CSR (lane-group kernel), 1 CSR in
 * length-sorted row order (irregular rows), 2 banded (<= 8 diagonals, the bulk-copy kernel
 * of band.cu; *ndiag = the diagonal count), 3 BSR-12. adjoint = 1: A^H's storage.
 * Errors: SRK_EINVAL (null matrix, adjoint without A^H). */
int srk_matrix_format(const srk_matrix* A, int adjoint, int* ndiag);

/* SELL-32-sigma form of op(A) (a0, SURVEY §8(a) "convert to SELL-C-sigma"; the read-A-once
 * product of P:66-74 for narrow blocks): built beside the length-sorted CSR when the row lengths
 * are irregular (max >= 4 mean + 8) and the padding stays under 25% of nnz — rows sorted by
 * decreasing length inside windows of sigma rows, chunks of C = 32 rows stored column-major and
 * padded to the chunk's longest row. Products with s * esz <= 32 bytes (one row per lane) use it;
 * wider blocks keep the lane-group CSR kernel. Returns 1 when the form exists (then *nchunk =
 * chunks, *entries = stored entries including padding, *sigma = the window; any may be null),
 * 0 when it does not. Errors: SRK_EINVAL (null matrix, adjoint without A^H). */
int srk_matrix_sell_info(const srk_matrix* A, int adjoint, int64_t* nchunk, int64_t* entries, int* sigma);

/* Distributed BSR-12 operator (config 4's lattice split into t-slabs): this
 * rank's nb_local block rows (DEVICE arrays, block columns renumbered as srk_plan_create does
 * for a block-row CSR: [0, nb_local) owned, nb_local + position in the sorted ghost list
 * for ghost block rows), and the halo in BLOCK units (host arrays). Every n x s block passed
 * to this operator holds (nb_local + nb_ghost) * 12 rows; the solver allocates its blocks
 * that way and each product first exchanges the 12 rows of every ghost block.
 * Errors: as srk_matrix_create_bsr; SRK_EINVAL for an inconsistent halo. */
int srk_matrix_create_bsr_dist(srk_ctx* ctx, int64_t nb_local, int bs, int64_t nnzb, const int64_t* block_row_ptr,
                               const int32_t* block_col, const void* values, int dtype, int unit_diag,
                               int64_t nb_ghost, const srk_halo* halo_blocks, srk_matrix** out);

/* ------------------------------------------------------ kernel-level calls */
/* Q = op(A) P, op = A (adjoint = 0) or A^H (adjoint = 1, needs need_adjoint),
 * P, Q: n x s row-major (a1/a2). If gram != SRK_GRAM_NONE the
 * reduction of mode `gram` between X = Q and Y (n x s block; n-vector for SUMVEC)
 * is fused into the epilogue and written to gram_out (device, dtype values):
 *   NORM2: ||Q||_F^2 (1 double); COLNORM2: s doubles; DIAG: (y_c^H q_c)_c (s);
 *   TRACE: tr(Y^H Q) (1); SUMVEC: sum(y^H Q) (1); FULL: Y^H Q (s x s).
 * FULL with s >= 8 is computed as the SpMM followed by Y^H Q on the FP64 tensor
 * cores (DMMA, the dense contraction north_star names); s < 8 fuses it into the
 * SpMM epilogue. Errors: SRK_EDIM (s < 1 or s > 64), SRK_EUNSUPPORTED (adjoint
 * without A^H). */
int srk_spmm_block(srk_ctx* ctx, const srk_matrix* A, int adjoint, const void* P, void* Q, int s,
                   int gram, const void* Y, void* gram_out);

/* out = reduction(X, Y) over n rows of two n x s blocks (mode as above; FULL gives
 * Y^H X, on the FP64 tensor cores for s >= 8). a3, P:155-158, 178, 192-195,
 * 243-249, 273-285, 443-447. */
int srk_gram_block(srk_ctx* ctx, const void* X, const void* Y, int64_t n, int s, int dtype, int gram,
                   void* out);

/* Yout = Yin + sign * X * coef (a5): coef is a scalar (Gl, Alg. 2), an s-vector
 * applied per column (Li, Alg. 1: X diag(coef)) or an s x s matrix (Bl, Alg. 3,
 * "BLAS3 GEMM" P:290-297); coef is a DEVICE pointer of dtype values. Yout may
 * alias Yin. sign = +1 or -1. */
int srk_block_update(srk_ctx* ctx, void* Yout, const void* Yin, const void* X, const void* coef, int coef_kind,
                     int sign, int64_t n, int s, int dtype);

/* Thin QR Z = Q C (a6; Eq. (3)) by CholQR2 on the device: C upper
 * triangular with real positive diagonal (s x s, device). *rank_host = s on
 * success; on rank deficiency (reading G11) returns SRK_OK with *rank_host < s
 * and Q unspecified. Synchronous (reads the rank flag). */
int srk_tsqr(srk_ctx* ctx, const void* Z, void* Q, void* C, int64_t n, int s, int dtype, int* rank_host);

/* ------------------------------------------------------------------ solve */
typedef struct {
  double tol;          /* stop when ||R||_F (||C||_F for rQ) <= tol ||R0||_F */
  int maxit;           /* iteration cap (reading G22: 2000) */
  int poll_every;      /* host reads the device convergence flag every k iterations (default 8) */
  int record_history;  /* keep ||R_k||_F/||R0||_F per iteration (srk_solver_history) */
  int check_true_residual; /* confirm convergence with B - AX (reading G26; default 1) */
  int use_graph;       /* replay the iterations between two polls as one CUDA graph (default 1;
                          off while srk_solver_profile is on) */
  int x0_zero;         /* X0 = 0 (the paper's protocol): X is output only — srk_solve does
                          not read it and srk_solve_host does not copy it in (default 0) */
  int shadow;          /* shadow block R̂0 / R̃: 0 = the paper's choice
                          (R0; the economic variants the column mean), 1 = conj(R0),
                          2 = column mean (every variant), 3 = shadow_given */
  const void* shadow_given; /* shadow == 3: DEVICE n x s block (economic variants: n-vector) */
  int preprocess_rhs;  /* 1: solve for the orthonormal factor Q of B = Q C and return X = Y C
                          (the paper's QR preprocessing of the right-hand sides; reading G9,
                          default 0); the tolerance is then relative to ||Q||_F = sqrt(s) */
  double eps_brk;      /* s x s LU pivot / scalar breakdown threshold, relative (0: 1e-14, G12) */
  double eps_defl;     /* CholQR pivot threshold relative to tr(Z^H Z) (0: 1e-14, R5) */
  int rank_policy;     /* rQ variants, rank-deficient thin QR: 0 = BREAKDOWN(rank) (reading G11),
                          1 = continue with the deficient columns of Q replaced by counter-based
                          random vectors orthogonalised against the others, C_jj = 0 (the implicit
                          deflation of P:396-403) */
  int trace_iterates;  /* K > 0 with on_iter set (srk_solve / srk_solve_host): the first K iterations run
                          one at a time and on_iter is called after each (lock-step parity, SURVEY
                          §8(b) / §4: "an iteration callback"); later iterations run as usual */
  /* k = iteration (1-based); X_k = the iterate (n x s) and R_or_C_k = the residual block R_k (n x s;
   * r_rows = n) or, for the rQ variants, C_k (s x s; r_rows = s): DEVICE pointers to copies owned by
   * the library, valid until the callback returns (the stream is synchronised before the call);
   * scalars_host[0] = the relative recursive residual ||R_k||_F / ||R_0||_F of the stopping rule
   * (P:643), scalars_host[1] = the solver state (0 running, 1 converged, 2 breakdown, 3 maxit). */
  void (*on_iter)(int k, const void* X_k, const void* R_or_C_k, int64_t r_rows, const double* scalars_host,
                  void* user);
  void* user;          /* passed back to on_iter */
} srk_opts;

/* Full solve (a1-a7): B, X device n x s blocks; X holds X0 on entry and the
 * iterate on exit. opts may be NULL (tol 1e-8, maxit 2000). s <= 64; the block
 * methods (s x s coefficients) take s <= 32, their s x s Grams from s = 8 on and their
 * s x s-coefficient updates on the FP64 tensor cores. The context keeps the last solver's workspace for the next
 * call with the same operator, s, method and options (freed by srk_destroy or
 * when the operator is destroyed). Errors: SRK_EUNSUPPORTED (e.g. a block method
 * with s > 32, a method needing A^H on an operator created without it). */
int srk_solve(srk_ctx* ctx, const srk_matrix* A, const void* B, void* X, int s, int method,
              const srk_opts* opts, srk_report* rep);
/* Same with HOST B and X (pinned or pageable): copies in, solves, copies out. */
int srk_solve_host(srk_ctx* ctx, const srk_matrix* A, const void* B_host, void* X_host, int s, int method,
                   const srk_opts* opts, srk_report* rep);

/* Stepping interface (lock-step parity and benchmarking): create, start with
 * (B, X0), run k iterations (stops early on convergence / breakdown), read the
 * current X / residual block, finish with a report. */
int srk_solver_create(srk_ctx* ctx, const srk_matrix* A, int s, int method, const srk_opts* opts,
                      srk_solver** out);
int srk_solver_destroy(srk_solver* sv);
int srk_solver_start(srk_solver* sv, const void* B, const void* X0);
/* run up to k more iterations; *state_host (optional) = 0 running, 1 converged,
 * 2 breakdown, 3 maxit */
int srk_solver_iterate(srk_solver* sv, int k, int* state_host);
/* copy the current iterate X_k (n x s) to X_out (device) */
int srk_solver_get_x(srk_solver* sv, void* X_out);
/* copy the current residual block R_k (n x s) — or, for the rQ variants, C_k
 * (s x s) — to out (device); *rows_host = n or s */
int srk_solver_get_residual(srk_solver* sv, void* out, int64_t* rows_host);
int srk_solver_report(srk_solver* sv, srk_report* rep);
/* Per-launch CUDA-event timing of the solver's kernels (off by default). Tags:
 * 0 SpMM with A, 1 SpMM with A^H, 2 block updates / Grams, 3 partial-sum
 * finalisation, 4 s x s coefficient phases. profile_read synchronises, returns
 * the summed milliseconds and launch counts per tag since the last read, and
 * resets them. */
int srk_solver_profile(srk_solver* sv, int enable);
int srk_solver_profile_read(srk_solver* sv, double* ms_host, int64_t* count_host, int ntag);
/* The same records launch by launch (instead of profile_read; resets them): tag
 * as above, signature (SpMM: block width s; update: 16 * inputs + outputs),
 * milliseconds, and the launch's algorithmic bytes (A's arrays
 * once, every block operand read once and every result written once). Host
 * arrays of max_records entries; returns the number of records (>= 0). */
int srk_solver_profile_launches(srk_solver* sv, int32_t* tag_host, int32_t* sig_host, double* ms_host,
                                double* bytes_host, int max_records);
/* history (host array of length >= iterations): relative recursive residuals */
int srk_solver_history(srk_solver* sv, double* hist_host, int cap);

#ifdef __cplusplus
}
#endif
#endif /* SRK_H */
