// api.cu — the C-ABI of include/srk.h. Argument checking and marshalling only;
// all arithmetic happens in the kernels of block_kernels.cu / coef.cu.
#include <cstdio>
#include <atomic>
#include <cstring>
#include <string>

#include "solver.h"

using namespace srk;

struct srk_ctx {
  Ctx c;  // first member: a Mat's Ctx* identifies its srk_ctx
  // srk_solve keeps the last solver (its n x s workspace) for the next call with the
  // same operator, width, method and options, and srk_solve_host its staging blocks,
  // so repeated solves do not reallocate gigabytes of device memory
  srk_solver* cached = nullptr;
  unsigned long long cached_mat = 0;
  int cached_s = 0, cached_method = -1;
  srk_opts cached_opts{};
  void* hbuf[2] = {nullptr, nullptr};
  size_t hcap = 0;
};
static std::atomic<unsigned long long> g_matrix_id{0};
struct srk_matrix {
  Mat m;
  unsigned long long id = ++g_matrix_id;
};
struct srk_solver {
  Solver* sv;
};

static thread_local std::string g_err;

static int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}
static int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return SRK_ECUDA;
}
static int check_cuda(int e, const char* where) {
  if (e == 0) return SRK_OK;
  return cuda_fail((cudaError_t)e, where);
}

extern "C" {

const char* srk_last_error(void) { return g_err.c_str(); }
int srk_version(void) { return 1; }

int srk_create(srk_ctx** out, int device, void* stream) {
  if (!out) return fail(SRK_EINVAL, "srk_create: null out");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return cuda_fail(e == cudaSuccess ? cudaErrorNoDevice : e, "srk_create");
  if (device < 0 || device >= ndev) return fail(SRK_EINVAL, "srk_create: bad device");
  if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  auto* ctx = new srk_ctx();
  ctx->c.dev = device;
  ctx->c.st = (cudaStream_t)stream;
  cudaDeviceGetAttribute(&ctx->c.nsm, cudaDevAttrMultiProcessorCount, device);
  *out = ctx;
  return SRK_OK;
}

static void drop_cache(srk_ctx* ctx) {
  if (ctx->cached) srk_solver_destroy(ctx->cached);
  ctx->cached = nullptr;
  ctx->cached_mat = 0;
}

int srk_destroy(srk_ctx* ctx) {
  if (!ctx) return SRK_OK;
  drop_cache(ctx);
  for (void* p : ctx->hbuf)
    if (p) cudaFree(p);
  if (ctx->c.partials) cudaFree(ctx->c.partials);
  if (ctx->c.side) cudaStreamDestroy(ctx->c.side);
  if (ctx->c.ev_p) cudaEventDestroy(ctx->c.ev_p);
  if (ctx->c.ev_h) cudaEventDestroy(ctx->c.ev_h);
  if (ctx->c.comm) comm_destroy(ctx->c.comm);
  delete ctx;
  return SRK_OK;
}

__global__ static void rp64to32(const int64_t* a, int* b, long long n, int* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= n; i += (long long)gridDim.x * blockDim.x) {
    const int64_t v = a[i];
    if (v < 0 || v > 2147483647LL) atomicOr(bad, 8);
    b[i] = (int)v;
  }
}

int srk_matrix_create(srk_ctx* ctx, const srk_csr* A, int need_adjoint, srk_matrix** out) {
  if (!ctx || !A || !out) return fail(SRK_EINVAL, "srk_matrix_create: null argument");
  if (A->n <= 0 || A->nnz < 0 || !A->row_ptr || (A->nnz > 0 && (!A->col_idx || !A->values)))
    return fail(SRK_EINVAL, "srk_matrix_create: invalid CSR header");
  if (A->dtype != SRK_F64 && A->dtype != SRK_C128) return fail(SRK_EINVAL, "srk_matrix_create: bad dtype");
  if (A->nnz >= 2147483647LL) return fail(SRK_EUNSUPPORTED, "srk_matrix_create: nnz >= 2^31");
  cudaStream_t st = ctx->c.st;
  auto* M = new srk_matrix();
  Mat& m = M->m;
  m.ctx = &ctx->c;
  m.n = A->n;
  m.nnz = A->nnz;
  m.cplx = A->dtype == SRK_C128;
  const size_t esz = m.cplx ? 16 : 8;
  int* dbad = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&m.rp, sizeof(int) * (m.n + 1))) != cudaSuccess ||
      (e = cudaMalloc(&m.ci, sizeof(int) * (m.nnz + 1))) != cudaSuccess ||
      (e = cudaMalloc(&m.val, esz * (m.nnz + 1))) != cudaSuccess || (e = cudaMalloc(&dbad, sizeof(int))) != cudaSuccess) {
    srk_matrix_destroy(M);
    if (dbad) cudaFree(dbad);
    return fail(SRK_ENOMEM, "srk_matrix_create: out of device memory");
  }
  cudaMemsetAsync(dbad, 0, sizeof(int), st);
  const int grid = (int)std::max<long long>(1, std::min<long long>((m.n + 256) / 256, 148 * 8));
  rp64to32<<<grid, 256, 0, st>>>(A->row_ptr, m.rp, m.n, dbad);
  if (m.nnz > 0) {
    cudaMemcpyAsync(m.ci, A->col_idx, sizeof(int) * m.nnz, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(m.val, A->values, esz * m.nnz, cudaMemcpyDeviceToDevice, st);
  }
  launch_csr_check(m.n, m.n, m.nnz, m.rp, m.ci, 1, dbad, st);
  int bad = 0;
  cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) {
    cudaFree(dbad);
    srk_matrix_destroy(M);
    return cuda_fail(e, "srk_matrix_create");
  }
  if (bad) {
    cudaFree(dbad);
    srk_matrix_destroy(M);
    char msg[128];
    snprintf(msg, sizeof msg, "srk_matrix_create: invalid CSR (code %d: 1 row_ptr, 2 column range, 4 unsorted, 8 int32)", bad);
    return fail(SRK_EINVAL, msg);
  }
  if (need_adjoint) {
    int* work = nullptr;
    if ((e = cudaMalloc(&m.rpH, sizeof(int) * (m.n + 1))) != cudaSuccess ||
        (e = cudaMalloc(&m.ciH, sizeof(int) * (m.nnz + 1))) != cudaSuccess ||
        (e = cudaMalloc(&m.valH, esz * (m.nnz + 1))) != cudaSuccess || (e = cudaMalloc(&work, sizeof(int) * (m.n + 1))) != cudaSuccess) {
      cudaFree(dbad);
      srk_matrix_destroy(M);
      return fail(SRK_ENOMEM, "srk_matrix_create: out of device memory (adjoint)");
    }
    launch_csr_transpose(m.cplx, m.n, m.nnz, m.rp, m.ci, m.val, m.rpH, m.ciH, m.valH, work, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) {
      cudaFree(work);
      cudaFree(dbad);
      srk_matrix_destroy(M);
      return cuda_fail(e, "srk_matrix_create: adjoint");
    }
    cudaFree(work);
    m.has_adj = true;
    m.nnzH = m.nnz;
  }
  cudaFree(dbad);
  if (build_balanced_order(m, false, st) || (m.has_adj && build_balanced_order(m, true, st))) {
    srk_matrix_destroy(M);
    return fail(SRK_ENOMEM, "srk_matrix_create: balanced row order");
  }
  // regular operators on <= 8 diagonals (the stencils): the banded form of a0 (band.cu)
  static const bool no_band = getenv("SRK_NO_BAND") != nullptr;  // A/B switch for measurements
  if (!no_band && !m.srt.perm) {
    if (build_band(m.cplx, m.n, m.rp, m.ci, m.val, m.band, st) ||
        (m.has_adj && build_band(m.cplx, m.n, m.rpH, m.ciH, m.valH, m.bandH, st))) {
      srk_matrix_destroy(M);
      return fail(SRK_ENOMEM, "srk_matrix_create: banded form");
    }
  }
  *out = M;
  return SRK_OK;
}

static int create_bsr(srk_ctx* ctx, int64_t nb, int bs, int64_t nnzb, const int64_t* block_row_ptr,
                      const int32_t* block_col, const void* values, int dtype, int unit_diag, int64_t nb_ghost,
                      const srk_halo* halo_blocks, srk_matrix** out);
static int upload_halo(Halo& H, const srk_halo* h, int nranks, long long n_ghost);

int srk_matrix_create_bsr(srk_ctx* ctx, int64_t nb, int bs, int64_t nnzb, const int64_t* block_row_ptr,
                          const int32_t* block_col, const void* values, int dtype, int unit_diag,
                          srk_matrix** out) {
  return create_bsr(ctx, nb, bs, nnzb, block_row_ptr, block_col, values, dtype, unit_diag, 0, nullptr, out);
}

int srk_matrix_create_bsr_dist(srk_ctx* ctx, int64_t nb_local, int bs, int64_t nnzb, const int64_t* block_row_ptr,
                               const int32_t* block_col, const void* values, int dtype, int unit_diag,
                               int64_t nb_ghost, const srk_halo* halo_blocks, srk_matrix** out) {
  if (nb_ghost < 0) return fail(SRK_EINVAL, "srk_matrix_create_bsr_dist: nb_ghost < 0");
  const int nranks = ctx && ctx->c.comm ? ctx->c.comm->nranks : 1;
  if ((nb_ghost > 0 || (halo_blocks && halo_blocks->n_send > 0)) && nranks == 1)
    return fail(SRK_EINVAL, "srk_matrix_create_bsr_dist: halo given but no communicator");
  return create_bsr(ctx, nb_local, bs, nnzb, block_row_ptr, block_col, values, dtype, unit_diag, nb_ghost, halo_blocks,
                    out);
}

static int create_bsr(srk_ctx* ctx, int64_t nb, int bs, int64_t nnzb, const int64_t* block_row_ptr,
                      const int32_t* block_col, const void* values, int dtype, int unit_diag, int64_t nb_ghost,
                      const srk_halo* halo_blocks, srk_matrix** out) {
  if (!ctx || !out || !block_row_ptr || nb < 1 || nnzb < 0 || (nnzb > 0 && (!block_col || !values)))
    return fail(SRK_EINVAL, "srk_matrix_create_bsr: bad argument");
  if (bs != 12 || dtype != SRK_C128)
    return fail(SRK_EUNSUPPORTED, "srk_matrix_create_bsr: 12 x 12 complex blocks only");
  if (nnzb >= 2147483647LL) return fail(SRK_EUNSUPPORTED, "srk_matrix_create_bsr: nnzb >= 2^31");
  cudaStream_t st = ctx->c.st;
  auto* M = new srk_matrix();
  Mat& m = M->m;
  m.ctx = &ctx->c;
  m.cplx = true;
  m.bsr = true;
  m.bs = bs;
  m.nb = nb;
  m.nnzb = nnzb;
  m.unit_diag = unit_diag ? 1 : 0;
  m.n = nb * bs;
  m.nnz = nnzb * bs * bs + (unit_diag ? m.n : 0);
  const size_t bbytes = (size_t)bs * bs * 16;
  int* dbad = nullptr;
  if (cudaMalloc(&m.brp, sizeof(int) * (nb + 1)) != cudaSuccess || cudaMalloc(&m.bci, sizeof(int) * (nnzb + 1)) != cudaSuccess ||
      cudaMalloc(&m.bval, bbytes * (nnzb + 1)) != cudaSuccess || cudaMalloc(&dbad, sizeof(int)) != cudaSuccess) {
    if (dbad) cudaFree(dbad);
    srk_matrix_destroy(M);
    return fail(SRK_ENOMEM, "srk_matrix_create_bsr: out of device memory");
  }
  cudaMemsetAsync(dbad, 0, sizeof(int), st);
  const int grid = (int)std::max<long long>(1, std::min<long long>((nb + 256) / 256, 148 * 8));
  rp64to32<<<grid, 256, 0, st>>>(block_row_ptr, m.brp, nb, dbad);
  if (nnzb > 0) {
    cudaMemcpyAsync(m.bci, block_col, sizeof(int) * nnzb, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(m.bval, values, bbytes * nnzb, cudaMemcpyDeviceToDevice, st);
  }
  // distributed (t-slab) operators: block columns >= nb are ghost block rows; the entries keep
  // the global block order, so a row's local columns need not ascend (sorted check off)
  launch_csr_check(nb, nb + nb_ghost, nnzb, m.brp, m.bci, nb_ghost > 0 ? 0 : 1, dbad, st);
  int bad = 0;
  cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(dbad);
  if (e != cudaSuccess) {
    srk_matrix_destroy(M);
    return cuda_fail(e, "srk_matrix_create_bsr");
  }
  if (bad) {
    srk_matrix_destroy(M);
    return fail(SRK_EINVAL, "srk_matrix_create_bsr: invalid block structure (row pointers / sorted block columns)");
  }
  if (nb_ghost > 0 || (halo_blocks && halo_blocks->n_send > 0)) {
    // the block halo as a halo of P rows: block b -> rows 12 b .. 12 b + 11
    const int nranks = ctx->c.comm->nranks;
    std::vector<int32_t> rc(nranks), sc(nranks), sl;
    for (int p = 0; p < nranks; ++p) {
      rc[p] = halo_blocks ? halo_blocks->recv_counts[p] * bs : 0;
      sc[p] = halo_blocks ? halo_blocks->send_counts[p] * bs : 0;
    }
    for (int64_t q = 0; halo_blocks && q < halo_blocks->n_send; ++q)
      for (int r = 0; r < bs; ++r) sl.push_back(halo_blocks->send_local[q] * bs + r);
    srk_halo hr{rc.data(), sc.data(), sl.empty() ? nullptr : sl.data(), (int64_t)sl.size()};
    m.dist = true;
    const int r = upload_halo(m.halo, &hr, nranks, nb_ghost * bs);
    if (r) {
      srk_matrix_destroy(M);
      return fail(r, "srk_matrix_create_bsr_dist: inconsistent block halo");
    }
  }
  *out = M;
  return SRK_OK;
}

int srk_matrix_ilu0(srk_matrix* A) {
  if (!A) return fail(SRK_EINVAL, "srk_matrix_ilu0: null matrix");
  Mat& m = A->m;
  if (m.bsr || m.dist) return fail(SRK_EUNSUPPORTED, "srk_matrix_ilu0: scalar single-GPU CSR operators only");
  srk_ctx* owner = reinterpret_cast<srk_ctx*>(m.ctx);
  if (owner && owner->cached_mat == A->id) drop_cache(owner);  // the operator changes
  const int r = build_ilu0(m, m.ctx->st);
  if (r == 1) return fail(SRK_EINVAL, "srk_matrix_ilu0: zero pivot (missing or vanishing diagonal)");
  if (r == 2) return fail(SRK_ENOMEM, "srk_matrix_ilu0: out of device memory");
  if (r) return fail(SRK_ECUDA, "srk_matrix_ilu0: CUDA error");
  return SRK_OK;
}

int srk_matrix_ilutp(srk_matrix* A, double droptol, double thresh) {
  if (!A) return fail(SRK_EINVAL, "srk_matrix_ilutp: null matrix");
  if (!(droptol >= 0.0) || !(thresh >= 0.0) || !(thresh <= 1.0))
    return fail(SRK_EINVAL, "srk_matrix_ilutp: droptol >= 0 and 0 <= thresh <= 1 required");
  Mat& m = A->m;
  if (m.bsr || m.dist) return fail(SRK_EUNSUPPORTED, "srk_matrix_ilutp: scalar single-GPU CSR operators only");
  srk_ctx* owner = reinterpret_cast<srk_ctx*>(m.ctx);
  if (owner && owner->cached_mat == A->id) drop_cache(owner);
  const int r = build_ilutp(m, droptol, thresh, m.ctx->st);
  if (r == 1) return fail(SRK_EINVAL, "srk_matrix_ilutp: a column without a nonzero pivot (structurally singular)");
  if (r == 2) return fail(SRK_ENOMEM, "srk_matrix_ilutp: out of memory");
  if (r) return fail(SRK_ECUDA, "srk_matrix_ilutp: CUDA error");
  return SRK_OK;
}

int srk_matrix_prec_info(const srk_matrix* A, int* kind, int64_t* nnz_factor, int* pivoted) {
  if (!A || !kind || !nnz_factor || !pivoted) return fail(SRK_EINVAL, "srk_matrix_prec_info: null argument");
  const Prec* P = A->m.prec;
  if (!P) return fail(SRK_EINVAL, "srk_matrix_prec_info: no preconditioner attached");
  *kind = P->kind;
  *nnz_factor = P->kind ? (int64_t)P->fci.size() : A->m.nnz;
  *pivoted = P->perm ? 1 : 0;
  return SRK_OK;
}

int srk_matrix_ilutp_factor(const srk_matrix* A, int64_t* row_ptr, int32_t* col_idx, void* values, int64_t* perm) {
  if (!A || !row_ptr || !col_idx || !values || !perm) return fail(SRK_EINVAL, "srk_matrix_ilutp_factor: null argument");
  const Prec* P = A->m.prec;
  if (!P || P->kind != 1) return fail(SRK_EINVAL, "srk_matrix_ilutp_factor: no ILUTP attached");
  for (size_t i = 0; i < P->frp.size(); ++i) row_ptr[i] = P->frp[i];
  for (size_t i = 0; i < P->fci.size(); ++i) col_idx[i] = P->fci[i];
  std::memcpy(values, P->factor.data(), P->factor.size() * sizeof(double));
  for (size_t i = 0; i < P->hperm.size(); ++i) perm[i] = P->hperm[i];
  return SRK_OK;
}

int srk_matrix_ilu0_factor(const srk_matrix* A, void* values_host) {
  if (!A || !values_host) return fail(SRK_EINVAL, "srk_matrix_ilu0_factor: null argument");
  if (!A->m.prec || A->m.prec->kind != 0) return fail(SRK_EINVAL, "srk_matrix_ilu0_factor: no ILU(0) attached");
  const std::vector<double>& f = A->m.prec->factor;
  std::memcpy(values_host, f.data(), f.size() * sizeof(double));
  return SRK_OK;
}

int srk_precond_apply(srk_ctx* ctx, const srk_matrix* A, int adjoint, const void* P, void* Z, int s) {
  if (!ctx || !A || !P || !Z) return fail(SRK_EINVAL, "srk_precond_apply: null argument");
  if (!A->m.prec) return fail(SRK_EINVAL, "srk_precond_apply: no ILU(0) attached");
  if (s < 1 || s > 64) return fail(SRK_EDIM, "srk_precond_apply: s must be in [1, 64]");
  Eng e;
  e.c = &ctx->c;
  e.A = &A->m;
  e.cplx = A->m.cplx;
  e.n = A->m.n;
  int r = e.prec_solve(adjoint != 0, P, Z, s);
  if (!r) r = (int)cudaStreamSynchronize(ctx->c.st);
  return check_cuda(r, "srk_precond_apply");
}

// ---------------------------------------------------------------- multi-GPU
int srk_nccl_unique_id(void* id128_host) {
  if (!id128_host) return fail(SRK_EINVAL, "srk_nccl_unique_id: null buffer");
  if (nccl_unique_id(id128_host)) return fail(SRK_ENCCL, "srk_nccl_unique_id: NCCL not available");
  return SRK_OK;
}

int srk_comm_init(srk_ctx* ctx, const void* id128_host, int nranks, int rank) {
  if (!ctx || !id128_host || nranks < 1 || rank < 0 || rank >= nranks) return fail(SRK_EINVAL, "srk_comm_init: bad argument");
  if (ctx->c.comm) comm_destroy(ctx->c.comm);
  ctx->c.comm = nullptr;
  if (nranks == 1) return SRK_OK;
  Comm* C = comm_create(id128_host, nranks, rank);
  if (!C) return fail(SRK_ENCCL, "srk_comm_init: ncclCommInitRank failed (or NCCL not available)");
  ctx->c.comm = C;
  return SRK_OK;
}

struct srk_vgroup {
  VGroup* g;
};

int srk_vgroup_create(int k, srk_vgroup** out) {
  if (!out || k < 1 || k > 16) return fail(SRK_EINVAL, "srk_vgroup_create: k must be in [1, 16]");
  VGroup* g = vgroup_create(k);
  if (!g) return fail(SRK_ECUDA, "srk_vgroup_create: event creation failed");
  *out = new srk_vgroup{g};
  return SRK_OK;
}

int srk_vgroup_destroy(srk_vgroup* g) {
  if (!g) return SRK_OK;
  vgroup_destroy(g->g);
  delete g;
  return SRK_OK;
}

int srk_comm_init_virtual(srk_ctx* ctx, srk_vgroup* g, int rank) {
  if (!ctx || !g || rank < 0 || rank >= vgroup_size(g->g)) return fail(SRK_EINVAL, "srk_comm_init_virtual: bad argument");
  if (ctx->c.comm) comm_destroy(ctx->c.comm);
  ctx->c.comm = nullptr;
  if (vgroup_size(g->g) == 1) return SRK_OK;
  auto* C = new Comm();
  C->nranks = vgroup_size(g->g);
  C->rank = rank;
  C->vg = g->g;
  ctx->c.comm = C;
  return SRK_OK;
}

static int upload_halo(Halo& H, const srk_halo* h, int nranks, long long n_ghost) {
  H.nranks = nranks;
  H.n_ghost = n_ghost;
  H.n_send = h ? h->n_send : 0;
  H.send_off = new int64_t[nranks + 1];
  H.recv_off = new int64_t[nranks + 1];
  H.send_off[0] = H.recv_off[0] = 0;
  for (int p = 0; p < nranks; ++p) {
    H.send_off[p + 1] = H.send_off[p] + (h ? h->send_counts[p] : 0);
    H.recv_off[p + 1] = H.recv_off[p] + (h ? h->recv_counts[p] : 0);
  }
  if (H.send_off[nranks] != H.n_send || H.recv_off[nranks] != n_ghost) return SRK_EINVAL;
  if (H.n_send > 0) {
    if (cudaMalloc(&H.send_idx, sizeof(int) * H.n_send) != cudaSuccess) return SRK_ENOMEM;
    if (cudaMemcpy(H.send_idx, h->send_local, sizeof(int) * H.n_send, cudaMemcpyHostToDevice) != cudaSuccess)
      return SRK_ECUDA;
  }
  return SRK_OK;
}

static int upload_csr(Mat& m, const srk_csr* A, long long ncols, int** rp, int** ci, void** val, cudaStream_t st) {
  const size_t esz = m.cplx ? 16 : 8;
  int* dbad = nullptr;
  if (cudaMalloc(rp, sizeof(int) * (A->n + 1)) != cudaSuccess || cudaMalloc(ci, sizeof(int) * (A->nnz + 1)) != cudaSuccess ||
      cudaMalloc(val, esz * (A->nnz + 1)) != cudaSuccess || cudaMalloc(&dbad, sizeof(int)) != cudaSuccess) {
    if (dbad) cudaFree(dbad);
    return SRK_ENOMEM;
  }
  cudaMemsetAsync(dbad, 0, sizeof(int), st);
  const int grid = (int)std::max<long long>(1, std::min<long long>((A->n + 256) / 256, 148 * 8));
  rp64to32<<<grid, 256, 0, st>>>(A->row_ptr, *rp, A->n, dbad);
  if (A->nnz > 0) {
    cudaMemcpyAsync(*ci, A->col_idx, sizeof(int) * A->nnz, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(*val, A->values, esz * A->nnz, cudaMemcpyDeviceToDevice, st);
  }
  launch_csr_check(A->n, ncols, A->nnz, *rp, *ci, 0, dbad, st);
  int bad = 0;
  cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(dbad);
  if (e != cudaSuccess) return SRK_ECUDA;
  return bad ? SRK_EINVAL : SRK_OK;
}

int srk_matrix_create_dist(srk_ctx* ctx, const srk_csr* A, int64_t n_ghost, const srk_halo* halo, const srk_csr* AH,
                           int64_t n_ghost_adj, const srk_halo* halo_adj, srk_matrix** out) {
  if (!ctx || !A || !out || n_ghost < 0) return fail(SRK_EINVAL, "srk_matrix_create_dist: bad argument");
  if (A->dtype != SRK_F64 && A->dtype != SRK_C128) return fail(SRK_EINVAL, "srk_matrix_create_dist: bad dtype");
  const int nranks = ctx->c.comm ? ctx->c.comm->nranks : 1;
  if ((n_ghost > 0 || (halo && halo->n_send > 0)) && nranks == 1)
    return fail(SRK_EINVAL, "srk_matrix_create_dist: halo given but srk_comm_init was not called");
  auto* M = new srk_matrix();
  Mat& m = M->m;
  m.ctx = &ctx->c;
  m.n = A->n;
  m.nnz = A->nnz;
  m.cplx = A->dtype == SRK_C128;
  m.dist = true;
  int r = upload_csr(m, A, A->n + n_ghost, &m.rp, &m.ci, &m.val, ctx->c.st);
  if (!r) r = upload_halo(m.halo, halo, nranks, n_ghost);
  if (!r && AH) {
    if (AH->n != A->n || AH->dtype != A->dtype) r = SRK_EDIM;
    if (!r) r = upload_csr(m, AH, AH->n + n_ghost_adj, &m.rpH, &m.ciH, &m.valH, ctx->c.st);
    if (!r) r = upload_halo(m.haloH, halo_adj, nranks, n_ghost_adj);
    if (!r) {
      m.has_adj = true;
      m.nnzH = AH->nnz;
    }
  }
  if (r) {
    srk_matrix_destroy(M);
    return fail(r, "srk_matrix_create_dist: invalid local CSR / halo (columns must be < n_local + n_ghost)");
  }
  if (build_balanced_order(m, false, ctx->c.st) || (m.has_adj && build_balanced_order(m, true, ctx->c.st))) {
    srk_matrix_destroy(M);
    return fail(SRK_ENOMEM, "srk_matrix_create_dist: balanced row order");
  }
  if (build_halo_split(m, false, ctx->c.st) || (m.has_adj && build_halo_split(m, true, ctx->c.st))) {
    srk_matrix_destroy(M);
    return fail(SRK_ENOMEM, "srk_matrix_create_dist: interior / boundary rows");
  }
  *out = M;
  return SRK_OK;
}

int srk_matrix_format(const srk_matrix* M, int adjoint, int* ndiag) {
  if (!M || (adjoint && !M->m.has_adj)) return fail(SRK_EINVAL, "srk_matrix_format: bad argument");
  const Mat& m = M->m;
  const Mat::Band& b = adjoint ? m.bandH : m.band;
  if (ndiag) *ndiag = b.K;
  if (m.bsr) return 3;
  if (b.K > 0) return 2;
  if ((adjoint ? m.srtH.perm : m.srt.perm) != nullptr) return 1;
  return 0;
}

int srk_matrix_set_row_order(srk_matrix* M, const int32_t* order_host, int64_t n) {
  if (!M) return fail(SRK_EINVAL, "srk_matrix_set_row_order: null matrix");
  Mat& m = M->m;
  if (!m.bsr) return fail(SRK_EUNSUPPORTED, "srk_matrix_set_row_order: block-sparse operators only");
  if (m.border) {
    cudaFree(m.border);
    m.border = nullptr;
  }
  if (!order_host) return SRK_OK;  // back to the natural order
  if (n != m.nb) return fail(SRK_EDIM, "srk_matrix_set_row_order: the order must list every block row");
  std::vector<char> seen((size_t)n, 0);
  for (int64_t k = 0; k < n; ++k) {
    const int32_t r = order_host[k];
    if (r < 0 || r >= n || seen[(size_t)r]) return fail(SRK_EINVAL, "srk_matrix_set_row_order: not a permutation");
    seen[(size_t)r] = 1;
  }
  if (cudaMalloc(&m.border, sizeof(int) * (size_t)n) != cudaSuccess) {
    m.border = nullptr;
    return fail(SRK_ENOMEM, "srk_matrix_set_row_order: out of device memory");
  }
  cudaError_t e = cudaMemcpy(m.border, order_host, sizeof(int) * (size_t)n, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "srk_matrix_set_row_order");
  return SRK_OK;
}

int srk_matrix_sell_info(const srk_matrix* M, int adjoint, int64_t* nchunk, int64_t* entries, int* sigma) {
  if (!M || (adjoint && !M->m.has_adj)) return fail(SRK_EINVAL, "srk_matrix_sell_info: bad argument");
  const Mat::Sell& se = adjoint ? M->m.sellH : M->m.sell;
  if (nchunk) *nchunk = se.nchunk;
  if (entries) *entries = se.entries;
  if (sigma) *sigma = se.sigma;
  return se.cs != nullptr ? 1 : 0;
}

int srk_matrix_destroy(srk_matrix* M) {
  if (!M) return SRK_OK;
  Mat& m = M->m;
  if (m.ctx) {  // a cached solver of this operator dies with it
    srk_ctx* owner = reinterpret_cast<srk_ctx*>(m.ctx);
    if (owner->cached_mat == M->id) drop_cache(owner);
  }
  if (m.border) cudaFree(m.border);
  if (m.rp) cudaFree(m.rp);
  if (m.ci) cudaFree(m.ci);
  if (m.val) cudaFree(m.val);
  if (m.rpH) cudaFree(m.rpH);
  if (m.ciH) cudaFree(m.ciH);
  if (m.valH) cudaFree(m.valH);
  for (Halo* H : {&m.halo, &m.haloH}) {
    if (H->send_idx) cudaFree(H->send_idx);
    delete[] H->send_off;
    delete[] H->recv_off;
  }
  if (m.sendbuf) cudaFree(m.sendbuf);
  free_prec(m.prec);
  m.prec = nullptr;
  if (m.brp) cudaFree(m.brp);
  if (m.bci) cudaFree(m.bci);
  if (m.bval) cudaFree(m.bval);
  free_balanced_order(m);
  if (m.band.val) cudaFree(m.band.val);
  if (m.bandH.val) cudaFree(m.bandH.val);
  delete M;
  return SRK_OK;
}

__global__ static void rp32to64(const int* a, int64_t* b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= n; i += (long long)gridDim.x * blockDim.x) b[i] = a[i];
}

int srk_matrix_adjoint(const srk_matrix* M, int64_t* row_ptr, int32_t* col_idx, void* values) {
  if (!M || !M->m.has_adj) return fail(SRK_EINVAL, "srk_matrix_adjoint: no adjoint");
  const Mat& m = M->m;
  cudaStream_t st = m.ctx->st;
  rp32to64<<<64, 256, 0, st>>>(m.rpH, row_ptr, m.n);
  cudaMemcpyAsync(col_idx, m.ciH, sizeof(int) * m.nnz, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(values, m.valH, (m.cplx ? 16 : 8) * m.nnz, cudaMemcpyDeviceToDevice, st);
  cudaError_t e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? SRK_OK : cuda_fail(e, "srk_matrix_adjoint");
}

static bool gram_ok(int g) { return g >= SRK_GRAM_NONE && g <= SRK_GRAM_COLNORM2; }

int srk_spmm_block(srk_ctx* ctx, const srk_matrix* A, int adjoint, const void* P, void* Q, int s, int gram,
                   const void* Y, void* gram_out) {
  if (!ctx || !A || !P || !Q) return fail(SRK_EINVAL, "srk_spmm_block: null argument");
  if (s < 1 || s > 64) return fail(SRK_EDIM, "srk_spmm_block: s must be in [1, 64]");
  if (!gram_ok(gram)) return fail(SRK_EINVAL, "srk_spmm_block: bad gram mode");
  if (adjoint && !A->m.has_adj) return fail(SRK_EUNSUPPORTED, "srk_spmm_block: matrix created without adjoint");
  if (gram != SRK_GRAM_NONE && (!gram_out || (gram != SRK_GRAM_NORM2 && gram != SRK_GRAM_COLNORM2 && !Y)))
    return fail(SRK_EINVAL, "srk_spmm_block: gram needs Y and gram_out");
  Eng e;
  e.c = &ctx->c;
  e.A = &A->m;
  e.cplx = A->m.cplx;
  e.n = A->m.n;
  e.ws = reinterpret_cast<double*>(gram_out);
  int r;
  // (Eng::spmm takes a FULL Gram with s >= 8 to the tensor cores after the product:
  // config 5, s = 16: 2.0 ms fused FMA epilogue vs ~0.2 ms DMMA pass)
  std::vector<RQ> reds;
  if (gram != SRK_GRAM_NONE) reds.push_back(RQ{gram, 0, -1, Y, 0});
  r = e.spmm(adjoint != 0, P, Q, s, reds);
  return check_cuda(r, "srk_spmm_block");
}

int srk_gram_block(srk_ctx* ctx, const void* X, const void* Y, int64_t n, int s, int dtype, int gram, void* out) {
  if (!ctx || !X || !out) return fail(SRK_EINVAL, "srk_gram_block: null argument");
  if (s < 1 || s > 64 || n < 1) return fail(SRK_EDIM, "srk_gram_block: bad n or s");
  if (!gram_ok(gram) || gram == SRK_GRAM_NONE) return fail(SRK_EINVAL, "srk_gram_block: bad gram mode");
  if (gram != SRK_GRAM_NORM2 && gram != SRK_GRAM_COLNORM2 && !Y) return fail(SRK_EINVAL, "srk_gram_block: Y needed");
  const bool cplx = dtype == SRK_C128;
  Eng e;
  e.c = &ctx->c;
  e.cplx = cplx;
  e.n = n;
  e.ws = reinterpret_cast<double*>(out);
  int r;
  if (gram == SRK_GRAM_SUMVEC) r = e.upd(s, {X}, {}, {RQ{gram, 0, -1, Y, 0}});
  else if (gram == SRK_GRAM_NORM2 || gram == SRK_GRAM_COLNORM2) r = e.upd(s, {X}, {}, {RQ{gram, 0, -1, nullptr, 0}});
  else if (gram == SRK_GRAM_FULL && s >= 8) r = e.gram_full(X, Y ? Y : X, s, 0);  // s >= 8: DMMA, as the solvers
  else r = e.upd(s, {X, Y}, {}, {RQ{gram, 0, 1, nullptr, 0}});
  return check_cuda(r, "srk_gram_block");
}

int srk_block_update(srk_ctx* ctx, void* Yout, const void* Yin, const void* X, const void* coef, int kind, int sign,
                     int64_t n, int s, int dtype) {
  if (!ctx || !Yout || !Yin || !X || !coef) return fail(SRK_EINVAL, "srk_block_update: null argument");
  if (s < 1 || s > 64 || n < 1) return fail(SRK_EDIM, "srk_block_update: bad n or s");
  if (kind != SRK_COEF_SCALAR && kind != SRK_COEF_DIAG && kind != SRK_COEF_FULL)
    return fail(SRK_EINVAL, "srk_block_update: bad coefficient kind");
  if (sign != 1 && sign != -1) return fail(SRK_EINVAL, "srk_block_update: sign must be +1 or -1");
  Eng e;
  e.c = &ctx->c;
  e.cplx = dtype == SRK_C128;
  e.n = n;
  e.ws = reinterpret_cast<double*>(const_cast<void*>(coef));
  Coef cf{kind, 0, sign < 0 ? 1 : 0, 0, 0};
  int r = e.upd(s, {Yin, X}, {OutSpec{Yout, {{0, C1()}, {1, cf}}}}, {});
  return check_cuda(r, "srk_block_update");
}

namespace {
struct TsqrSolver : Solver {
  int alloc() override { return 0; }
  int init() override { return 0; }
  void seg(int) override {}
};
}  // namespace

static void fill_opts(srk_opts* o, const srk_opts* in) {
  o->tol = 1e-8;
  o->maxit = 2000;
  o->poll_every = 8;
  o->record_history = 1;
  o->check_true_residual = 1;
  o->use_graph = 1;
  o->x0_zero = 0;
  if (in) {
    if (in->tol > 0) o->tol = in->tol;
    if (in->maxit > 0) o->maxit = in->maxit;
    if (in->poll_every > 0) o->poll_every = in->poll_every;
    o->record_history = in->record_history;
    o->check_true_residual = in->check_true_residual;
    o->use_graph = in->use_graph;
    o->x0_zero = in->x0_zero;
    o->shadow = in->shadow;
    o->shadow_given = in->shadow_given;
    o->preprocess_rhs = in->preprocess_rhs;
    o->eps_brk = in->eps_brk;
    o->eps_defl = in->eps_defl;
    o->rank_policy = in->rank_policy;
    o->trace_iterates = in->on_iter ? std::max(0, in->trace_iterates) : 0;
    o->on_iter = o->trace_iterates > 0 ? in->on_iter : nullptr;
    o->user = o->trace_iterates > 0 ? in->user : nullptr;
    if (o->trace_iterates > 0) o->record_history = 1;  // the callback's residual norm
  }
}

int srk_tsqr(srk_ctx* ctx, const void* Z, void* Q, void* C, int64_t n, int s, int dtype, int* rank_host) {
  if (!ctx || !Z || !Q || !C) return fail(SRK_EINVAL, "srk_tsqr: null argument");
  if (s < 1 || s > 64 || n < s) return fail(SRK_EDIM, "srk_tsqr: need 1 <= s <= 64 and n >= s");
  const bool cplx = dtype == SRK_C128;
  if (!full_supported(cplx, cap_for(s))) return fail(SRK_EUNSUPPORTED, "srk_tsqr: s <= 32");
  TsqrSolver T;
  T.c = &ctx->c;
  T.s = s;
  T.n = n;
  T.cplx = cplx;
  T.method = M_BL_BICG_RQ;
  fill_opts(&T.o, nullptr);
  T.o.maxit = 1;
  int r = T.setup();
  if (r) return fail(r, "srk_tsqr: setup");
  cudaMemsetAsync(T.ctl, 0, CTL_SIZE * sizeof(int), ctx->c.st);
  Eng& e = T.e;
  e.upd(s, {Z}, {OutSpec{nullptr, {{0, C1()}}}}, {RQ{RED_FULL, O0, O0, nullptr, T.off[SL_GZ]}});
  T.coef(10);
  e.upd(s, {Z}, {OutSpec{Q, {{0, FU(T.off[SL_R1I])}}}}, {RQ{RED_FULL, O0, O0, nullptr, T.off[SL_GZ]}});
  T.coef(11);
  e.upd(s, {Q}, {OutSpec{Q, {{0, FU(T.off[SL_R2I])}}}}, {});
  cudaMemcpyAsync(C, T.ws + T.off[SL_C], (size_t)s * s * (cplx ? 16 : 8), cudaMemcpyDeviceToDevice, ctx->c.st);
  if (T.read_ctl()) return cuda_fail((cudaError_t)T.e.err, "srk_tsqr");
  if (rank_host) *rank_host = (T.ctl_host[CTL_FLAG] == FLAG_BRK) ? s - 1 : s;
  return SRK_OK;
}

// ------------------------------------------------------------------ solver
int srk_solver_create(srk_ctx* ctx, const srk_matrix* A, int s, int method, const srk_opts* opts, srk_solver** out) {
  if (!ctx || !A || !out) return fail(SRK_EINVAL, "srk_solver_create: null argument");
  if (s < 1 || s > 64) return fail(SRK_EDIM, "srk_solver_create: s must be in [1, 64]");
  if (method < 0 || method > SRK_BL_BICGSTAB_SQ) return fail(SRK_EINVAL, "srk_solver_create: unknown method");
  if (opts && (opts->tol < 0 || opts->maxit < 0)) return fail(SRK_EINVAL, "srk_solver_create: tol/maxit");
  const bool needs_adj = !(method == SRK_LI_BICGSTAB || method == SRK_GL_BICGSTAB || method == SRK_BL_BICGSTAB ||
                           method == SRK_BL_BICGSTAB_RQ || method == SRK_BL_BICGSTAB_SQ);
  if (needs_adj && !A->m.has_adj) return fail(SRK_EUNSUPPORTED, "srk_solver_create: method needs A^H (need_adjoint=1)");
  const bool block = method == SRK_BL_BICG || method == SRK_BL_BICG_RQ || method == SRK_BL_QMR ||
                     method == SRK_BL_BICGSTAB || method == SRK_BL_BICGSTAB_RQ || method == SRK_BL_BICG_SQ ||
                     method == SRK_BL_BICGSTAB_SQ;
  if (opts && (opts->rank_policy < 0 || opts->rank_policy > 1)) return fail(SRK_EINVAL, "srk_solver_create: rank_policy");
  if (opts && (opts->eps_brk < 0 || opts->eps_defl < 0)) return fail(SRK_EINVAL, "srk_solver_create: eps");
  if (opts && opts->rank_policy && method != SRK_BL_BICG_RQ && method != SRK_BL_BICGSTAB_RQ)
    return fail(SRK_EUNSUPPORTED, "srk_solver_create: rank_policy 1 applies to the rQ variants");
  if (block && !full_supported(A->m.cplx, cap_for(s)))
    return fail(SRK_EUNSUPPORTED, "srk_solver_create: block methods need s <= 32");
  if (A->m.bsr && !bsr_supported(A->m.bs, A->m.cplx, s))
    return fail(SRK_EUNSUPPORTED, "srk_solver_create: BSR operators take s in {4, 8, 12, 16}");
  Solver* sv = make_solver(method);
  if (!sv) return fail(SRK_EINVAL, "srk_solver_create: unknown method");
  sv->c = &ctx->c;
  sv->A = &A->m;
  sv->s = s;
  sv->method = method;
  sv->cplx = A->m.cplx;
  sv->n = A->m.n;
  fill_opts(&sv->o, opts);
  int r = sv->setup();
  if (r) {
    delete sv;
    return fail(r, "srk_solver_create: out of device memory");
  }
  auto* h = new srk_solver();
  h->sv = sv;
  *out = h;
  return SRK_OK;
}

int srk_solver_destroy(srk_solver* h) {
  if (!h) return SRK_OK;
  delete h->sv;
  delete h;
  return SRK_OK;
}

int srk_solver_start(srk_solver* h, const void* B, const void* X0) {
  if (!h || !B) return fail(SRK_EINVAL, "srk_solver_start: null argument");
  int r = h->sv->start(B, X0);
  if (r) return check_cuda(h->sv->e.err ? h->sv->e.err : (int)cudaErrorUnknown, "srk_solver_start");
  return SRK_OK;
}

int srk_solver_iterate(srk_solver* h, int k, int* state) {
  if (!h) return fail(SRK_EINVAL, "srk_solver_iterate: null solver");
  if (k < 0) return fail(SRK_EINVAL, "srk_solver_iterate: k < 0");
  int r = h->sv->iterate(k);
  if (r) return check_cuda(h->sv->e.err ? h->sv->e.err : (int)cudaErrorUnknown, "srk_solver_iterate");
  if (state) *state = h->sv->state;
  return SRK_OK;
}

int srk_solver_get_x(srk_solver* h, void* X) {
  if (!h || !X) return fail(SRK_EINVAL, "srk_solver_get_x: null argument");
  Solver* sv = h->sv;
  if (sv->A && sv->A->prec) {  // X = M^-1 Y (right preconditioning)
    if (sv->e.prec_solve(false, sv->X, X, sv->s)) return fail(SRK_ECUDA, "srk_solver_get_x: preconditioner");
  } else {
    cudaMemcpyAsync(X, sv->X, (size_t)sv->n * sv->s * sv->esz(), cudaMemcpyDeviceToDevice, sv->c->st);
  }
  if (sv->o.preprocess_rhs) {  // X = Y C_B (the solution for the original B)
    const int* saved = sv->e.done;
    sv->e.done = nullptr;
    sv->e.upd(sv->s, {X}, {OutSpec{X, {{0, FU(sv->off[SL_CB])}}}}, {});
    sv->e.done = saved;
  }
  cudaError_t e = cudaStreamSynchronize(sv->c->st);
  return e == cudaSuccess ? SRK_OK : cuda_fail(e, "srk_solver_get_x");
}

int srk_solver_get_residual(srk_solver* h, void* out, int64_t* rows) {
  if (!h || !out) return fail(SRK_EINVAL, "srk_solver_get_residual: null argument");
  int r = h->sv->residual(out, rows);
  return r ? fail(r, "srk_solver_get_residual") : SRK_OK;
}

// Vector operations of k iterations in Proposition 1's convention (an inner
// product or a SAXPY of length n counts one; the s x s algebra is neglected):
// BiCG 7s (Li / Gl) and 7s^2 (Bl) as the proposition states; the other variants by the
// same count of their step lists (a thin QR counts 3s^2; QMR's
// first iteration skips the P / Q and D / S recurrences). A BiCGStab half-step exit is
// counted as a whole iteration.
static int64_t vector_ops(int m, int64_t s, int64_t k) {
  const int64_t s2 = s * s;
  switch (m) {
    case SRK_LI_BICG: case SRK_GL_BICG: return 7 * s * k;
    case SRK_EGL_BICG: return (5 * s + 2) * k;
    case SRK_BL_BICG: return 7 * s2 * k;
    case SRK_BL_BICG_RQ: return 13 * s2 * k;
    case SRK_LI_QMR: case SRK_GL_QMR: return k > 0 ? 10 * s * k - 2 * s : 0;
    case SRK_EGL_QMR: return k > 0 ? (8 * s + 2) * k - (s + 1) : 0;
    case SRK_BL_QMR: return k > 0 ? 16 * s2 * k - 2 * s2 : 0;
    case SRK_LI_BICGSTAB: case SRK_GL_BICGSTAB: return 10 * s * k;
    case SRK_BL_BICGSTAB: return (6 * s2 + 5 * s) * k;
    case SRK_BL_BICGSTAB_RQ: return (12 * s2 + s) * k;
    case SRK_BL_BICG_SQ: return 16 * s2 * k;
    case SRK_BL_BICGSTAB_SQ: return (9 * s2 + 5 * s) * k;
    default: return 0;
  }
}

int srk_solver_report(srk_solver* h, srk_report* rep) {
  if (!h || !rep) return fail(SRK_EINVAL, "srk_solver_report: null argument");
  Solver* sv = h->sv;
  memset(rep, 0, sizeof(*rep));
  if (sv->read_ctl()) return cuda_fail((cudaError_t)sv->e.err, "srk_solver_report");
  const int it = sv->ctl_host[CTL_ITER];
  rep->iterations = it;
  rep->half_step = sv->half;
  rep->breakdown_kind = sv->state == 2 ? sv->brk_kind : 0;
  rep->breakdown_iter = sv->state == 2 ? sv->brk_iter : -1;
  rep->frozen_cols = sv->ctl_host[CTL_NFROZEN];
  rep->matvec_cols_A = (int64_t)it * sv->cols_A - (sv->half ? sv->s : 0);
  rep->matvec_cols_AH = (int64_t)it * sv->cols_AH;
  rep->final_true_rel_residual = sv->true_rel(sv->X);
  double last = 0.0;
  if (it > 0 && it <= sv->hist_cap) cudaMemcpy(&last, sv->hist + (it - 1), sizeof(double), cudaMemcpyDeviceToHost);
  rep->final_recursive_rel_residual = last;
  rep->seconds = sv->seconds;
  rep->kernel_launches = sv->launches;
  rep->vector_ops = vector_ops(sv->method, sv->s, it);
  rep->deflated_cols = sv->ctl_host[CTL_DEFL];
  rep->breakdown_col = -1;
  for (int c = 0; c < sv->s && c < 64; ++c)
    if (sv->ctl_host[CTL_FROZEN + c]) {
      rep->breakdown_col = c;
      break;
    }
  if (sv->state == 1) rep->outcome = SRK_CONVERGED;
  else if (sv->state == 2) rep->outcome = SRK_BREAKDOWN;
  else rep->outcome = rep->final_true_rel_residual > 1.0 ? SRK_DIVERGED : SRK_MAXIT;
  return SRK_OK;
}

int srk_solver_profile(srk_solver* h, int enable) {
  if (!h) return fail(SRK_EINVAL, "srk_solver_profile: null solver");
  h->sv->prof.on = enable != 0;
  h->sv->prof.used = 0;
  return SRK_OK;
}

int srk_solver_profile_read(srk_solver* h, double* ms_host, int64_t* count_host, int ntag) {
  if (!h || !ms_host || !count_host) return fail(SRK_EINVAL, "srk_solver_profile_read: null argument");
  std::vector<long long> cnt(ntag);
  h->sv->prof.read(ms_host, cnt.data(), ntag);
  for (int i = 0; i < ntag; ++i) count_host[i] = cnt[i];
  return SRK_OK;
}

int srk_solver_profile_launches(srk_solver* h, int32_t* tag_host, int32_t* sig_host, double* ms_host,
                                double* bytes_host, int max_records) {
  if (!h || !tag_host || !sig_host || !ms_host || !bytes_host || max_records < 0)
    return fail(SRK_EINVAL, "srk_solver_profile_launches: null argument");
  return h->sv->prof.read_launches(tag_host, sig_host, ms_host, bytes_host, max_records);
}

int srk_solver_history(srk_solver* h, double* hist_host, int cap) {
  if (!h || !hist_host) return fail(SRK_EINVAL, "srk_solver_history: null argument");
  Solver* sv = h->sv;
  const int n = std::min(cap, sv->hist_cap);
  cudaError_t e = cudaMemcpy(hist_host, sv->hist, sizeof(double) * n, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? SRK_OK : cuda_fail(e, "srk_solver_history");
}

int srk_solve(srk_ctx* ctx, const srk_matrix* A, const void* B, void* X, int s, int method, const srk_opts* opts,
              srk_report* rep) {
  if (!ctx || !A || !B || !X) return fail(SRK_EINVAL, "srk_solve: null argument");
  srk_opts o{};
  fill_opts(&o, opts);
  srk_solver* h = nullptr;
  if (ctx->cached && ctx->cached_mat == A->id && ctx->cached_s == s && ctx->cached_method == method &&
      std::memcmp(&ctx->cached_opts, &o, sizeof o) == 0) {
    h = ctx->cached;  // same operator, width, method and options: reuse the workspace
  } else {
    drop_cache(ctx);
    int r = srk_solver_create(ctx, A, s, method, &o, &h);
    if (r) return r;
    ctx->cached = h;
    ctx->cached_mat = A->id;
    ctx->cached_s = s;
    ctx->cached_method = method;
    ctx->cached_opts = o;
  }
  int r = srk_solver_start(h, B, o.x0_zero ? nullptr : X);
  if (!r && o.trace_iterates > 0 && o.on_iter) {  // the first K iterations one at a time, with the callback
    const size_t bytes = (size_t)A->m.n * s * (A->m.cplx ? 16 : 8);
    void *Xt = nullptr, *Rt = nullptr;
    if (cudaMalloc(&Xt, bytes) != cudaSuccess || cudaMalloc(&Rt, bytes) != cudaSuccess) {
      if (Xt) cudaFree(Xt);
      drop_cache(ctx);
      return fail(SRK_ENOMEM, "srk_solve: out of device memory (trace_iterates)");
    }
    int state = 0;
    for (int k = 1; !r && k <= o.trace_iterates && k <= o.maxit && state == 0; ++k) {
      r = srk_solver_iterate(h, 1, &state);
      int64_t rows = 0;
      if (!r) r = srk_solver_get_x(h, Xt);
      if (!r) r = srk_solver_get_residual(h, Rt, &rows);
      double sc[2] = {-1.0, (double)state};
      int it = 0;
      if (!r && !h->sv->read_ctl()) it = h->sv->ctl_host[CTL_ITER];
      if (!r && it >= 1 && it <= h->sv->hist_cap) {
        std::vector<double> hist((size_t)it);
        if (srk_solver_history(h, hist.data(), it) == SRK_OK) sc[0] = hist.back();
      }
      if (!r) r = check_cuda((int)cudaStreamSynchronize(ctx->c.st), "srk_solve");
      if (!r && it >= k) o.on_iter(k, Xt, Rt, rows, sc, o.user);  // (a breakdown inside iteration k: no iterate k)
    }
    cudaFree(Xt);
    cudaFree(Rt);
  }
  if (!r) r = srk_solver_iterate(h, h->sv->o.maxit, nullptr);
  if (!r) r = srk_solver_get_x(h, X);
  if (!r && rep) r = srk_solver_report(h, rep);
  if (r) drop_cache(ctx);
  return r;
}

int srk_solve_host(srk_ctx* ctx, const srk_matrix* A, const void* B_host, void* X_host, int s, int method,
                   const srk_opts* opts, srk_report* rep) {
  if (!ctx || !A || !B_host || !X_host) return fail(SRK_EINVAL, "srk_solve_host: null argument");
  const size_t bytes = (size_t)A->m.n * s * (A->m.cplx ? 16 : 8);
  if (ctx->hcap < bytes) {  // staging blocks, kept by the context
    for (void*& p : ctx->hbuf) {
      if (p) cudaFree(p);
      p = nullptr;
    }
    ctx->hcap = 0;
    if (cudaMalloc(&ctx->hbuf[0], bytes) != cudaSuccess || cudaMalloc(&ctx->hbuf[1], bytes) != cudaSuccess)
      return fail(SRK_ENOMEM, "srk_solve_host: out of device memory");
    ctx->hcap = bytes;
  }
  void *Bd = ctx->hbuf[0], *Xd = ctx->hbuf[1];
  cudaMemcpyAsync(Bd, B_host, bytes, cudaMemcpyHostToDevice, ctx->c.st);
  if (!(opts && opts->x0_zero)) cudaMemcpyAsync(Xd, X_host, bytes, cudaMemcpyHostToDevice, ctx->c.st);
  int r = srk_solve(ctx, A, Bd, Xd, s, method, opts, rep);
  if (!r) {
    cudaMemcpyAsync(X_host, Xd, bytes, cudaMemcpyDeviceToHost, ctx->c.st);
    cudaError_t e = cudaStreamSynchronize(ctx->c.st);
    if (e != cudaSuccess) r = cuda_fail(e, "srk_solve_host");
  }
  return r;
}

}  // extern "C"
