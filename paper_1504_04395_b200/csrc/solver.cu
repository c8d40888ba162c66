// solver.cu — host drivers of the 13 simultaneous methods. Each iteration is
// enqueued as a fixed sequence of block kernels (SpMM with fused Grams, fused
// block updates) and single-CTA coefficient phases, all on one stream with no
// host synchronisation; the host polls a device flag every `poll_every`
// iterations (kernels after a raised flag are no-ops). Step lists follow
// PAPER.md Alg. 1-5 and SURVEY App. A (the same order as oracle/solvers.py,
// with which this file shares no code).
#include <chrono>
#include <cstring>

#include "solver.h"

namespace srk {

static size_t slot_doubles(int s) {
  size_t v = (size_t)4 * s * s * 2;  // (2s x 2s) complex: the Bl-QMR unitary
  if (v < 128) v = 128;
  return v;
}

Solver::~Solver() {
  if (gexec) cudaGraphExecDestroy(gexec);
  if (cap_st) cudaStreamDestroy(cap_st);
  for (void* p : owned) cudaFree(p);
  if (ws) cudaFree(ws);
  if (wstage) cudaFree(wstage);
  if (ctl) cudaFree(ctl);
  if (hist) cudaFree(hist);
  if (ctl_host) cudaFreeHost(ctl_host);
}

// blocks carry a tail of ghost rows (multi-GPU: filled by the halo exchange before each SpMM)
void* Solver::blk() {
  void* p = nullptr;
  const size_t rows = (size_t)(n + (A ? A->ghost_rows() : 0));
  if (cudaMalloc(&p, rows * s * esz()) != cudaSuccess) return nullptr;
  owned.push_back(p);
  return p;
}
void* Solver::vecn() {
  void* p = nullptr;
  const size_t rows = (size_t)(n + (A ? A->ghost_rows() : 0));
  if (cudaMalloc(&p, rows * esz()) != cudaSuccess) return nullptr;
  owned.push_back(p);
  return p;
}

int Solver::setup() {
  const size_t sd = slot_doubles(s);
  for (int i = 0; i < NSLOT; ++i) off[i] = (int)(i * sd);
  if (cudaMalloc(&ws, sd * NSLOT * sizeof(double)) != cudaSuccess) return SRK_ENOMEM;
  cudaMemset(ws, 0, sd * NSLOT * sizeof(double));
  if (c->comm && c->comm->nranks > 1) {  // per-rank sums staged before each allreduce (engine.cu)
    if (cudaMalloc(&wstage, sd * NSLOT * sizeof(double)) != cudaSuccess) return SRK_ENOMEM;
    cudaMemset(wstage, 0, sd * NSLOT * sizeof(double));
  }
  if (cudaMalloc(&ctl, CTL_SIZE * sizeof(int)) != cudaSuccess) return SRK_ENOMEM;
  if (cudaMallocHost(&ctl_host, CTL_SIZE * sizeof(int)) != cudaSuccess) return SRK_ENOMEM;
  hist_cap = o.maxit + 2;
  if (cudaMalloc(&hist, sizeof(double) * hist_cap) != cudaSuccess) return SRK_ENOMEM;
  e.c = c;
  e.A = A;
  e.cplx = cplx;
  e.n = n;
  e.ws = ws;
  e.wstage = wstage;
  e.done = ctl + CTL_FLAG;
  e.prof = &prof;
  B = blk();
  X = blk();
  R = blk();
  tmp = blk();
  if (!B || !X || !R || !tmp) return SRK_ENOMEM;
  return alloc();
}

int Solver::coef(int phase, int k1) {
  if (e.err) return e.err;
  CoefArgs a{};
  a.method = method;
  a.phase = phase;
  a.s = s;
  a.k1 = k1;
  a.tol = o.tol;
  a.defl = o.rank_policy;
  a.eps_brk = eps_brk();
  a.eps_chol = eps_chol();
  a.ws = ws;
  a.ctl = ctl;
  a.hist = hist;
  a.hist_cap = hist_cap;
  for (int i = 0; i < NSLOT; ++i) a.off[i] = off[i];
  const size_t sm = (size_t)(3 * s * s + 64) * esz() + 1024;
  e.nlaunch++;
  prof.begin(PT_COEF, c->st);
  e.err = launch_coef(cplx, a, sm, c->st);
  prof.end(c->st);
  return e.err;
}

int Solver::read_ctl() {
  cudaMemcpyAsync(ctl_host, ctl, CTL_SIZE * sizeof(int), cudaMemcpyDeviceToHost, c->st);
  cudaError_t err = cudaStreamSynchronize(c->st);
  if (err != cudaSuccess) return e.err = (int)err;
  return e.err;
}

// ||B - A Xc||_F / ||R0||_F, computed with the same kernels (reading G26)
double Solver::true_rel(const void* Xc) {
  const int* saved = e.done;
  e.done = nullptr;
  e.spmm(false, Xc, tmp, s, {});
  e.upd(s, {B, tmp}, {OutSpec{nullptr, {{0, C1()}, {1, Coef{CK_ONE, 0, 1, 0, 0}}}}},
        {RQ{RED_NORM2, O0, -1, nullptr, off[SL_TRUE]}});
  e.done = saved;
  double v[2] = {0, 0};
  cudaMemcpyAsync(v, ws + off[SL_TRUE], sizeof(double), cudaMemcpyDeviceToHost, c->st);
  cudaMemcpyAsync(v + 1, ws + off[SL_R0N], sizeof(double), cudaMemcpyDeviceToHost, c->st);
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return -1.0;
  if (v[1] == 0.0) return 0.0;
  return sqrt(v[0]) / v[1];
}

__global__ static void ctl_init_kernel(int* ctl) { ctl[CTL_DIDLE] = 1; }
static void dev_tsqr(Solver& S, const void* Z, void* Q, bool hat, void* zsave = nullptr);

int Solver::start(const void* Bd, const void* X0d) {
  cudaStream_t st = c->st;
  if (o.preprocess_rhs && X0d) return SRK_EUNSUPPORTED;  // X0 = 0 with the QR preprocessing
  cudaMemcpyAsync(B, Bd, (size_t)n * s * esz(), cudaMemcpyDeviceToDevice, st);
  cudaMemsetAsync(ctl, 0, CTL_SIZE * sizeof(int), st);
  ctl_init_kernel<<<1, 1, 0, st>>>(ctl);  // CTL_DIDLE = 1: no thin-QR repair pending (f4)
  if (o.preprocess_rhs) {  // B = Q C_B; solve A Y = Q and return X = Y C_B (reading G9)
    dev_tsqr(*this, B, B, false);
    cudaMemcpyAsync(ws + off[SL_CB], ws + off[SL_C], (size_t)s * s * esz(), cudaMemcpyDeviceToDevice, st);
  }
  host_iter = 0;
  state = 0;
  half = 0;
  brk_kind = 0;
  brk_iter = -1;
  frozen = 0;
  final_true = final_rec = -1.0;
  e.err = 0;
  e.nlaunch = 0;
  if (X0d) {
    // right preconditioning iterates on Y = M X: Y0 = M X0 (then R0 = B - A M^-1 Y0 = B - A X0)
    if (A && A->prec) e.prec_mul(X0d, X, s);
    else cudaMemcpyAsync(X, X0d, (size_t)n * s * esz(), cudaMemcpyDeviceToDevice, st);
    e.spmm(false, X, tmp, s, {});
    e.upd(s, {B, tmp}, {OutSpec{R, {{0, C1()}, {1, Coef{CK_ONE, 0, 1, 0, 0}}}}},
          {RQ{RED_NORM2, O0, -1, nullptr, off[SL_R0N2]}});
  } else {
    cudaMemsetAsync(X, 0, (size_t)n * s * esz(), st);
    e.upd(s, {B}, {OutSpec{R, {{0, C1()}}}}, {RQ{RED_NORM2, O0, -1, nullptr, off[SL_R0N2]}});
  }
  coef(9);  // ||R0|| (and the R0 = 0 shortcut)
  int r = init();
  if (r) return r;
  started = true;
  if (e.err) return SRK_ECUDA;
  return SRK_OK;
}

int Solver::iterate(int k) {
  if (!started) return SRK_EINVAL;
  if (state != 0) return SRK_OK;
  auto t0 = std::chrono::steady_clock::now();
  const int poll = o.poll_every > 0 ? o.poll_every : 8;
  // device iteration count = host_iter at every poll point
  if (read_ctl()) return SRK_ECUDA;
  int dev_iter = ctl_host[CTL_ITER];
  const int target = std::min(dev_iter + k, o.maxit);
  host_iter = dev_iter;
  while (true) {
    int flag = ctl_host[CTL_FLAG];
    dev_iter = ctl_host[CTL_ITER];
    if (flag == FLAG_RUN) {
      if (dev_iter >= target) {
        if (dev_iter >= o.maxit) state = 3;
        break;
      }
      host_iter = dev_iter;
      int launched = 0;
      while (host_iter < target && launched < poll) {
        // a method with a whole-iteration kernel runs the remaining iterations in one launch
        // (the kernel stops by itself once the control flag leaves RUN, so the host polls
        // right after a convergence candidate, a breakdown or the last iteration)
        if (const int m = seg_multi(std::min(target - host_iter, 4096)); m > 0) {
          host_iter += m;
          launched += m;
          continue;
        }
        // after the first iteration every iteration launches the same kernels with the
        // same arguments: replay a captured CUDA graph of `poll` iterations
        // (not across ranks: the NCCL calls stay eager, capture is validated on one GPU only)
        const bool multi = c->comm && c->comm->nranks > 1;
        if (o.use_graph && !multi && !prof.on && host_iter > 0 && launched == 0 && target - host_iter >= poll && poll > 1) {
          if (capture(poll)) return SRK_ECUDA;
          if (cudaGraphLaunch(gexec, c->st) != cudaSuccess) return SRK_ECUDA;
          e.nlaunch += graph_launches;
          host_iter += poll;
          launched += poll;
          continue;
        }
        for (int q = 0; q < nseg(); ++q) seg(q);
        if (!ends_iter()) {
          launch_end_iter(ctl, c->st);
          e.nlaunch++;
        }
        host_iter++;
        launched++;
      }
      if (e.err) return SRK_ECUDA;
      if (read_ctl()) return SRK_ECUDA;
      continue;
    }
    if (flag == FLAG_CONV) {
      const double tr = o.check_true_residual ? true_rel(X) : 0.0;
      if (tr <= o.tol) {
        state = 1;
        break;
      }
      // recursive residual met tol but the true residual does not: continue (G26)
      cudaMemsetAsync(ctl + CTL_FLAG, 0, sizeof(int), c->st);
      if (read_ctl()) return SRK_ECUDA;
      continue;
    }
    if (flag == FLAG_HALF) {
      // BiCGStab half step (S small): X_h = X + P alpha; accept if the true residual agrees
      half_x(tmp2);
      const double tr = o.check_true_residual ? true_rel(tmp2) : 0.0;
      if (tr <= o.tol) {
        cudaMemcpyAsync(X, tmp2, (size_t)n * s * esz(), cudaMemcpyDeviceToDevice, c->st);
        cudaMemsetAsync(ctl + CTL_FLAG, 0, sizeof(int), c->st);
        launch_end_iter(ctl, c->st);  // counts the half iteration
        cudaMemsetAsync(ctl + CTL_FLAG, 0, sizeof(int), c->st);
        half = 1;
        state = 1;
        if (read_ctl()) return SRK_ECUDA;
        break;
      }
      cudaMemsetAsync(ctl + CTL_FLAG, 0, sizeof(int), c->st);
      for (int q = 1; q < nseg(); ++q) seg(q);  // finish this iteration
      launch_end_iter(ctl, c->st);
      if (read_ctl()) return SRK_ECUDA;
      continue;
    }
    if (flag == FLAG_BRK) {
      brk_kind = ctl_host[CTL_BKIND];
      brk_iter = ctl_host[CTL_BITER];
      // a breakdown at an iterate that already satisfies the stopping rule is a lucky breakdown
      const double tr = true_rel(X);
      if (brk_iter > 0 && tr <= o.tol) {
        state = 1;
        cudaMemcpyAsync(ctl + CTL_ITER, &brk_iter, sizeof(int), cudaMemcpyHostToDevice, c->st);
        if (read_ctl()) return SRK_ECUDA;
      } else {
        state = 2;
      }
      break;
    }
    break;
  }
  cudaStreamSynchronize(c->st);
  auto t1 = std::chrono::steady_clock::now();
  seconds += std::chrono::duration<double>(t1 - t0).count();
  launches = e.nlaunch;
  frozen = ctl_host[CTL_NFROZEN];
  if (e.err) return SRK_ECUDA;
  return SRK_OK;
}

// Capture `iters` iterations on a private stream (the caller's stream may be the
// legacy default stream, which cannot be captured) into an executable graph;
// re-captured only if the graph's baked-in scratch buffer moved.
int Solver::capture(int iters) {
  if (gexec && graph_iters == iters && graph_partials == c->partials) return 0;
  if (gexec) {
    cudaGraphExecDestroy(gexec);
    gexec = nullptr;
  }
  if (!cap_st && cudaStreamCreateWithFlags(&cap_st, cudaStreamNonBlocking) != cudaSuccess) return SRK_ECUDA;
  cudaStream_t user = c->st;
  // the scratch partials must not be reallocated inside the capture
  cudaStreamSynchronize(user);
  c->st = cap_st;
  const long long l0 = e.nlaunch;
  cudaGraph_t g = nullptr;
  if (cudaStreamBeginCapture(cap_st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    c->st = user;
    return SRK_ECUDA;
  }
  for (int i = 0; i < iters; ++i) {
    for (int q = 0; q < nseg(); ++q) seg(q);
    if (!ends_iter()) {
      launch_end_iter(ctl, cap_st);
      e.nlaunch++;
    }
  }
  cudaError_t ce = cudaStreamEndCapture(cap_st, &g);
  c->st = user;
  if (ce != cudaSuccess || e.err) return SRK_ECUDA;
  graph_launches = e.nlaunch - l0;
  e.nlaunch = l0;
  ce = cudaGraphInstantiate(&gexec, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) return SRK_ECUDA;
  graph_iters = iters;
  graph_partials = c->partials;
  return 0;
}

int Solver::residual(void* out, int64_t* rows) {
  cudaMemcpyAsync(out, R, (size_t)n * s * esz(), cudaMemcpyDeviceToDevice, c->st);
  if (rows) *rows = n;
  return cudaStreamSynchronize(c->st) == cudaSuccess ? SRK_OK : SRK_ECUDA;
}

// ---------------------------------------------------------------------------
// Rank-deficiency continuation (reading R8): the replacement vectors
// come from a counter-based generator (SplitMix64, the definition oracle/linalg.py's
// counter_uniform also implements — no shared code): vector `key` = event * 64 + column,
// entry i = 2u - 1 with u = (splitmix64(h + 2i + part) >> 11) 2^-53, stream
// h = splitmix64(seed ^ (key * 0x9E3779B97F4A7C15)), part 0 real / 1 imaginary.
// ---------------------------------------------------------------------------
constexpr unsigned long long DEFL_SEED = 0x5EED1504ull;

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double counter_u(unsigned long long h, unsigned long long i, int part) {
  return (double)(splitmix64(h + 2ull * i + (unsigned long long)part) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

// Armed only while a repair is pending (ctl[CTL_DIDLE] == 0): Zsave = Z, and every
// deficient column j of Z (mask in ctl[maskoff..+1]) becomes replacement vector
// (event, j), event = 0 for the initial QR, else 2 k + hat in iteration k.
__global__ void defl_fill_kernel(double* Z, double* Zsave, long long n, int s, int cplx, const int* ctl, int maskoff,
                                 int hat, int init) {
  if (ctl[CTL_DIDLE]) return;
  const unsigned long long m = (unsigned long long)(unsigned)ctl[maskoff] |
                               ((unsigned long long)(unsigned)ctl[maskoff + 1] << 32);
  const unsigned long long event = init ? 0ull : 2ull * (unsigned long long)(ctl[CTL_ITER] + 1) + (unsigned long long)hat;
  const int nd = cplx ? 2 : 1;
  const long long total = n * s;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / s;
    const int c = (int)(e % s);
    for (int p = 0; p < nd; ++p) Zsave[e * nd + p] = Z[e * nd + p];
    if ((m >> c) & 1ull) {
      const unsigned long long key = event * 64ull + (unsigned long long)c;
      const unsigned long long h = splitmix64(DEFL_SEED ^ (key * 0x9E3779B97F4A7C15ull));
      for (int p = 0; p < nd; ++p) Z[e * nd + p] = counter_u(h, (unsigned long long)i, p);
    }
  }
}

// The repair sequence between pass 1 and the rest of a thin QR (all no-ops unless armed):
// fill Z (and Ẑ), the Gram of the modified blocks, phase 20 (redo pass 1, keep C_old).
void Solver::defl_repair(void* Z, void* Zs, void* Zh, void* Zhs, bool init) {
  const int g = std::max(1, std::min(c->nsm * 8, (int)((n * s + 255) / 256)));
  const int* saved = e.done;
  e.done = ctl + CTL_DIDLE;
  defl_fill_kernel<<<g, 256, 0, c->st>>>((double*)Z, (double*)Zs, n, s, cplx, ctl, CTL_DMASK, 0, init);
  e.nlaunch++;
  e.upd(s, {Z}, {}, {RQ{RED_FULL, 0, 0, nullptr, off[SL_GZ]}});
  if (Zh) {
    defl_fill_kernel<<<g, 256, 0, c->st>>>((double*)Zh, (double*)Zhs, n, s, cplx, ctl, CTL_DMASKH, 1, init);
    e.nlaunch++;
    e.upd(s, {Zh}, {}, {RQ{RED_FULL, 0, 0, nullptr, off[SL_GZH]}});
  }
  e.done = saved;
  coef(20, (Zh ? 3 : 1) | (init ? 4 : 0));
}

// After Q (and Q̂) of the modified blocks exist: SIGT = Q^H Z_orig, then phase 21.
void Solver::defl_fixup(const void* Q, const void* Zs, const void* Qh, const void* Zhs, bool init) {
  const int* saved = e.done;
  e.done = ctl + CTL_DIDLE;
  e.upd(s, {Zs, Q}, {}, {RQ{RED_FULL, 0, 1, nullptr, off[SL_SIGT]}});
  if (Qh) e.upd(s, {Zhs, Qh}, {}, {RQ{RED_FULL, 0, 1, nullptr, off[SL_SIGTH]}});
  e.done = saved;
  coef(21, (Qh ? 3 : 1) | (init ? 4 : 0));
}

// ---------------------------------------------------------------------------
// Shadow residuals (srk_opts.shadow): 0 the paper's choice (R̂0 =
// R0, economic r̂0 = mean of the columns), 1 conj(R0) (economic: conj of the mean),
// 2 the column mean (rank-one block r̂0 1^T for the non-economic variants),
// 3 a caller-given block / vector.
// ---------------------------------------------------------------------------
__global__ static void conj_copy_kernel(const double2* src, double2* dst, long long cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x) {
    const double2 v = src[i];
    dst[i] = make_double2(v.x, -v.y);
  }
}
template <typename T>
__global__ static void bcast_cols_kernel(const T* v, T* dst, long long n, int s) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * s; e += (long long)gridDim.x * blockDim.x)
    dst[e] = v[e / s];
}

int Solver::shadow_vec_into(void* dst) {
  const int g = std::max(1, std::min(c->nsm * 8, (int)((n + 255) / 256)));
  if (o.shadow == 3) {
    if (!o.shadow_given) return SRK_EINVAL;
    cudaMemcpyAsync(dst, o.shadow_given, (size_t)n * esz(), cudaMemcpyDeviceToDevice, c->st);
    return 0;
  }
  launch_row_mean(cplx, R, dst, n, s, nullptr, c->st);
  if (o.shadow == 1 && cplx) conj_copy_kernel<<<g, 256, 0, c->st>>>((const double2*)dst, (double2*)dst, n);
  return 0;
}

int Solver::shadow_into(void* dst) {
  const size_t b = (size_t)n * s * esz();
  const int g = std::max(1, std::min(c->nsm * 8, (int)((n * s + 255) / 256)));
  switch (o.shadow) {
    case 0: cudaMemcpyAsync(dst, R, b, cudaMemcpyDeviceToDevice, c->st); return 0;
    case 1:
      if (cplx) conj_copy_kernel<<<g, 256, 0, c->st>>>((const double2*)R, (double2*)dst, n * s);
      else cudaMemcpyAsync(dst, R, b, cudaMemcpyDeviceToDevice, c->st);
      return 0;
    case 2:
      launch_row_mean(cplx, R, tmp, n, s, nullptr, c->st);  // tmp: scratch (its first n entries)
      if (cplx) bcast_cols_kernel<double2><<<g, 256, 0, c->st>>>((const double2*)tmp, (double2*)dst, n, s);
      else bcast_cols_kernel<double><<<g, 256, 0, c->st>>>((const double*)tmp, (double*)dst, n, s);
      return 0;
    case 3:
      if (!o.shadow_given) return SRK_EINVAL;
      cudaMemcpyAsync(dst, o.shadow_given, b, cudaMemcpyDeviceToDevice, c->st);
      return 0;
    default: return SRK_EINVAL;
  }
}

// ---------------------------------------------------------------------------
// device thin QR (CholQR2) used by the rQ variants' initialisation and srk_tsqr
// Phases 10/11 (slots GZ -> R1, C) and 12/13 (GZH -> R1H, CH) of the coefficient kernel.
// ---------------------------------------------------------------------------
// (zsave != null: the rQ rank continuation is on — Z may be modified in place by the repair)
static void dev_tsqr(Solver& S, const void* Z, void* Q, bool hat, void* zsave) {
  Eng& e = S.e;
  const int gz = hat ? SL_GZH : SL_GZ;
  e.upd(S.s, {Z}, {OutSpec{nullptr, {{0, C1()}}}}, {RQ{RED_FULL, O0, O0, nullptr, S.off[gz]}});
  S.coef(hat ? 12 : 10);
  if (zsave) S.defl_repair(const_cast<void*>(Z), zsave, nullptr, nullptr, true);
  e.upd(S.s, {Z}, {OutSpec{Q, {{0, FU(S.off[hat ? SL_R1HI : SL_R1I])}}}}, {RQ{RED_FULL, O0, O0, nullptr, S.off[gz]}});
  S.coef(hat ? 13 : 11);
  e.upd(S.s, {Q}, {OutSpec{Q, {{0, FU(S.off[hat ? SL_R2HI : SL_R2I])}}}}, {});
  if (zsave) S.defl_fixup(Q, zsave, nullptr, nullptr, true);
}

static inline Coef NEG1() { return Coef{CK_ONE, 0, 1, 0, 0}; }

// =============================================================================
// BiCG family
// =============================================================================
struct GlBiCG : Solver {  // Alg. 2 (Gl) and Alg. 1 (Li: diag coefficients)
  bool li = false;
  void *P, *Q, *Rh, *Ph, *Qh;
  int alloc() override {
    P = blk(); Q = blk(); Rh = blk(); Ph = blk(); Qh = blk();
    cols_A = s; cols_AH = s;
    return (P && Q && Rh && Ph && Qh) ? 0 : SRK_ENOMEM;
  }
  int rmode() const { return li ? RED_DIAG : RED_TRACE; }
  Coef K(int slot, int neg = 0, int cj = 0) const { return li ? DG(off[slot], neg, cj) : SC(off[slot], neg, cj); }
  int init() override {
    const size_t b = (size_t)n * s * esz();
    if (int r = shadow_into(Rh)) return r;  // shadow R̂0 (default R0)
    cudaMemcpyAsync(P, R, b, cudaMemcpyDeviceToDevice, c->st);
    cudaMemcpyAsync(Ph, Rh, b, cudaMemcpyDeviceToDevice, c->st);
    e.upd(s, {R, Rh}, {}, {RQ{rmode(), 0, 1, nullptr, off[SL_RHO]}});
    return coef(0);
  }
  void seg(int) override {
    e.spmm(false, P, Q, s, {RQ{rmode(), 0, -1, Ph, off[SL_DEN]}});   // Q = A P ; <q, p̂>
    e.spmm(true, Ph, Qh, s, {});                                     // A^H P̂
    coef(1);
    static const bool no_flat = getenv("SRK_NO_FLAT_UPDATE") != nullptr;  // A/B switch
    if (!li && !no_flat && e.qmr_tail_ok(s)) {  // Gl (scalar coefficients): flat plans (flat_upd.cu)
      e.flat(FP_BICG_XR, s, {X, P, R, Q, Rh, Qh}, {X, R, Rh}, {off[SL_ALPHA], off[SL_ALPHA], off[SL_ALPHA]},
             {off[SL_RHON], off[SL_R2]});
      coef(2);
      // (the reduction-free (P, P^) update stays on upd_kernel: 1.94 ms = 101% of the copy-measured peak
      // on config 3 against 2.05 ms for the flat plan FP_BICG_P)
      e.upd(s, {R, P, Rh, Ph},
            {OutSpec{P, {{0, C1()}, {1, K(SL_BETA)}}}, OutSpec{Ph, {{2, C1()}, {3, K(SL_BETA, 0, 1)}}}}, {});
      return;
    }
    e.upd(s, {X, P, R, Q, Rh, Qh},
          {OutSpec{X, {{0, C1()}, {1, K(SL_ALPHA)}}},
           OutSpec{R, {{2, C1()}, {3, K(SL_ALPHA, 1)}}},
           OutSpec{Rh, {{4, C1()}, {5, K(SL_ALPHA, 1, 1)}}}},
          {RQ{rmode(), O1, O2, nullptr, off[SL_RHON]}, RQ{RED_NORM2, O1, -1, nullptr, off[SL_R2]}});
    coef(2);
    e.upd(s, {R, P, Rh, Ph},
          {OutSpec{P, {{0, C1()}, {1, K(SL_BETA)}}}, OutSpec{Ph, {{2, C1()}, {3, K(SL_BETA, 0, 1)}}}}, {});
  }
};

struct EglBiCG : Solver {  // Alg. 4
  void *P, *Q, *rh, *ph, *qh;
  int alloc() override {
    P = blk(); Q = blk(); rh = vecn(); ph = vecn(); qh = vecn();
    cols_A = s; cols_AH = 1;
    return (P && Q && rh && ph && qh) ? 0 : SRK_ENOMEM;
  }
  int init() override {
    cudaMemcpyAsync(P, R, (size_t)n * s * esz(), cudaMemcpyDeviceToDevice, c->st);
    if (int r = shadow_vec_into(rh)) return r;  // r̂0 (default: mean of the columns)
    cudaMemcpyAsync(ph, rh, (size_t)n * esz(), cudaMemcpyDeviceToDevice, c->st);
    e.upd(s, {R}, {}, {RQ{RED_SUMVEC, 0, -1, rh, off[SL_RHO]}});
    return coef(0);
  }
  // small operators (latency-bound): the whole iteration as one single-CTA kernel
  bool small() const {
    static const bool off_env = getenv("SRK_NO_SMALL_KERNEL") != nullptr;  // A/B switch
    return !off_env && A && !A->bsr && !A->prec && A->ghost_rows() == 0 && A->has_adj && n <= SMALL_N_MAX &&
           !(c->comm && c->comm->nranks > 1);
  }
  bool ends_iter() const override { return small(); }
  int seg_multi(int k) override {
    if (!small() || k < 1 || e.err) return 0;
    launch_small(k);
    return k;
  }
  void launch_small(int iters) {
    SmallBiCGArgs g{};
    g.rp = A->rp;
    g.ci = A->ci;
    g.val = A->val;
    g.rpH = A->rpH;
    g.ciH = A->ciH;
    g.valH = A->valH;
    g.X = X; g.R = R; g.P = P; g.Q = Q; g.rh = rh; g.ph = ph; g.qh = qh;
    g.n = n;
    g.iters = iters;
    g.ca.method = method;
    g.ca.s = s;
    g.ca.tol = o.tol;
    g.ca.eps_brk = eps_brk();
    g.ca.eps_chol = eps_chol();
    g.ca.ws = ws;
    g.ca.ctl = ctl;
    g.ca.hist = hist;
    g.ca.hist_cap = hist_cap;
    for (int i = 0; i < NSLOT; ++i) g.ca.off[i] = off[i];
    e.nlaunch++;
    prof.begin(PT_OTHER, c->st);
    e.err = launch_egl_bicg_small(cplx, g, c->st);
    prof.end(c->st);
  }
  void seg(int) override {
    if (small()) {
      if (!e.err) launch_small(1);
      return;
    }
    e.spmm(false, P, Q, s, {RQ{RED_SUMVEC, 0, -1, ph, off[SL_DEN]}});  // sum(p̂^H Q)
    e.spmm(true, ph, qh, 1, {});                                        // A^H p̂ (one vector)
    coef(1);
    static const bool no_lean = getenv("SRK_NO_FLAT_UPDATE") != nullptr;  // A/B switch
    if (!no_lean && e.qmr_vec_ok(s)) {
      // the two block updates as lean flat kernels that carry r̂ and p̂ (egl_flat.cu)
      e.egl_bicg_flat(0, s, X, R, P, Q, rh, ph, qh, off[SL_ALPHA], off[SL_BETA], off[SL_RHON], off[SL_R2]);
      coef(2);
      e.egl_bicg_flat(1, s, X, R, P, Q, rh, ph, qh, off[SL_ALPHA], off[SL_BETA], off[SL_RHON], off[SL_R2]);
      return;
    }
    e.upd(1, {rh, qh}, {OutSpec{rh, {{0, C1()}, {1, SC(off[SL_ALPHA], 1, 1)}}}}, {});
    e.upd(s, {X, P, R, Q},
          {OutSpec{X, {{0, C1()}, {1, SC(off[SL_ALPHA])}}}, OutSpec{R, {{2, C1()}, {3, SC(off[SL_ALPHA], 1)}}}},
          {RQ{RED_SUMVEC, O1, -1, rh, off[SL_RHON]}, RQ{RED_NORM2, O1, -1, nullptr, off[SL_R2]}});
    coef(2);
    e.upd(s, {R, P}, {OutSpec{P, {{0, C1()}, {1, SC(off[SL_BETA])}}}}, {});
    e.upd(1, {rh, ph}, {OutSpec{ph, {{0, C1()}, {1, SC(off[SL_BETA], 0, 1)}}}}, {});
  }
};

struct BlBiCG : Solver {  // Alg. 3
  void *P, *Q, *Rh, *Ph, *Qh;
  int alloc() override {
    P = blk(); Q = blk(); Rh = blk(); Ph = blk(); Qh = blk();
    cols_A = s; cols_AH = s;
    return (P && Q && Rh && Ph && Qh) ? 0 : SRK_ENOMEM;
  }
  int init() override {
    const size_t b = (size_t)n * s * esz();
    if (int r = shadow_into(Rh)) return r;
    cudaMemcpyAsync(P, R, b, cudaMemcpyDeviceToDevice, c->st);
    cudaMemcpyAsync(Ph, Rh, b, cudaMemcpyDeviceToDevice, c->st);
    e.upd(s, {R, Rh}, {}, {RQ{RED_FULL, 0, 1, nullptr, off[SL_M]}});  // M = R̂^H R
    return coef(0);
  }
  void seg(int) override {
    e.spmm(false, P, Q, s, {RQ{RED_FULL, 0, -1, Ph, off[SL_G]}});  // G = P̂^H Q
    e.spmm(true, Ph, Qh, s, {});
    coef(1);
    e.upd(s, {X, P, R, Q, Rh, Qh},
          {OutSpec{X, {{0, C1()}, {1, FU(off[SL_ALPHA])}}},
           OutSpec{R, {{2, C1()}, {3, FU(off[SL_ALPHA], 1)}}},
           OutSpec{Rh, {{4, C1()}, {5, FU(off[SL_AH], 1)}}}},
          {RQ{RED_FULL, O1, O2, nullptr, off[SL_MN]}, RQ{RED_NORM2, O1, -1, nullptr, off[SL_R2]}});
    coef(2);
    e.upd(s, {R, P, Rh, Ph},
          {OutSpec{P, {{0, C1()}, {1, FU(off[SL_BETA])}}}, OutSpec{Ph, {{2, C1()}, {3, FU(off[SL_BH])}}}}, {});
  }
};

struct BlBiCGrQ : Solver {  // Alg. 5
  void *Qr, *Qh, *V, *Vh, *W, *Wh, *Z, *Zh;
  void *Zs = nullptr, *Zhs = nullptr;  // rank continuation (f4): the blocks before the repair
  bool is_rq() const override { return true; }
  int alloc() override {
    Qr = blk(); Qh = blk(); V = blk(); Vh = blk(); W = blk(); Wh = blk(); Z = blk(); Zh = blk();
    if (o.rank_policy) {
      Zs = blk();
      Zhs = blk();
      if (!Zs || !Zhs) return SRK_ENOMEM;
    }
    cols_A = s; cols_AH = s;
    return (Qr && Qh && V && Vh && W && Wh && Z && Zh) ? 0 : SRK_ENOMEM;
  }
  int init() override {
    const size_t b = (size_t)n * s * esz();
    dev_tsqr(*this, R, Qr, false, Zs);  // Q(0) C(0) = R(0)
    if (o.shadow == 0) {  // shadow R̂0 = R0: Q̂(0) = Q(0), Ĉ(0) = C(0)
      cudaMemcpyAsync(Qh, Qr, b, cudaMemcpyDeviceToDevice, c->st);
      cudaMemcpyAsync(ws + off[SL_CH], ws + off[SL_C], s * s * esz(), cudaMemcpyDeviceToDevice, c->st);
    } else {              // Q̂(0) Ĉ(0) = R̂0
      if (int r = shadow_into(Zh)) return r;
      dev_tsqr(*this, Zh, Qh, true);
    }
    cudaMemcpyAsync(V, Qr, b, cudaMemcpyDeviceToDevice, c->st);
    cudaMemcpyAsync(Vh, Qh, b, cudaMemcpyDeviceToDevice, c->st);
    e.upd(s, {Qr, Qh}, {}, {RQ{RED_FULL, 0, 1, nullptr, off[SL_G2]}});  // G2 = Q̂^H Q
    return coef(0);
  }
  void seg(int) override {
    e.spmm(false, V, W, s, {RQ{RED_FULL, 0, -1, Vh, off[SL_G1]}});  // G1 = V̂^H W
    e.spmm(true, Vh, Wh, s, {});
    coef(1);
    e.upd(s, {X, V, Qr, W, Qh, Wh},
          {OutSpec{X, {{0, C1()}, {1, FU(off[SL_AC])}}},
           OutSpec{Z, {{2, C1()}, {3, FU(off[SL_ALPHA], 1)}}},
           OutSpec{Zh, {{4, C1()}, {5, FU(off[SL_AH], 1)}}}},
          {RQ{RED_FULL, O1, O1, nullptr, off[SL_GZ]}, RQ{RED_FULL, O2, O2, nullptr, off[SL_GZH]}});
    coef(2);
    if (Zs) defl_repair(Z, Zs, Zh, Zhs, false);
    e.upd(s, {Z, Zh}, {OutSpec{Z, {{0, FU(off[SL_R1I])}}}, OutSpec{Zh, {{1, FU(off[SL_R1HI])}}}},
          {RQ{RED_FULL, O0, O0, nullptr, off[SL_GZ]}, RQ{RED_FULL, O1, O1, nullptr, off[SL_GZH]}});
    coef(3);
    e.upd(s, {Z, Zh}, {OutSpec{Qr, {{0, FU(off[SL_R2I])}}}, OutSpec{Qh, {{1, FU(off[SL_R2HI])}}}},
          {RQ{RED_FULL, O0, O1, nullptr, off[SL_G2N]}});
    if (Zs) defl_fixup(Qr, Zs, Qh, Zhs, false);
    coef(4);
    e.upd(s, {Qr, V, Qh, Vh},
          {OutSpec{V, {{0, C1()}, {1, FU(off[SL_BETA])}}}, OutSpec{Vh, {{2, C1()}, {3, FU(off[SL_BH])}}}}, {});
  }
  int residual(void* out, int64_t* rows) override {  // C(k): ||R|| = ||C||
    cudaMemcpyAsync(out, ws + off[SL_C], (size_t)s * s * esz(), cudaMemcpyDeviceToDevice, c->st);
    if (rows) *rows = s;
    return cudaStreamSynchronize(c->st) == cudaSuccess ? SRK_OK : SRK_ECUDA;
  }
};

// =============================================================================
// BiCGStab family
// =============================================================================
struct GlBiCGStab : Solver {  // Gl (scalar) and Li (diag)
  bool li = false;
  void *P, *V, *S, *T, *Rt;
  int nseg() const override { return 2; }
  int alloc() override {
    P = blk(); V = blk(); S = blk(); T = blk(); Rt = blk(); tmp2 = blk();
    cols_A = 2 * s; cols_AH = 0;
    return (P && V && S && T && Rt && tmp2) ? 0 : SRK_ENOMEM;
  }
  int rmode() const { return li ? RED_DIAG : RED_TRACE; }
  Coef K(int slot, int neg = 0) const { return li ? DG(off[slot], neg) : SC(off[slot], neg); }
  int init() override {
    const size_t b = (size_t)n * s * esz();
    if (int r = shadow_into(Rt)) return r;  // R̃ (default R0)
    cudaMemcpyAsync(P, R, b, cudaMemcpyDeviceToDevice, c->st);
    e.upd(s, {R, Rt}, {}, {RQ{rmode(), 0, 1, nullptr, off[SL_RHO]}});
    return coef(0);
  }
  // Gl (scalar coefficients): the three updates as flat plans (flat_upd.cu)
  bool flat() const {
    static const bool off_env = getenv("SRK_NO_FLAT_UPDATE") != nullptr;  // A/B switch
    return !li && !off_env && e.qmr_tail_ok(s);
  }
  void seg(int q) override {
    if (q == 0) {
      e.spmm(false, P, V, s, {RQ{rmode(), 0, -1, Rt, off[SL_DEN]}});  // V = A P ; <v, r̃>
      coef(1);
      if (flat()) e.flat(FP_STAB_S, s, {R, V}, {S}, {off[SL_ALPHA]}, {off[SL_S2]});
      else e.upd(s, {R, V}, {OutSpec{S, {{0, C1()}, {1, K(SL_ALPHA, 1)}}}}, {RQ{RED_NORM2, O0, -1, nullptr, off[SL_S2]}});
      coef(2);  // half-step test on ||S||_F
    } else {
      e.spmm(false, S, T, s,
             {RQ{rmode(), 0, -1, S, off[SL_ST]}, RQ{li ? RED_COLNORM2 : RED_NORM2, 0, -1, nullptr, off[SL_TT]}});
      coef(3);
      if (flat()) {
        e.flat(FP_STAB_XR, s, {X, P, S, T, Rt}, {X, R}, {off[SL_ALPHA], off[SL_OMEGA], off[SL_OMEGA]},
               {off[SL_RHON], off[SL_R2]});
        coef(4);
        e.flat(FP_STAB_P, s, {R, P, V}, {P}, {off[SL_BETA], off[SL_BW]}, {});
        return;
      }
      e.upd(s, {X, P, S, T, Rt},
            {OutSpec{X, {{0, C1()}, {1, K(SL_ALPHA)}, {2, K(SL_OMEGA)}}},
             OutSpec{R, {{2, C1()}, {3, K(SL_OMEGA, 1)}}}},
            {RQ{rmode(), O1, 4, nullptr, off[SL_RHON]}, RQ{RED_NORM2, O1, -1, nullptr, off[SL_R2]}});
      coef(4);
      e.upd(s, {R, P, V}, {OutSpec{P, {{0, C1()}, {1, K(SL_BETA)}, {2, K(SL_BW, 1)}}}}, {});
    }
  }
  void half_x(void* Xh) override {
    const int* sv = e.done;
    e.done = nullptr;
    e.upd(s, {X, P}, {OutSpec{Xh, {{0, C1()}, {1, K(SL_ALPHA)}}}}, {});
    e.done = sv;
  }
};

struct BlBiCGStab : Solver {  // [ELg03], SURVEY App. A.4
  void *P, *U, *S, *T, *Rt;
  int nseg() const override { return 2; }
  int alloc() override {
    P = blk(); U = blk(); S = blk(); T = blk(); Rt = blk(); tmp2 = blk();
    cols_A = 2 * s; cols_AH = 0;
    return (P && U && S && T && Rt && tmp2) ? 0 : SRK_ENOMEM;
  }
  int init() override {
    const size_t b = (size_t)n * s * esz();
    if (int r = shadow_into(Rt)) return r;
    cudaMemcpyAsync(P, R, b, cudaMemcpyDeviceToDevice, c->st);
    e.upd(s, {R, Rt}, {}, {RQ{RED_FULL, 0, 1, nullptr, off[SL_M]}});  // R̃^H R
    return coef(0);
  }
  void seg(int q) override {
    if (q == 0) {
      e.spmm(false, P, U, s, {RQ{RED_FULL, 0, -1, Rt, off[SL_G]}});  // G = R̃^H U
      coef(1);
      e.upd(s, {R, U}, {OutSpec{S, {{0, C1()}, {1, FU(off[SL_ALPHA], 1)}}}}, {RQ{RED_NORM2, O0, -1, nullptr, off[SL_S2]}});
      coef(2);
    } else {
      e.spmm(false, S, T, s, {RQ{RED_TRACE, 0, -1, S, off[SL_ST]}, RQ{RED_NORM2, 0, -1, nullptr, off[SL_TT]}});
      coef(3);
      e.upd(s, {X, P, S, T, Rt},
            {OutSpec{X, {{0, C1()}, {1, FU(off[SL_ALPHA])}, {2, SC(off[SL_OMEGA])}}},
             OutSpec{R, {{2, C1()}, {3, SC(off[SL_OMEGA], 1)}}}},
            {RQ{RED_FULL, 3, 4, nullptr, off[SL_MN]}, RQ{RED_FULL, O1, 4, nullptr, off[SL_M]},
             RQ{RED_NORM2, O1, -1, nullptr, off[SL_R2]}});
      coef(4);
      e.upd(s, {R, P, U}, {OutSpec{P, {{0, C1()}, {1, FU(off[SL_BETA])}, {2, FU(off[SL_BW], 1)}}}}, {});
    }
  }
  void half_x(void* Xh) override {
    const int* sv = e.done;
    e.done = nullptr;
    e.upd(s, {X, P}, {OutSpec{Xh, {{0, C1()}, {1, FU(off[SL_ALPHA])}}}}, {});
    e.done = sv;
  }
};

struct BlBiCGStabrQ : Solver {
  void *Qr, *Q0, *V, *W, *Z, *Y;
  void* Zs = nullptr;  // rank continuation (f4)
  bool is_rq() const override { return true; }
  int nseg() const override { return 2; }
  // small operators (latency-bound, config 1): whole iterations in one single-CTA kernel
  bool small() const {
    static const bool off_env = getenv("SRK_NO_SMALL_KERNEL") != nullptr;  // A/B switch
    return !off_env && A && !A->bsr && !A->prec && A->ghost_rows() == 0 && n <= SMALL_N_MAX && s <= SMALL_BL_SMAX &&
           !o.rank_policy && !(c->comm && c->comm->nranks > 1);
  }
  bool ends_iter() const override { return small(); }
  int seg_multi(int k) override {
    if (!small() || k < 1 || e.err) return 0;
    SmallBlStabArgs g{};
    g.rp = A->rp;
    g.ci = A->ci;
    g.val = A->val;
    g.X = X; g.Qr = Qr; g.Q0 = Q0; g.V = V; g.W = W; g.Z = Z; g.Y = Y;
    g.n = n;
    g.iters = k;
    g.ws_doubles = (long long)slot_doubles(s) * NSLOT;
    g.ca.method = method;
    g.ca.s = s;
    g.ca.tol = o.tol;
    g.ca.eps_brk = eps_brk();
    g.ca.eps_chol = eps_chol();
    g.ca.ws = ws;
    g.ca.ctl = ctl;
    g.ca.hist = hist;
    g.ca.hist_cap = hist_cap;
    for (int i = 0; i < NSLOT; ++i) g.ca.off[i] = off[i];
    e.nlaunch++;
    prof.begin(PT_OTHER, c->st);
    e.err = launch_bl_bicgstab_rq_small(cplx, g, c->st);
    prof.end(c->st);
    return k;
  }
  int alloc() override {
    Qr = blk(); Q0 = blk(); V = blk(); W = blk(); Z = blk(); Y = blk(); tmp2 = blk();
    if (o.rank_policy && !(Zs = blk())) return SRK_ENOMEM;
    cols_A = 2 * s; cols_AH = 0;
    return (Qr && Q0 && V && W && Z && Y && tmp2) ? 0 : SRK_ENOMEM;
  }
  int init() override {
    const size_t b = (size_t)n * s * esz();
    dev_tsqr(*this, R, Qr, false, Zs);
    if (o.shadow == 0) {
      cudaMemcpyAsync(Q0, Qr, b, cudaMemcpyDeviceToDevice, c->st);  // Q̂0 = Qr when R̃ = R0
    } else {  // Q̂0 = orthonormal factor of R̃ (its R factor cancels, App. A.5)
      if (int r = shadow_into(Z)) return r;
      dev_tsqr(*this, Z, Q0, true);
    }
    cudaMemcpyAsync(V, Qr, b, cudaMemcpyDeviceToDevice, c->st);
    e.upd(s, {Qr, Q0}, {}, {RQ{RED_FULL, 0, 1, nullptr, off[SL_GQ]}});
    return coef(0);
  }
  void seg(int q) override {
    if (q == 0) {
      e.spmm(false, V, W, s, {RQ{RED_FULL, 0, -1, Q0, off[SL_G]}});  // G = Q̂0^H W
      coef(1);
      e.upd(s, {Qr, W}, {OutSpec{Z, {{0, C1()}, {1, FU(off[SL_ALPHA], 1)}}}}, {RQ{RED_FULL, O0, O0, nullptr, off[SL_ZZ]}});
      coef(2);
    } else {
      e.spmm(false, Z, Y, s, {RQ{RED_FULL, 0, -1, Z, off[SL_YZ]}, RQ{RED_FULL, 0, -1, Y, off[SL_YY]}});
      coef(3);
      e.upd(s, {X, V, Z, Y},
            {OutSpec{X, {{0, C1()}, {1, FU(off[SL_AC])}, {2, FU(off[SL_WC])}}},
             OutSpec{Z, {{2, C1()}, {3, SC(off[SL_OMEGA], 1)}}}},
            {RQ{RED_FULL, O1, O1, nullptr, off[SL_GZ]}});
      coef(4);
      if (Zs) defl_repair(Z, Zs, nullptr, nullptr, false);
      e.upd(s, {Z}, {OutSpec{Z, {{0, FU(off[SL_R1I])}}}}, {RQ{RED_FULL, O0, O0, nullptr, off[SL_GZ]}});
      coef(5);
      e.upd(s, {Z, Q0}, {OutSpec{Qr, {{0, FU(off[SL_R2I])}}}}, {RQ{RED_FULL, O0, 1, nullptr, off[SL_GQN]}});
      if (Zs) defl_fixup(Qr, Zs, nullptr, nullptr, false);
      coef(6);
      e.upd(s, {Qr, V, W}, {OutSpec{V, {{0, C1()}, {1, FU(off[SL_BETA])}, {2, FU(off[SL_BW], 1)}}}}, {});
    }
  }
  void half_x(void* Xh) override {
    const int* sv = e.done;
    e.done = nullptr;
    e.upd(s, {X, V}, {OutSpec{Xh, {{0, C1()}, {1, FU(off[SL_AC])}}}}, {});
    e.done = sv;
  }
  int residual(void* out, int64_t* rows) override {
    cudaMemcpyAsync(out, ws + off[SL_C], (size_t)s * s * esz(), cudaMemcpyDeviceToDevice, c->st);
    if (rows) *rows = s;
    return cudaStreamSynchronize(c->st) == cudaSuccess ? SRK_OK : SRK_ECUDA;
  }
};

// =============================================================================
// QMR family
// =============================================================================
// Li / Gl / eGl-QMR. The normalised Lanczos blocks V = Ṽ/ρ and
// W = W̃/ξ are never materialised: 1/ρ and 1/ξ are folded into the coefficients
// of the kernels that read Ṽ and W̃, and δ = <V, W> = <Ṽ, W̃>/(ρ ξ) is fused into
// the kernel that produces Ṽ — an iteration moves 18 n x s blocks
// instead of 20, and 17 with the fused tail (Gl / eGl: the last update also forms the
// next P, qmr_tail.cu). Same recurrences as oracle/solvers.py::_qmr_li_gl.
struct QMR : Solver {  // mode 0 Li, 1 Gl, 2 eGl
  int mode = 1;
  void *Vt, *P, *Pt, *D, *S, *Wt, *Qv, *AHQ;
  int alloc() override {
    Vt = blk(); P = blk(); Pt = blk(); D = blk(); S = blk();
    if (mode == 2) { Wt = vecn(); Qv = vecn(); AHQ = vecn(); }
    else { Wt = blk(); Qv = blk(); AHQ = blk(); }
    cols_A = s; cols_AH = (mode == 2) ? 1 : s;
    return (Vt && P && Pt && D && S && Wt && Qv && AHQ) ? 0 : SRK_ENOMEM;
  }
  int ws_() const { return mode == 2 ? 1 : s; }  // width of the left Lanczos block
  int nrm() const { return mode == 0 ? RED_COLNORM2 : RED_NORM2; }
  int dmode() const { return mode == 0 ? RED_DIAG : (mode == 1 ? RED_TRACE : RED_SUMVEC); }
  Coef K(int slot, int neg = 0, int cj = 0) const { return mode == 0 ? DG(off[slot], neg, cj) : SC(off[slot], neg, cj); }
  // Ṽ-producing reduction set: ||Ṽ||^2 and <Ṽ, W̃> (W̃ an input block, or the vector for eGl)
  std::vector<RQ> vt_reds(int vt_src, int wt_src) const {
    if (mode == 2) return {RQ{nrm(), vt_src, -1, nullptr, off[SL_RHON2]}, RQ{RED_SUMVEC, vt_src, -1, Wt, off[SL_K1]}};
    return {RQ{nrm(), vt_src, -1, nullptr, off[SL_RHON2]}, RQ{dmode(), vt_src, wt_src, nullptr, off[SL_K1]}};
  }
  int init() override {
    const size_t b = (size_t)n * s * esz();
    cudaMemcpyAsync(Vt, R, b, cudaMemcpyDeviceToDevice, c->st);
    if (int r = (mode == 2) ? shadow_vec_into(Wt) : shadow_into(Wt)) return r;  // w̃0 = mean / W̃0 = R0 by default
    e.upd(ws_(), {Wt}, {}, {RQ{nrm(), 0, -1, nullptr, off[SL_XI2]}});
    if (mode == 2) e.upd(s, {Vt}, {}, vt_reds(0, -1));
    else e.upd(s, {Vt, Wt}, {}, vt_reds(0, 1));
    cudaMemsetAsync(P, 0, b, c->st);
    cudaMemsetAsync(D, 0, b, c->st);
    cudaMemsetAsync(S, 0, b, c->st);
    cudaMemsetAsync(Qv, 0, (size_t)n * ws_() * esz(), c->st);
    return coef(0);
  }
  // small operators (latency-bound), eGl only: the whole iteration as one single-CTA kernel
  bool small() const {
    static const bool off_env = getenv("SRK_NO_SMALL_KERNEL") != nullptr;  // A/B switch
    return mode == 2 && !off_env && A && !A->bsr && !A->prec && A->ghost_rows() == 0 && A->has_adj && n <= SMALL_N_MAX &&
           !(c->comm && c->comm->nranks > 1);
  }
  // Gl / eGl-QMR (scalar coefficients): the iteration's last update also forms the next P
  bool fused_tail() const {
    static const bool off_env = getenv("SRK_NO_QMR_FUSE") != nullptr;  // A/B switch
    return mode != 0 && !off_env && e.qmr_tail_ok(s);
  }
  bool flat_vw() const {
    static const bool off_env = getenv("SRK_NO_FLAT_UPDATE") != nullptr;  // A/B switch
    return !off_env && e.qmr_tail_ok(s);
  }
  bool fused_vec() const {
    static const bool off_env = getenv("SRK_NO_QMR_VEC_FUSE") != nullptr;  // A/B switch
    return mode == 2 && !off_env && e.qmr_vec_ok(s);
  }
  bool ends_iter() const override { return small(); }
  int seg_multi(int k) override {
    if (!small() || k < 1 || e.err) return 0;
    launch_small(k);
    return k;
  }
  void launch_small(int iters) {
    SmallQMRArgs g{};
    g.rp = A->rp;
    g.ci = A->ci;
    g.val = A->val;
    g.rpH = A->rpH;
    g.ciH = A->ciH;
    g.valH = A->valH;
    g.X = X; g.R = R; g.Vt = Vt; g.P = P; g.Pt = Pt; g.D = D; g.S = S; g.Wt = Wt; g.Qv = Qv; g.AHQ = AHQ;
    g.n = n;
    g.iters = iters;
    g.ca.method = method;
    g.ca.s = s;
    g.ca.tol = o.tol;
    g.ca.eps_brk = eps_brk();
    g.ca.eps_chol = eps_chol();
    g.ca.ws = ws;
    g.ca.ctl = ctl;
    g.ca.hist = hist;
    g.ca.hist_cap = hist_cap;
    for (int i = 0; i < NSLOT; ++i) g.ca.off[i] = off[i];
    e.nlaunch++;
    prof.begin(PT_OTHER, c->st);
    e.err = launch_egl_qmr_small(cplx, g, c->st);
    prof.end(c->st);
  }
  void seg(int) override {
    if (small()) {
      if (!e.err) launch_small(1);
      return;
    }
    coef(1);                   // 1/rho, 1/xi
    coef(2, host_iter == 0);   // delta = <Ṽ, W̃>/(rho xi); c1 = xi delta/eps, c2 = conj(rho delta/eps)
    // P = V - c1 P = Ṽ/rho - c1 P ;  Q = W - c2 Q = W̃/xi - c2 Q
    // (fused tail: after the first iteration P was already formed by the previous iteration's last kernel)
    const bool fuse = fused_tail();
    const bool vfuse = fuse && fused_vec();  // eGl: w̃ and q ride in the block kernels as well
    const bool p_done = fuse && host_iter > 0;
    if (mode == 2) {
      if (!p_done) e.upd(s, {Vt, P}, {OutSpec{P, {{0, SC(off[SL_INVRHO])}, {1, SC(off[SL_C1], 1)}}}}, {});
      if (!(vfuse && p_done)) e.upd(1, {Wt, Qv}, {OutSpec{Qv, {{0, SC(off[SL_INVXI])}, {1, SC(off[SL_C2], 1)}}}}, {});
    } else if (p_done) {
      e.upd(s, {Wt, Qv}, {OutSpec{Qv, {{0, K(SL_INVXI)}, {1, K(SL_C2, 1)}}}}, {});
    } else {
      e.upd(s, {Vt, P, Wt, Qv},
            {OutSpec{P, {{0, K(SL_INVRHO)}, {1, K(SL_C1, 1)}}}, OutSpec{Qv, {{2, K(SL_INVXI)}, {3, K(SL_C2, 1)}}}}, {});
    }
    e.spmm(false, P, Pt, s, {RQ{dmode(), 0, -1, Qv, off[SL_EPS]}});  // P~ = A P ; eps = <P~, Q>
    e.spmm(true, Qv, AHQ, ws_(), {});                                // A^H Q
    coef(3);  // beta = eps/delta ; BR = beta/rho ; BX = conj(beta)/xi
    if (vfuse) {
      // one kernel: Ṽ = P~ - (beta/rho) Ṽ with ||Ṽ||^2, <Ṽ, W̃> and ||W̃||^2 for the new
      // W̃ = A^H Q - (conj(beta)/xi) W̃, formed per row in registers (stored by the tail below)
      e.qmr_vt(s, Pt, Vt, AHQ, Wt, off[SL_BR], off[SL_BX], off[SL_RHON2], off[SL_K1], off[SL_XI2]);
    } else if (mode == 1 && flat_vw()) {
      // Gl: both Lanczos blocks and their three reductions as one flat plan (flat_upd.cu)
      e.flat(FP_QMR_VW, s, {Pt, Vt, AHQ, Wt}, {Vt, Wt}, {off[SL_BR], off[SL_BX]}, {off[SL_RHON2], off[SL_K1], off[SL_XI2]});
    } else {
      // W̃ = A^H Q - conj(beta) W = A^H Q - (conj(beta)/xi) W̃   (first: Ṽ's kernel reads the new W̃)
      e.upd(ws_(), {AHQ, Wt}, {OutSpec{Wt, {{0, C1()}, {1, K(SL_BX, 1)}}}}, {RQ{nrm(), O0, -1, nullptr, off[SL_XI2]}});
      // Ṽ = P~ - beta V = P~ - (beta/rho) Ṽ, with ||Ṽ||^2 and the next <Ṽ, W̃>
      if (mode == 2) e.upd(s, {Pt, Vt}, {OutSpec{Vt, {{0, C1()}, {1, K(SL_BR, 1)}}}}, vt_reds(O0, -1));
      else e.upd(s, {Pt, Vt, Wt}, {OutSpec{Vt, {{0, C1()}, {1, K(SL_BR, 1)}}}}, vt_reds(O0, 2));
    }
    coef(4);  // theta, gamma, eta, f (and the next iteration's 1/rho, c1, 1/xi, c2)
    if (fuse) {
      // (D, S, X, R) of this iteration and P = Ṽ/rho' - c1' P of the next in one pass (qmr_tail.cu):
      // 12 block passes instead of 10 + 3; eGl: also W̃ (stored here) and q = W̃/xi' - c2' q
      const QmrVec v{Wt, Qv, AHQ, off[SL_BX], off[SL_INVXI_N], off[SL_C2_N]};
      e.qmr_tail(s, P, D, Pt, S, X, R, Vt, off[SL_ETA], off[SL_F], off[SL_INVRHO_N], off[SL_C1_N], off[SL_R2],
                 vfuse ? &v : nullptr);
      coef(5);
      return;
    }
    e.upd(s, {P, D, Pt, S, X, R},
          {OutSpec{D, {{0, K(SL_ETA)}, {1, K(SL_F)}}},
           OutSpec{S, {{2, K(SL_ETA)}, {3, K(SL_F)}}},
           OutSpec{X, {{4, C1()}, {O0, C1()}}},
           OutSpec{R, {{5, C1()}, {O1, NEG1()}}}},
          {RQ{RED_NORM2, O3, -1, nullptr, off[SL_R2]}});
    coef(5);
  }
};

struct BlQMR : Solver {
  void *V, *Wb, *P, *Qb, *AP, *AHQ, *D, *F, *Zv, *Zw;
  int alloc() override {
    V = blk(); Wb = blk(); P = blk(); Qb = blk(); AP = blk(); AHQ = blk(); D = blk(); F = blk(); Zv = blk(); Zw = blk();
    cols_A = s; cols_AH = s;
    return (V && Wb && P && Qb && AP && AHQ && D && F && Zv && Zw) ? 0 : SRK_ENOMEM;
  }
  int init() override {
    const size_t b = (size_t)n * s * esz();
    dev_tsqr(*this, R, V, false);  // V rho = R0
    cudaMemcpyAsync(ws + off[SL_RHOB], ws + off[SL_C], (size_t)s * s * esz(), cudaMemcpyDeviceToDevice, c->st);
    if (o.shadow == 0) {
      cudaMemcpyAsync(Wb, V, b, cudaMemcpyDeviceToDevice, c->st);  // W xi = R̂0 = R0
      cudaMemcpyAsync(ws + off[SL_XIB], ws + off[SL_C], (size_t)s * s * esz(), cudaMemcpyDeviceToDevice, c->st);
    } else {  // W xi = R̂0 (thin QR)
      if (int r = shadow_into(Wb)) return r;
      dev_tsqr(*this, Wb, Wb, true);
      cudaMemcpyAsync(ws + off[SL_XIB], ws + off[SL_CH], (size_t)s * s * esz(), cudaMemcpyDeviceToDevice, c->st);
    }
    cudaMemsetAsync(P, 0, b, c->st);
    cudaMemsetAsync(Qb, 0, b, c->st);
    cudaMemsetAsync(D, 0, b, c->st);
    cudaMemsetAsync(F, 0, b, c->st);
    return coef(0);
  }
  void seg(int) override {
    e.upd(s, {V, Wb}, {}, {RQ{RED_FULL, 0, 1, nullptr, off[SL_DELTA]}});  // delta = W^H V
    coef(1, host_iter == 0);
    e.upd(s, {V, P, Wb, Qb},
          {OutSpec{P, {{0, C1()}, {1, FU(off[SL_C1], 1)}}}, OutSpec{Qb, {{2, C1()}, {3, FU(off[SL_C2], 1)}}}}, {});
    e.spmm(false, P, AP, s, {RQ{RED_FULL, 0, -1, Qb, off[SL_EPS]}});  // eps = Q^H A P
    e.spmm(true, Qb, AHQ, s, {});
    coef(2);
    e.upd(s, {AP, V, AHQ, Wb},
          {OutSpec{Zv, {{0, C1()}, {1, FU(off[SL_BETA], 1)}}}, OutSpec{Zw, {{2, C1()}, {3, FU(off[SL_GHAT], 1)}}}},
          {RQ{RED_FULL, O0, O0, nullptr, off[SL_GZ]}, RQ{RED_FULL, O1, O1, nullptr, off[SL_GZH]}});
    coef(3);
    e.upd(s, {Zv, Zw}, {OutSpec{Zv, {{0, FU(off[SL_R1I])}}}, OutSpec{Zw, {{1, FU(off[SL_R1HI])}}}},
          {RQ{RED_FULL, O0, O0, nullptr, off[SL_GZ]}, RQ{RED_FULL, O1, O1, nullptr, off[SL_GZH]}});
    coef(4, host_iter == 0);
    e.upd(s, {Zv, Zw}, {OutSpec{V, {{0, FU(off[SL_R2I])}}}, OutSpec{Wb, {{1, FU(off[SL_R2HI])}}}}, {});
    e.upd(s, {P, D, X},
          {OutSpec{D, {{0, FU(off[SL_RIII])}, {1, FU(off[SL_TR], 1)}}}, OutSpec{X, {{2, C1()}, {O0, FU(off[SL_TAU])}}}}, {});
    e.upd(s, {AP, F, R},
          {OutSpec{F, {{0, FU(off[SL_RIII])}, {1, FU(off[SL_TR], 1)}}}, OutSpec{R, {{2, C1()}, {O0, FU(off[SL_TAU], 1)}}}},
          {RQ{RED_NORM2, O1, -1, nullptr, off[SL_R2]}});
    coef(5);
  }
};

// =============================================================================
// QR of the search directions: the
// [O'Leary] stabilisation the paper compares with; oracle bl_bicg_sq / bl_bicgstab_sq
// (reading R9). P (and P̂) are kept orthonormal by a CholQR2 per iteration.
// =============================================================================
struct BlBiCGsQ : Solver {
  void *P, *Q, *Rh, *Ph, *Qh;
  int alloc() override {
    P = blk(); Q = blk(); Rh = blk(); Ph = blk(); Qh = blk();
    cols_A = s; cols_AH = s;
    return (P && Q && Rh && Ph && Qh) ? 0 : SRK_ENOMEM;
  }
  int init() override {
    const size_t b = (size_t)n * s * esz();
    if (int r = shadow_into(Rh)) return r;  // R̂0 (default R0)
    dev_tsqr(*this, R, P, false);           // P = orthonormal basis of R0
    if (o.shadow == 0) cudaMemcpyAsync(Ph, P, b, cudaMemcpyDeviceToDevice, c->st);
    else dev_tsqr(*this, Rh, Ph, true);
    e.upd(s, {R, Ph, Rh, P}, {}, {RQ{RED_FULL, 0, 1, nullptr, off[SL_M]}, RQ{RED_FULL, 2, 3, nullptr, off[SL_MH]}});
    return coef(0);
  }
  void seg(int) override {
    e.spmm(false, P, Q, s, {RQ{RED_FULL, 0, -1, Ph, off[SL_G]}});  // G = P̂^H A P
    e.spmm(true, Ph, Qh, s, {});
    coef(1);  // alpha = G^-1 P̂^H R, alpha_hat = G^-H P^H R̂
    e.upd(s, {X, P, R, Q, Rh, Qh},
          {OutSpec{X, {{0, C1()}, {1, FU(off[SL_ALPHA])}}},
           OutSpec{R, {{2, C1()}, {3, FU(off[SL_ALPHA], 1)}}},
           OutSpec{Rh, {{4, C1()}, {5, FU(off[SL_AH], 1)}}}},
          {RQ{RED_NORM2, O1, -1, nullptr, off[SL_R2]}, RQ{RED_FULL, O1, 5, nullptr, off[SL_MN]},
           RQ{RED_FULL, O2, 3, nullptr, off[SL_MNH]}});
    coef(2);  // beta = -G^-1 Q̂^H R+, beta_hat = -G^-H Q^H R̂+
    e.upd(s, {R, P, Rh, Ph}, {OutSpec{P, {{0, C1()}, {1, FU(off[SL_BETA])}}}, OutSpec{Ph, {{2, C1()}, {3, FU(off[SL_BH])}}}},
          {RQ{RED_FULL, O0, O0, nullptr, off[SL_GZ]}, RQ{RED_FULL, O1, O1, nullptr, off[SL_GZH]}});
    coef(3);  // CholQR2 pass 1 (rank test)
    e.upd(s, {P, Ph}, {OutSpec{P, {{0, FU(off[SL_R1I])}}}, OutSpec{Ph, {{1, FU(off[SL_R1HI])}}}},
          {RQ{RED_FULL, O0, O0, nullptr, off[SL_GZ]}, RQ{RED_FULL, O1, O1, nullptr, off[SL_GZH]}});
    coef(4);  // pass 2; the next alpha's Grams with the new orthonormal directions
    e.upd(s, {P, Ph, R, Rh}, {OutSpec{P, {{0, FU(off[SL_R2I])}}}, OutSpec{Ph, {{1, FU(off[SL_R2HI])}}}},
          {RQ{RED_FULL, 2, O1, nullptr, off[SL_M]}, RQ{RED_FULL, 3, O0, nullptr, off[SL_MH]}});
  }
};

struct BlBiCGStabsQ : Solver {
  void *P, *U, *S, *T, *Rt;
  int nseg() const override { return 2; }
  int alloc() override {
    P = blk(); U = blk(); S = blk(); T = blk(); Rt = blk(); tmp2 = blk();
    cols_A = 2 * s; cols_AH = 0;
    return (P && U && S && T && Rt && tmp2) ? 0 : SRK_ENOMEM;
  }
  int init() override {
    const size_t b = (size_t)n * s * esz();
    if (int r = shadow_into(Rt)) return r;
    dev_tsqr(*this, R, P, false);  // P = orthonormal basis of R0
    e.upd(s, {R, Rt}, {}, {RQ{RED_FULL, 0, 1, nullptr, off[SL_M]}});  // R̃^H R
    return coef(0);
  }
  void seg(int q) override {
    if (q == 0) {
      e.spmm(false, P, U, s, {RQ{RED_FULL, 0, -1, Rt, off[SL_G]}});  // G = R̃^H U
      coef(1);
      e.upd(s, {R, U}, {OutSpec{S, {{0, C1()}, {1, FU(off[SL_ALPHA], 1)}}}}, {RQ{RED_NORM2, O0, -1, nullptr, off[SL_S2]}});
      coef(2);
    } else {
      e.spmm(false, S, T, s, {RQ{RED_TRACE, 0, -1, S, off[SL_ST]}, RQ{RED_NORM2, 0, -1, nullptr, off[SL_TT]}});
      coef(3);
      e.upd(s, {X, P, S, T, Rt},
            {OutSpec{X, {{0, C1()}, {1, FU(off[SL_ALPHA])}, {2, SC(off[SL_OMEGA])}}},
             OutSpec{R, {{2, C1()}, {3, SC(off[SL_OMEGA], 1)}}}},
            {RQ{RED_FULL, 3, 4, nullptr, off[SL_MN]}, RQ{RED_FULL, O1, 4, nullptr, off[SL_M]},
             RQ{RED_NORM2, O1, -1, nullptr, off[SL_R2]}});
      coef(4);
      e.upd(s, {R, P, U}, {OutSpec{P, {{0, C1()}, {1, FU(off[SL_BETA])}, {2, FU(off[SL_BW], 1)}}}},
            {RQ{RED_FULL, O0, O0, nullptr, off[SL_GZ]}});
      coef(5);  // CholQR2 of the new search directions
      e.upd(s, {P}, {OutSpec{P, {{0, FU(off[SL_R1I])}}}}, {RQ{RED_FULL, O0, O0, nullptr, off[SL_GZ]}});
      coef(6);
      e.upd(s, {P}, {OutSpec{P, {{0, FU(off[SL_R2I])}}}}, {});
    }
  }
  void half_x(void* Xh) override {
    const int* sv = e.done;
    e.done = nullptr;
    e.upd(s, {X, P}, {OutSpec{Xh, {{0, C1()}, {1, FU(off[SL_ALPHA])}}}}, {});
    e.done = sv;
  }
};

Solver* make_solver(int m) {
  switch (m) {
    case M_LI_BICG: { auto* p = new GlBiCG(); p->li = true; return p; }
    case M_GL_BICG: return new GlBiCG();
    case M_EGL_BICG: return new EglBiCG();
    case M_BL_BICG: return new BlBiCG();
    case M_BL_BICG_RQ: return new BlBiCGrQ();
    case M_LI_QMR: { auto* p = new QMR(); p->mode = 0; return p; }
    case M_GL_QMR: { auto* p = new QMR(); p->mode = 1; return p; }
    case M_EGL_QMR: { auto* p = new QMR(); p->mode = 2; return p; }
    case M_BL_QMR: return new BlQMR();
    case M_LI_BICGSTAB: { auto* p = new GlBiCGStab(); p->li = true; return p; }
    case M_GL_BICGSTAB: return new GlBiCGStab();
    case M_BL_BICGSTAB: return new BlBiCGStab();
    case M_BL_BICGSTAB_RQ: return new BlBiCGStabrQ();
    case M_BL_BICG_SQ: return new BlBiCGsQ();
    case M_BL_BICGSTAB_SQ: return new BlBiCGStabsQ();
    default: return nullptr;
  }
}

}  // namespace srk
