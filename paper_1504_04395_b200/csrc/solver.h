// solver.h — host drivers of the 13 methods.
#pragma once
#include <vector>

#include "../../include/srk.h"
#include "coef.cuh"
#include "engine.h"

namespace srk {

int launch_coef(bool cplx, const CoefArgs& a, size_t smem, cudaStream_t st);
int launch_end_iter(int* ctl, cudaStream_t st);

struct Solver {
  Ctx* c = nullptr;
  const Mat* A = nullptr;
  int s = 0, method = 0;
  bool cplx = false;
  long long n = 0;
  srk_opts o{};
  Eng e;
  Prof prof;
  double* ws = nullptr;
  double* wstage = nullptr;  // multi-rank: staging of the per-rank sums (engine.cu finish_reds)
  int* ctl = nullptr;
  int* ctl_host = nullptr;  // pinned mirror
  double* hist = nullptr;
  int hist_cap = 0;
  int off[NSLOT];
  std::vector<void*> owned;
  void* B = nullptr;  // internal copy of the right-hand sides
  void* X = nullptr;  // iterate
  void* R = nullptr;  // residual block
  void* tmp = nullptr;
  void* tmp2 = nullptr;
  int host_iter = 0;
  int state = 0;  // 0 running, 1 converged, 2 breakdown, 3 maxit
  int half = 0;
  int brk_kind = 0, brk_iter = -1, frozen = 0;
  long long launches = 0;
  double seconds = 0.0;
  double final_true = -1.0, final_rec = -1.0;
  int cols_A = 0, cols_AH = 0;  // per iteration (Prop. 1 counters)
  long long matA = 0, matAH = 0;
  bool started = false;
  // CUDA graph of `graph_iters` iterations (replayed between host polls)
  cudaStream_t cap_st = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int graph_iters = 0;
  long long graph_launches = 0;
  const double* graph_partials = nullptr;
  int capture(int iters);

  virtual ~Solver();
  int setup();                 // allocate common state
  void* blk();                 // allocate an n x s block
  void* vecn();                // allocate an n-vector
  int coef(int phase, int k1 = 0);
  int shadow_into(void* dst);      // n x s shadow block per o.shadow
  int shadow_vec_into(void* dst);  // economic shadow vector
  // rank-deficiency continuation of the rQ thin QRs (f4): armed by pass 1, else no-ops
  void defl_repair(void* Z, void* Zs, void* Zh, void* Zhs, bool init);
  void defl_fixup(const void* Q, const void* Zs, const void* Qh, const void* Zhs, bool init);
  size_t esz() const { return cplx ? 16 : 8; }
  double eps_brk() const { return o.eps_brk > 0 ? o.eps_brk : 1e-14; }    // reading G12
  double eps_chol() const { return o.eps_defl > 0 ? o.eps_defl : 1e-14; }  // reading R5
  int start(const void* Bd, const void* X0d);
  int iterate(int k);
  double true_rel(const void* Xc);  // sync
  int read_ctl();

  virtual int alloc() = 0;
  virtual int init() = 0;          // R holds R0, ws[SL_R0N2] = ||R0||^2 after the common start
  virtual void seg(int idx) = 0;   // enqueue segment idx of one iteration
  virtual int nseg() const { return 1; }
  virtual void half_x(void* Xh) { (void)Xh; }
  virtual bool is_rq() const { return false; }
  virtual bool ends_iter() const { return false; }  // seg() also ends the iteration (fused kernel)
  virtual int seg_multi(int k) { (void)k; return 0; }  // enqueue up to k whole iterations as one launch
  virtual int residual(void* out, int64_t* rows);
};

Solver* make_solver(int method);

}  // namespace srk
