// engine.h — host-side engine: context, prepared operator, kernel-call helpers.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "comm.h"
#include "kernels.cuh"

namespace srk {

int cap_for(int s);
int rows_per_cta(int cap, bool cplx);
bool full_supported(bool cplx, int cap);
bool full_red_supported(bool cplx, int cap);
int padded_width(int cap, bool cplx);
int launch_spmm(bool cplx, int cap, bool full, const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st);
int launch_upd(bool cplx, int cap, bool full, const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st);
int launch_fin(const FinArgs& a, cudaStream_t st);
int launch_qmr_tail(bool cplx, const QmrTailArgs& a, int grid, cudaStream_t st);  // grid < 0: resident CTAs per SM
int launch_qmr_vt(bool cplx, const QmrVtArgs& a, int grid, cudaStream_t st);
FlatPlanInfo flat_plan_info(int plan);
int launch_egl_flat(int which, bool cplx, const EglFlatArgs& a, int grid, cudaStream_t st);  // grid < 0: resident CTAs per SM
int launch_flat(int plan, bool cplx, const FlatArgs& a, int grid, cudaStream_t st);  // grid < 0: resident CTAs per SM
int launch_gram_mma(const GramArgs& g, int grid, cudaStream_t st);
int launch_bsr(const BsrArgs& a, int s, int grid, cudaStream_t st);  // grid < 0: resident WARPS per SM
int bsr_warps_per_cta();
// block updates with s x s coefficients on the FP64 tensor cores (blk_mma.cu)
int upd_mma_width(int w);
size_t upd_mma_smem(int w, int nterm);
int launch_upd_mma(const UpdArgs& a, bool cplx, int nterm, int grid, cudaStream_t st);
bool bsr_supported(int bs, bool cplx, int s);

int gram_mma_chunks(long long n);
int launch_row_mean(bool cplx, const void* X, void* out, long long n, int s, const int* done, cudaStream_t st);
int launch_csr_transpose(bool cplx, long long n, long long nnz, const int* rp, const int* ci, const void* val,
                         int* rpT, int* ciT, void* valT, int* work, cudaStream_t st);
int launch_csr_check(long long n, long long ncols, long long nnz, const int* rp, const int* ci, int sorted, int* bad,
                     cudaStream_t st);
int launch_gather_rows(const double* src, double* dst, const int* idx, long long nrows, int doubles_per_row,
                       const int* done, cudaStream_t st);

struct Comm;  // multi-GPU plumbing (comm.cpp)

struct Ctx {
  int dev = 0;
  cudaStream_t st = nullptr;
  cudaStream_t side = nullptr;         // multi-GPU: the halo exchange overlapped with the interior SpMM
  cudaEvent_t ev_p = nullptr, ev_h = nullptr;
  int nsm = 148;
  double* partials = nullptr;
  size_t pcap = 0;  // doubles
  Comm* comm = nullptr;
  int ensure_partials(size_t n);
};

// One triangular factor of the ILU(0) preconditioner on the device: the off-diagonal
// part as CSR, the inverse diagonal (null: unit), and the rows ordered by level
// (host level boundaries; every row of a level is independent of the others).
struct DevTri {
  int* rp = nullptr;
  int* ci = nullptr;
  void* val = nullptr;
  void* dinv = nullptr;
  void* diag = nullptr;  // the diagonal itself (null: unit), for products with the factor
  int* order = nullptr;
  std::vector<int> lvl;
  int* flags = nullptr;  // n row-done flags + a work counter (sync-free solve; allocated on first use)
};
// Right ILU(0) preconditioner M = L U (ilu.cu): M^-1 = U^-1 L^-1, M^-H = L^-H U^-H
struct Prec {
  long long n = 0;
  bool cplx = false;
  DevTri L, U, UH, LH;
  std::vector<double> factor;  // the factor values on A's pattern (host copy, for parity tests)
  // ILUTP (kind 1): M = Pi^T L U; perm[k] = the row of A pivoted at step k (device, null when
  // no row moved); host copies of the factor's pivot-order CSR and of perm, for tests
  int kind = 0;
  int* perm = nullptr;
  std::vector<int> frp, fci, hperm;
  void* scratch[2] = {nullptr, nullptr};
  size_t scratch_bytes = 0;
};

struct Mat {
  Ctx* ctx = nullptr;
  long long n = 0, nnz = 0, nnzH = 0;
  bool cplx = false;
  int* rp = nullptr;
  int* ci = nullptr;
  void* val = nullptr;
  bool has_adj = false;
  int* rpH = nullptr;
  int* ciH = nullptr;
  void* valH = nullptr;
  // Block-sparse form (srk_matrix_create_bsr): nb block rows of bs x bs blocks
  bool bsr = false;
  int bs = 0, unit_diag = 0;
  long long nb = 0, nnzb = 0;
  int* brp = nullptr;
  int* bci = nullptr;
  void* bval = nullptr;
  int* border = nullptr;  // visiting order of the block rows (srk_matrix_set_row_order) or null
  Prec* prec = nullptr;  // right ILU(0) preconditioner (srk_matrix_ilu0), or null
  // Balanced row order (irregular row lengths, e.g. config 5's power law): a copy
  // of the CSR with rows sorted by decreasing length (stable), so that the rows a
  // warp processes together have similar lengths; perm[l] = original row of
  // sorted row l (the SpMM writes Q[perm[l]]). Null when the lengths are regular.
  struct Sorted {
    int* rp = nullptr;
    int* ci = nullptr;
    void* val = nullptr;
    int* perm = nullptr;
  } srt, srtH;
  // SELL-32-sigma form of an irregular operator (narrow blocks, s * esz <= 32 B): rows sorted by
  // decreasing length inside windows of sigma rows, chunks of 32 rows stored column-major and
  // padded to the chunk's longest row (column -1), chunks visited by decreasing width
  struct Sell {
    int* cs = nullptr;     // nchunk + 1 chunk offsets (entries)
    int* ci = nullptr;
    void* val = nullptr;
    int* row = nullptr;    // 32 * nchunk output rows (-1: none)
    int* order = nullptr;  // chunk visiting order
    long long nchunk = 0, entries = 0;
    int sigma = 0;
  } sell, sellH;
  // multi-GPU (dist): the local rows split into interior rows (owned columns only) and
  // boundary rows (at least one ghost column), each as a row-list copy (Sorted layout,
  // perm = output row), so the interior product runs while the halo is in flight
  Sorted inner, bnd, innerH, bndH;
  long long n_inner = 0, n_bnd = 0, n_innerH = 0, n_bndH = 0;
  // Banded form (band.cu): K <= 8 diagonals d_k (ascending), K arrays of npad values
  // (zero where a row has no entry on the diagonal); K = 0 when A is not banded
  struct Band {
    int K = 0;
    int off[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long npad = 0;
    void* val = nullptr;
  } band, bandH;
  // multi-GPU (row-partitioned) operator: local rows, columns [0, n) owned and
  // [n, n + n_ghost) ghost rows received from the owning ranks before each SpMM
  bool dist = false;
  Halo halo, haloH;
  double* sendbuf = nullptr;  // packed rows for the halo exchange
  size_t sendcap = 0;         // doubles
  long long ghost_rows() const { return dist ? std::max(halo.n_ghost, haloH.n_ghost) : 0; }
};

// banded operators (band.cu): detection + diagonal storage at a0, the bulk-copy SpMM
int build_band(bool cplx, long long n, const int* rp, const int* ci, const void* val, Mat::Band& b, cudaStream_t st);
bool band_supported(bool cplx, int s);
bool band_plane_pattern(const Mat::Band& b);  // 7-point operators: band_plane_kernel (takes SUMVEC epilogues)
int launch_band(bool cplx, int s, const Mat::Band& b, const void* P, void* Q, long long n, const Red* red, int nred,
                double* partials, int pstride, const int* done, int nsm, cudaStream_t st, int* grid_out);

// builds m.srt / m.srtH when the row lengths are irregular (engine.cu)
int build_balanced_order(Mat& m, bool adj, cudaStream_t st);
void free_balanced_order(Mat& m);
int build_halo_split(Mat& m, bool adj, cudaStream_t st);  // interior / boundary rows (dist operators)

int build_ilutp(Mat& m, double droptol, double thresh, cudaStream_t st);  // as build_ilu0
int build_ilu0(Mat& m, cudaStream_t st);  // 0, or 1 zero pivot / 2 out of memory / 3 CUDA error
void free_prec(Prec* p);
// Z = T^-1 R for one triangular factor (n x s row-major blocks; Z may alias R); returns
// the number of launches (>= 0) or a negative CUDA error
int launch_trsv(const DevTri& t, bool cplx, long long n, int s, const void* R, void* Z, const int* done, cudaStream_t st);
// Z = T R (the factor itself, diagonal included; Z must not alias R)
int launch_trimul(const DevTri& t, bool cplx, long long n, int s, const void* R, void* Z, cudaStream_t st);
int launch_permute(const int* perm, bool gather, bool cplx, long long n, int s, const void* src, void* dst,
                   cudaStream_t st);

// reduction request: X = source (or the SpMM output), Y = source or external
struct RQ {
  int mode;
  int x;             // source index (SpMM: ignored, X = Q)
  int y;             // source index, or -1 for yext
  const void* yext;
  int woff;          // destination offset (doubles) in the coefficient workspace
};

struct TermSpec {
  int src;
  Coef c;
};
struct OutSpec {
  void* ptr;
  std::vector<TermSpec> t;
};

inline Coef C1() { return Coef{CK_ONE, 0, 0, 0, 0}; }
inline Coef SC(int off, int neg = 0, int conj = 0) { return Coef{CK_SCALAR, off, neg, conj, 0}; }
inline Coef DG(int off, int neg = 0, int conj = 0) { return Coef{CK_DIAG, off, neg, conj, 0}; }
inline Coef FU(int off, int neg = 0, int herm = 0) { return Coef{CK_FULL, off, neg, 0, herm}; }
constexpr int O0 = SRC_OUT, O1 = SRC_OUT + 1, O2 = SRC_OUT + 2, O3 = SRC_OUT + 3;

// Kernel-call helper bound to one (ctx, operator, dtype, n).
// Per-launch CUDA-event timing (bench.py's live roofline): tags
enum ProfTag : int { PT_SPMM = 0, PT_SPMM_ADJ = 1, PT_UPD = 2, PT_FIN = 3, PT_COEF = 4, PT_OTHER = 5, PT_N = 6 };
// Each record also carries the launch's algorithmic bytes (every
// operand read once, every result written once, A's arrays once) and a signature
// (SpMM: block width; update: 16 * inputs + outputs) so that a caller can compute
// the achieved bandwidth of every kernel of an iteration.
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> ev;   // pairs (start, stop)
  std::vector<int> tag, sig;
  std::vector<double> bytes;
  size_t used = 0;               // pairs used since the last read
  void begin(int t, cudaStream_t st, int signature = 0, double nbytes = 0.0);
  void end(cudaStream_t st);
  int read(double* ms, long long* cnt, int ntag);  // sums per tag, resets
  // per-launch records since the last read (resets); returns the record count
  int read_launches(int* tag_out, int* sig_out, double* ms_out, double* bytes_out, int max);
  ~Prof();
};

struct QmrVec {  // eGl-QMR fused tail: the left Lanczos vectors and their coefficients' offsets in ws
  void *Wt, *Qv;
  const void* AHQ;
  int off_bx, off_invxi, off_c2;
};

struct Eng {
  Prof* prof = nullptr;
  Ctx* c = nullptr;
  const Mat* A = nullptr;
  bool cplx = false;
  long long n = 0;
  double* ws = nullptr;   // coefficient workspace (device)
  double* wstage = nullptr;  // multi-rank: per-rank sums before the allreduce (same layout as ws)
  const int* done = nullptr;
  int err = 0;            // first CUDA error
  int nlaunch = 0;        // kernels launched (instrumentation)
  int spmm(bool adj, const void* P, void* Q, int s, std::vector<RQ> reds);
  int halo(bool adj, const void* P, int s, cudaStream_t hs = nullptr);
  int spmm_split(bool adj, const void* P, void* Q, int s, const std::vector<RQ>& reds, const Mat::Sorted& in,
                 long long ni, const Mat::Sorted& bd, long long nbd);
  int upd(int s, std::vector<const void*> in, std::vector<OutSpec> outs, std::vector<RQ> reds);
  // Gl / eGl-QMR: (D, S, X, R) of this iteration and P of the next in one pass (qmr_tail.cu);
  // offsets into ws of eta, f, 1/rho', c1' and of ||R||^2. qmr_tail_ok: the blocks are whole 16-byte units
  bool qmr_tail_ok(int s) const { return ((n * (long long)s * (cplx ? 16 : 8)) % 16) == 0; }
  int qmr_tail(int s, void* P, void* D, const void* Pt, void* S, void* X, void* R, const void* Vt, int off_eta,
               int off_f, int off_invrho, int off_c1, int woff_r2, const QmrVec* v = nullptr);
  // a scalar-coefficient update as a flat plan (flat_upd.cu): inputs, outputs, coefficient offsets in ws
  // and the workspace offsets of the plan's reductions, in the plan's order; needs qmr_tail_ok(s)
  int flat(int plan, int s, std::vector<const void*> in, std::vector<void*> out, std::vector<int> coff,
           std::vector<int> woff);
  // eGl-BiCG (egl_flat.cu; needs qmr_vec_ok(s)): which = 0: X += alpha P, R -= alpha Q with sum(r̂^H R) and
  // ||R||^2 for the new r̂ = r̂ - conj(alpha) q̂ (kept in registers); which = 1: P = R + beta P, r̂ stored,
  // p̂ = r̂ + conj(beta) p̂
  int egl_bicg_flat(int which, int s, void* X, void* R, void* P, const void* Q, void* rh, void* ph, const void* qh,
                    int off_alpha, int off_beta, int woff_rhon, int woff_r2);
  // eGl: the n-vector updates ride in the two block kernels (whole 16-byte units per block row)
  bool qmr_vec_ok(int s) const { return ((long long)s * (cplx ? 16 : 8)) % 16 == 0; }
  int qmr_vt(int s, const void* Pt, void* Vt, const void* AHQ, const void* Wt, int off_br, int off_bx, int woff_rho2,
             int woff_k1, int woff_xi2);
  // s x s Gram Y^H X on the FP64 tensor cores (gram_mma.cu), written to ws + woff
  int gram_full(const void* X, const void* Y, int s, int woff);
  int spmm_bsr(bool adj, const void* P, void* Q, int s, const std::vector<RQ>& reds);
  // right-preconditioned operator A M^-1 (adjoint: M^-H A^H), M = the operator's ILU(0)
  int spmm_prec(bool adj, const void* P, void* Q, int s, const std::vector<RQ>& reds);
  // X = M^-1 Y (the iterate of the preconditioned system back to the original one)
  int prec_solve(bool adj, const void* Y, void* X, int s);
  // Y = M X
  int prec_mul(const void* X, void* Y, int s);
  bool raw = false;  // inside spmm_prec: the plain operator
  int grid_for(int cap, bool full, bool is_spmm, size_t smem, int nin) const;
};

}  // namespace srk
