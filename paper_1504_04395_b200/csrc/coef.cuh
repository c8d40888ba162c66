// coef.cuh — device-side s x s / scalar coefficient phases of every method
// (SURVEY §8(a) a4), executed by one CTA between the block kernels. Each phase
// mirrors the corresponding lines of oracle/solvers.py (same formulas, same
// breakdown rules), but shares no code with it.
#pragma once
#include "small.cuh"

namespace srk {

// ---- control block (ints, device) ----
enum Ctl : int {
  CTL_FLAG = 0,      // 0 running, 1 converged candidate, 2 half-step candidate, 3 breakdown
  CTL_ITER = 1,      // completed iterations
  CTL_BKIND = 2,
  CTL_BITER = 3,
  CTL_CONVPEND = 4,  // set by the last coefficient phase, committed by end_iter
  CTL_NFROZEN = 5,
  CTL_DIDLE = 6,     // rank continuation (f4): 1 = no thin-QR repair pending (block kernels skip on it)
  CTL_DMASK = 8,     // deficient columns of the pending repair: Z (2 ints, 64 bits), Ẑ (2 ints)
  CTL_DMASKH = 10,
  CTL_DEFL = 12,     // columns replaced so far (report)
  CTL_FROZEN = 16,   // 64 per-column frozen flags (Li variants, reading G13)
  CTL_SIZE = 96
};
enum Flag : int { FLAG_RUN = 0, FLAG_CONV = 1, FLAG_HALF = 2, FLAG_BRK = 3 };
enum BK : int { BK_NONE = 0, BK_LANCZOS = 1, BK_GRAM = 2, BK_RANK = 3, BK_NONFINITE = 4, BK_OMEGA = 5 };

// ---- coefficient workspace slots ----
enum Slot : int {
  SL_R0N2 = 0, SL_R0N, SL_TRUE, SL_C0N,
  SL_RHO, SL_RHON, SL_DEN, SL_ALPHA, SL_BETA, SL_OMEGA, SL_BW, SL_R2, SL_S2, SL_ST, SL_TT,
  SL_G, SL_M, SL_MN, SL_AH, SL_BH,
  SL_C, SL_CH, SL_G1, SL_G2, SL_G2N, SL_GZ, SL_GZH, SL_R1, SL_R1I, SL_R1H, SL_R1HI,
  SL_R2F, SL_R2I, SL_R2H, SL_R2HI, SL_SIG, SL_SIGH, SL_AC, SL_WC, SL_GQ, SL_GQN, SL_ZZ, SL_YZ, SL_YY,
  // QMR
  SL_QRHO, SL_QXI, SL_INVRHO, SL_INVXI, SL_DELTA, SL_EPS, SL_C1, SL_C2, SL_GAMP, SL_ETA, SL_THETAP, SL_F,
  SL_RHON2, SL_XI2, SL_K1, SL_BR, SL_BX,
  SL_INVRHO_N, SL_C1_N, SL_INVXI_N, SL_C2_N,  // next iteration's 1/rho, c1 (and 1/xi, c2), known once Ṽ is formed (the fused tail, qmr_tail.cu)
  // Bl-QMR
  SL_OMP, SL_TAUT, SL_TAU, SL_TOP, SL_RII, SL_RIII, SL_TR, SL_GHAT, SL_RHOB, SL_XIB, SL_RHOBN, SL_XIBN,
  SL_PEND,
  // QR of the search directions (f3) and the rank continuation (f4)
  SL_MH, SL_MNH, SL_COLD, SL_COLDH, SL_SIGT, SL_SIGTH,
  SL_CB,  // R factor of the right-hand sides under preprocess_rhs (B = Q C_B)
  SL_TMP0, SL_TMP1, SL_TMP2, SL_TMP3, SL_TMP4,
  NSLOT
};

enum MethodId : int {
  M_LI_BICG = 0, M_GL_BICG, M_EGL_BICG, M_BL_BICG, M_BL_BICG_RQ,
  M_LI_QMR, M_GL_QMR, M_EGL_QMR, M_BL_QMR,
  M_LI_BICGSTAB, M_GL_BICGSTAB, M_BL_BICGSTAB, M_BL_BICGSTAB_RQ,
  M_BL_BICG_SQ, M_BL_BICGSTAB_SQ  // QR of the search directions (f3)
};

struct CoefArgs {
  int method;
  int phase;
  int s;
  int k1;            // 1 on the first iteration (QMR)
  int defl;          // rank policy of the rQ thin QRs: 0 BREAKDOWN(rank) (G11), 1 continuation (f4)
  double eps_brk;    // s x s LU pivot threshold relative to max|G| (G12)
  double eps_chol;   // CholQR pivot threshold relative to tr(G) (R5)
  double tol;
  double* ws;
  int* ctl;
  double* hist;
  int hist_cap;
  int off[NSLOT];
};

// One eGl-BiCG iteration (Alg. 4) for a small operator in ONE kernel on one
// CTA (latency-bound sizes, e.g. config 1: n = 1024): the same steps as the
// multi-kernel sequence of EglBiCG::seg — Q = A P with sum(p̂^H Q), q̂ = A^H p̂, the
// alpha phase, r̂ and X / R updates with sum(r̂^H R) and ||R||^2, the beta phase (with the
// convergence test), P and p̂ — separated by CTA barriers instead of kernel boundaries,
// reductions in a fixed order, the coefficient phases the same device code; it also
// ends the iteration (end_iter_kernel's counting and convergence commit).
struct SmallBiCGArgs {
  const int* rp;
  const int* ci;
  const void* val;
  const int* rpH;
  const int* ciH;
  const void* valH;
  void *X, *R, *P, *Q, *rh, *ph, *qh;
  long long n;
  int iters;  // iterations in this launch (stops early once the control flag leaves RUN)
  CoefArgs ca;
};
int launch_egl_bicg_small(bool cplx, const SmallBiCGArgs& g, cudaStream_t st);
// The same for eGl-QMR (the 18-block plan of QMR::seg): the coefficient
// phases 1-5 of qmr_scalar, the P / q and W̃ / Ṽ / (D, S, X, R) updates with their
// reductions, and Q~ = A P with sum(q^H P~), A^H q.
struct SmallQMRArgs {
  const int* rp;
  const int* ci;
  const void* val;
  const int* rpH;
  const int* ciH;
  const void* valH;
  void *X, *R, *Vt, *P, *Pt, *D, *S, *Wt, *Qv, *AHQ;
  long long n;
  int iters;
  CoefArgs ca;
};
int launch_egl_qmr_small(bool cplx, const SmallQMRArgs& g, cudaStream_t st);
// Bl-BiCGStab-rQ for a small operator, one iteration per pass of ONE CTA
// (config 1's second method): the products, the s x s Grams (fixed-order CTA sums), the
// coefficient phases 1-6 (the same device code as the multi-kernel path), the updates.
struct SmallBlStabArgs {
  const int* rp;
  const int* ci;
  const void* val;
  void *X, *Qr, *Q0, *V, *W, *Z, *Y;
  long long n;
  int iters;
  long long ws_doubles;  // the coefficient workspace is staged in shared memory for the launch
  CoefArgs ca;
};
int launch_bl_bicgstab_rq_small(bool cplx, const SmallBlStabArgs& g, cudaStream_t st);
constexpr int SMALL_BL_SMAX = 4;  // widths of the one-CTA block kernel
constexpr long long SMALL_N_MAX = 16384;  // one-CTA eGl-BiCG up to this many rows

}  // namespace srk
