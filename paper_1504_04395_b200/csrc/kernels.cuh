// kernels.cuh — argument structs shared by the host driver and the block kernels.
#pragma once
#include "common.cuh"

namespace srk {

// ----- reductions fused into the epilogue of a block kernel -----
// Inner-product convention <x, y> = y^H x, <X, Y> = tr(Y^H X).
enum RedMode : int {
  RED_NONE = 0,
  RED_NORM2 = 1,     // ||X||_F^2                            -> 1 double
  RED_DIAG = 2,      // (y_c^H x_c)_c, per column (Alg. 1)    -> s values
  RED_TRACE = 3,     // tr(Y^H X) (Alg. 2)                    -> 1 value
  RED_SUMVEC = 4,    // sum(y^H X), y an n-vector (Alg. 4)    -> 1 value
  RED_FULL = 5,      // Y^H X, s x s (Alg. 3/5 Grams)         -> s*s values (row-major: [a][c] = y_a^H x_c)
  RED_COLNORM2 = 6,  // (||x_c||^2)_c                        -> s doubles
};

// number of doubles a reduction produces
__host__ __device__ inline int red_len(int mode, int s, bool cplx) {
  const int nd = cplx ? 2 : 1;
  switch (mode) {
    case RED_NORM2: return 1;
    case RED_DIAG: return s * nd;
    case RED_TRACE: return nd;
    case RED_SUMVEC: return nd;
    case RED_FULL: return s * s * nd;
    case RED_COLNORM2: return s;
    default: return 0;
  }
}

// source encoding for terms / reductions: 0..5 = input block b, 6..9 = output j (6 + j)
constexpr int SRC_OUT = 6;

struct Red {
  int mode;
  int xsrc;          // block whose rows are X
  int ysrc;          // block whose rows are Y (-1: yext)
  const void* yext;  // external Y (n x s block, or n-vector for RED_SUMVEC)
  int poff;          // offset of this reduction inside a CTA partial (doubles)
};

enum CoefKind : int { CK_ONE = 0, CK_SCALAR = 1, CK_DIAG = 2, CK_FULL = 3 };

struct Coef {
  int kind;  // CoefKind
  int off;   // offset into the coefficient workspace (doubles); value(s) in the block's dtype
  int neg;   // multiply by -1
  int conj;  // conjugate the coefficient values
  int herm;  // CK_FULL only: use M^H instead of M
};

constexpr int MAX_IN = 6;
constexpr int MAX_OUT = 4;
constexpr int MAX_RED = 3;
constexpr int MAX_SRC = MAX_IN + MAX_OUT;  // a term's source: input b, or an earlier output (MAX_IN + o)
constexpr int CK_NONE = -1;

// Generic fused block update / Gram kernel arguments:
//   out_o = sum_b in_b * cf[o][b] + sum_{o' < o} out_o' * cf[o][MAX_IN + o']   (row by row)
// with every coefficient scalar, diagonal or s x s (CK_NONE = absent term), plus up to
// MAX_RED reductions over inputs/outputs, written as per-CTA partials.
struct UpdArgs {
  const void* in[MAX_IN];
  void* out[MAX_OUT];    // nullptr: output kept in registers only (e.g. a Gram operand)
  Coef cf[MAX_OUT][MAX_SRC];
  int cslot[MAX_OUT][MAX_SRC];  // offset (in values of T) of each staged coefficient in smem
  int cslot_total;
  Red red[MAX_RED];
  int nin, nout, nred;
  const double* ws;    // coefficient workspace
  double* partials;    // [gridDim.x][pstride]
  int pstride;
  long long n;
  int s;
  int vec;             // rows 16-byte aligned (real: s even)
  const int* done;     // skip everything when *done != 0 (device convergence flag)
};

// SpMM Q = A P (CSR, row-interleaved blocks) with fused epilogue reductions over
// (X = Q) and an optional on-the-fly axpy of the output: Q = A P (never in place).
struct SpmmArgs {
  const int* row_ptr;
  const int* col_idx;
  const void* val;
  const void* P;
  void* Q;
  long long n;
  int s;
  int vec;
  Red red[2];
  int nred;
  double* partials;
  int pstride;
  const int* done;
  const int* perm;  // balanced row order: CSR arrays are in sorted order, output row = perm[row]
  int team;         // narrow rows: a team of lanes per row (long / irregular rows) instead of a lane per row
  // SELL-32-sigma form (narrow blocks on irregular operators; null: not used): chunk c holds the
  // entries of 32 rows column-major at [cs[c], cs[c + 1]) (width = that / 32, padding column -1),
  // row[32 c + lane] = the output row (-1: none), order = chunks by decreasing width (or null)
  const int* sell_cs;
  const int* sell_ci;
  const void* sell_val;
  const int* sell_row;
  const int* sell_order;
  long long sell_nchunk;
};

// s x s Gram Y^H X on the FP64 tensor cores (gram_mma.cu); the real view of the
// blocks: n rows of w = s (real) or 2s (complex, interleaved) doubles.
struct GramArgs {
  const double* X;
  const double* Y;
  long long n;
  int w;
  int s;
  int cplx;
  double* partials;  // [gridDim.x][pstride], the Gram at offset 0 in the FULL layout
  int pstride;
  const int* done;
};

// Block-sparse (BSR) SpMM, 12 x 12 complex blocks (bsr.cu)
struct BsrArgs {
  const int* brp;   // nb + 1 block-row pointers
  const int* bci;   // block columns (sorted within a block row)
  const void* val;  // nnzb blocks of 12 x 12 complex, row-major
  const void* P;
  void* Q;
  long long nb;
  const int* order;  // visiting order of the block rows (a permutation of [0, nb)) or null
  int unit_diag;    // Q_I += P_I (identity diagonal blocks not stored)
  const int* done;
  // fused epilogue reductions over X = Q (NORM2, COLNORM2, DIAG, TRACE, SUMVEC)
  Red red[2];
  int nred;
  double* partials;  // [gridDim.x][pstride]
  int pstride;
};

// Gl / eGl-QMR fused tail (qmr_tail.cu): D, S, X, R of iteration k and P of iteration k+1
// in one pass over flat blocks of `units` 16-byte units; ||R||^2 into partials[cta*pstride + poff].
struct QmrTailArgs {
  void *P, *D, *S, *X, *R;   // read and rewritten
  const void *Pt, *Vt;       // read
  long long units;
  const double* ws;
  int off_eta, off_f, off_invrho, off_c1;  // offsets (doubles) of eta, f, 1/rho', c1' in ws
  double* partials;
  int pstride, poff;
  const int* done;
  // eGl (upr > 0): the n-vectors w̃ (rewritten: A^H q - bx w̃) and q (rewritten: w̃/xi' - c2' q);
  // upr = 16-byte units per block row, sh = log2(upr) or -1
  void *Wt, *Qv;
  const void* AHQ;
  int upr, sh;
  int off_bx, off_invxi, off_c2;
};
// eGl-QMR Ṽ update with the reductions of Ṽ and of the new w̃ (qmr_tail.cu); partials per CTA:
// [||Ṽ||^2, sum(w̃^H Ṽ) (ND doubles), ||w̃||^2]
struct QmrVtArgs {
  const void* Pt;
  void* Vt;
  const void *AHQ, *Wt;
  long long units;
  int upr, sh;
  const double* ws;
  int off_br, off_bx;
  double* partials;
  int pstride;
  const int* done;
};

// Flat scalar-coefficient updates as compile-time plans (flat_upd.cu)
enum FlatPlan : int { FP_STAB_S = 0, FP_STAB_XR = 1, FP_STAB_P = 2, FP_BICG_XR = 3, FP_BICG_P = 4, FP_QMR_VW = 5 };
struct FlatPlanInfo {
  int ni, no, nc, nr;
  int rmode[3];
};
struct FlatArgs {
  const void* in[6];
  void* out[3];       // may alias inputs (a unit is read and rewritten by the same thread)
  long long units;    // 16-byte units per block
  const double* ws;
  int coff[4];        // offsets (doubles) of the plan's coefficients in ws
  double* partials;   // per CTA: the plan's reductions back to back
  int pstride;
  const int* done;
};

// eGl-BiCG lean kernels (egl_flat.cu): flat blocks of `units` 16-byte units, upr units per block row
// (sh = log2(upr) or -1); n-vectors r̂, q̂, p̂; partials per CTA: [sum(r̂^H R) (ND doubles), ||R||^2]
struct EglFlatArgs {
  void *X, *R, *P;
  const void* Q;
  void *rh, *ph;
  const void* qh;
  long long units;
  int upr, sh;
  const double* ws;
  int off_alpha, off_beta;
  double* partials;
  int pstride;
  const int* done;
};

// Segments for the deterministic second-stage reduction of CTA partials.
struct FinSeg {
  int poff, len, woff;
};
struct FinArgs {
  const double* partials;
  int nblk, pstride;
  FinSeg seg[4];
  int nseg;
  double* ws;
  const int* done;
};

}  // namespace srk
