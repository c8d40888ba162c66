// block_kernels.cuh — templates of the hot-path kernels over row-interleaved
// n x s blocks (instantiated per dtype in blk_f64.cu / blk_c128.cu).
//
//  * spmm_kernel   Q = A P, CSR, one lane group per row, R rows per group in
//                  flight: each nonzero a_ij is read once and applied to the s
//                  contiguous values of P row j (PAPER.md P:66-74, P:128-132,
//                  P:142-144), with the s x s / trace / sum /
//                  diag Gram partials fused into the epilogue (
//                  P:155-158, 178, 192-195, 243-249, 443-447).
//  * upd_kernel    fused multi-output block updates out = sum_t src_t*coef_t with
//                  scalar (Gl/eGl), diagonal (Li) or s x s (Bl, "BLAS3 GEMM"
//                  P:290-297) coefficients read from device memory, plus fused
//                  reductions. All NI inputs of R rows are
//                  loaded before any arithmetic (memory-level parallelism).
#pragma once
#include <algorithm>

#include "kernels.cuh"

namespace srk {

// Accumulators for one reduction held by one lane (capacity S).
template <typename T, int S, bool FC>
struct RedAcc {
  using L = Lay<T, S>;
  // FULL (FC) needs S x EPL values; the other modes use the first EPL.
  // (the in-kernel s x s Gram is compiled up to S = 16; wider Grams run on the tensor cores)
  static constexpr int N = (FC && S <= 16) ? S * L::EPL : L::EPL;
  T v[N];
};

template <typename T, int S, bool FC>
__device__ __forceinline__ void red_zero(RedAcc<T, S, FC>& a) {
#pragma unroll
  for (int i = 0; i < RedAcc<T, S, FC>::N; ++i) a.v[i] = Ar<T>::zero();
}

__device__ __forceinline__ double re_of(double v) { return v; }
__device__ __forceinline__ double re_of(double2 v) { return v.x; }

// Every non-FULL reduction accumulates the same per-row form  acc += conj(y) .* x
// (lane elements): y = x for NORM2 / COLNORM2 (|x|^2 in the real part), the
// broadcast vector entry for SUMVEC, the Y row for DIAG / TRACE — so the per-row
// cost is EPL fused multiply-adds and no mode dispatch; the mode only matters in
// red_flush.
template <typename T, int S, bool FC>
__device__ __forceinline__ void red_acc(RedAcc<T, S, FC>& a, const T (&x)[Lay<T, S>::EPL],
                                        const T (&y)[Lay<T, S>::EPL]) {
#pragma unroll
  for (int e = 0; e < Lay<T, S>::EPL; ++e) a.v[e] = Ar<T>::cfma(y[e], x[e], a.v[e]);
}

// FULL (s x s Gram X^H Y, block methods only): a.v[k][e] += conj(Y[:, k]) X[:, col(e)]
template <typename T, int S, bool FC>
__device__ __forceinline__ void red_full(RedAcc<T, S, FC>& a, const T (&x)[Lay<T, S>::EPL],
                                         const T (&y)[Lay<T, S>::EPL], int base, int s, unsigned gmask) {
  using L = Lay<T, S>;
  if constexpr (FC && S <= 16) {
#pragma unroll
    for (int k = 0; k < S; ++k) {
      if (k < s) {
        const T yk = row_get<T, S>(y, base, k, gmask);
#pragma unroll
        for (int e = 0; e < L::EPL; ++e) a.v[k * L::EPL + e] = Ar<T>::cfma(yk, x[e], a.v[k * L::EPL + e]);
      }
    }
  }
}

// y operand kind of a reduction (CTA-uniform): 0 = x itself, 1 = broadcast n-vector
// entry, 2 = a row (source block or external block)
__device__ __forceinline__ int red_ykind(int mode) {
  return (mode == RED_NORM2 || mode == RED_COLNORM2) ? 0 : (mode == RED_SUMVEC ? 1 : 2);
}

// One row of one reduction with a runtime (CTA-uniform) mode.
template <typename T, int S, bool FC>
__device__ __forceinline__ void red_dispatch_row(int mode, RedAcc<T, S, FC>& a, const T (&x)[Lay<T, S>::EPL],
                                                 const T (&y)[Lay<T, S>::EPL], T yv, int base, int s,
                                                 unsigned gmask) {
  using L = Lay<T, S>;
  if constexpr (FC) {
    if (mode == RED_FULL) {
      red_full<T, S, FC>(a, x, y, base, s, gmask);
      return;
    }
  }
  const int yk = red_ykind(mode);
  T yy[L::EPL];
#pragma unroll
  for (int e = 0; e < L::EPL; ++e) yy[e] = yk == 0 ? x[e] : (yk == 1 ? yv : y[e]);
  red_acc<T, S, FC>(a, x, yy);
}

// CTA-level reduction of one RedAcc into partials[blockIdx.x*pstride + poff ...].
// Order: xor-butterfly over lane groups, then warps summed in index order by
// thread 0..len-1 — fixed for a given launch configuration.
// The participating warps are wfirst .. wfirst+nw-1 (all warps by default); they
// synchronise with named barrier `bar` (0 = __syncthreads).
template <typename T, int S, int MODE, bool FC>
__device__ void red_flush(RedAcc<T, S, FC>& a, double* __restrict__ partials, int pstride, int poff, int s,
                          double* smem /* >= nwarps * len doubles */, int wfirst = 0, int nw = 0, int bar = 0) {
  using L = Lay<T, S>;
  constexpr int ND = Ar<T>::ND;
  const int nwarps = nw > 0 ? nw : (int)(blockDim.x >> 5);
  const int lane = threadIdx.x & 31, warp = (int)(threadIdx.x >> 5) - wfirst;
  auto sync = [&]() {
    if (bar == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nwarps * 32) : "memory");
  };
  const int g = lane % L::G;
  // 1) sum over the lane groups of this warp (lanes with equal g hold the same entries)
#pragma unroll
  for (int m = L::G; m < 32; m <<= 1) {
#pragma unroll
    for (int i = 0; i < RedAcc<T, S, FC>::N; ++i) a.v[i] = Ar<T>::add(a.v[i], Ar<T>::shfl_xor(a.v[i], m));
  }
  const int len = red_len(MODE, s, Ar<T>::cplx);
  // 2) lanes of group 0 scatter their entries into this warp's smem slice
  double* w = smem + warp * len;
  if constexpr (MODE == RED_NORM2 || MODE == RED_TRACE || MODE == RED_SUMVEC) {
    // scalar result: reduce over the G lanes of group 0 first (fixed xor order)
    double rs = 0.0;
    T vs = Ar<T>::zero();
#pragma unroll
    for (int e = 0; e < L::EPL; ++e) {
      rs += re_of(a.v[e]);
      vs = Ar<T>::add(vs, a.v[e]);
    }
#pragma unroll
    for (int m = 1; m < L::G; m <<= 1) {
      rs += __shfl_xor_sync(0xffffffffu, rs, m);
      vs = Ar<T>::add(vs, Ar<T>::shfl_xor(vs, m));
    }
    if (lane == 0) {
      if constexpr (MODE == RED_NORM2) w[0] = rs;
      else Ar<T>::st(w, vs);
    }
  } else if constexpr (MODE == RED_DIAG || MODE == RED_COLNORM2) {
    if (lane < L::G) {
#pragma unroll
      for (int e = 0; e < L::EPL; ++e) {
        const int c = L::col(g, e);
        if (c < s) {
          if constexpr (MODE == RED_COLNORM2) w[c] = re_of(a.v[e]);
          else Ar<T>::st(w + c * ND, a.v[e]);
        }
      }
    }
  } else if constexpr (MODE == RED_FULL && FC && S <= 16) {
    if (lane < L::G) {
#pragma unroll
      for (int k = 0; k < S; ++k) {
        if (k < s) {
#pragma unroll
          for (int e = 0; e < L::EPL; ++e) {
            const int c = L::col(g, e);
            if (c < s) Ar<T>::st(w + (k * s + c) * ND, a.v[k * L::EPL + e]);
          }
        }
      }
    }
  }
  sync();
  // 3) sum the warps' slices in warp order
  for (int j = (int)threadIdx.x - wfirst * 32; j < len; j += nwarps * 32) {
    double acc = 0.0;
    for (int q = 0; q < nwarps; ++q) acc += smem[q * len + j];
    partials[(size_t)blockIdx.x * pstride + poff + j] = acc;
  }
  sync();
}

template <typename T, int S, bool FC>
__device__ void red_dispatch_flush(int mode, RedAcc<T, S, FC>& a, double* partials, int pstride, int poff, int s,
                                   double* smem, int wfirst = 0, int nw = 0, int bar = 0) {
  switch (mode) {
    case RED_NORM2: red_flush<T, S, RED_NORM2, FC>(a, partials, pstride, poff, s, smem, wfirst, nw, bar); break;
    case RED_COLNORM2: red_flush<T, S, RED_COLNORM2, FC>(a, partials, pstride, poff, s, smem, wfirst, nw, bar); break;
    case RED_DIAG: red_flush<T, S, RED_DIAG, FC>(a, partials, pstride, poff, s, smem, wfirst, nw, bar); break;
    case RED_TRACE: red_flush<T, S, RED_TRACE, FC>(a, partials, pstride, poff, s, smem, wfirst, nw, bar); break;
    case RED_SUMVEC: red_flush<T, S, RED_SUMVEC, FC>(a, partials, pstride, poff, s, smem, wfirst, nw, bar); break;
    case RED_FULL: red_flush<T, S, RED_FULL, FC>(a, partials, pstride, poff, s, smem, wfirst, nw, bar); break;
    default: break;
  }
}

// ============================================================================
// SpMM: Q = A P  (R rows per lane group in flight; EX = exact width s == S)
// The nonzero loop is warp-uniform (trip count = the warp's longest row batch)
// and every gather load is unconditional (absent entries use column 0 with a
// zero value), so the CW*R loads of a step issue back to back.
// ============================================================================
template <typename T, int S, bool FC, int R, bool EX, int BC = 8, bool YPRE = true, int MINB = 2, int BATCH = 8, int PD = 1>
__global__ void __launch_bounds__(256, FC ? (S <= 8 ? 2 : 1) : MINB) spmm_kernel(SpmmArgs a) {
  if (a.done && *a.done) return;
  using L = Lay<T, S>;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int g = lane % L::G;
  const int base = lane - g;
  const unsigned gmask = (L::G == 32) ? 0xffffffffu : (((1u << L::G) - 1u) << base);
  // Block-cyclic row mapping: a CTA owns blocks of BC consecutive steps (step =
  // 8 warps x RPW groups x R rows), blocks dealt round-robin over the grid. Within
  // a block the CTA sweeps in order, so stencil neighbours a few grid lines away
  // are re-read from L1; all CTAs sweep neighbouring blocks concurrently, so the
  // far neighbours (other planes) are L2 hits and P streams from HBM about once.
  const int gin = lane / L::G;
  const long long step = (long long)(blockDim.x / 32) * L::RPW * R;
  const long long warp_off = (long long)(threadIdx.x >> 5) * L::RPW * R + (long long)gin * R;
  auto row_of = [&](long long k) {  // first row of this warp-lane-group in local step k
    const long long blk = (long long)blockIdx.x + (k / BC) * gridDim.x;
    return (blk * BC + (k % BC)) * step + warp_off;
  };
  auto step_live = [&](long long k) {  // warp-uniform
    const long long blk = (long long)blockIdx.x + (k / BC) * gridDim.x;
    return (blk * BC + (k % BC)) * step < a.n;
  };
  const T* __restrict__ P = reinterpret_cast<const T*>(a.P);
  const T* __restrict__ val = reinterpret_cast<const T*>(a.val);
  const int* __restrict__ rp = a.row_ptr;
  const int* __restrict__ ci = a.col_idx;
  T* __restrict__ Q = reinterpret_cast<T*>(a.Q);
  const int s = a.s;
  const long long n = a.n;
  const int nred = a.nred;
  const int mode0 = nred > 0 ? a.red[0].mode : RED_NONE;
  const int mode1 = nred > 1 ? a.red[1].mode : RED_NONE;
  const T* y0 = reinterpret_cast<const T*>(nred > 0 ? a.red[0].yext : nullptr);
  const T* y1 = reinterpret_cast<const T*>(nred > 1 ? a.red[1].yext : nullptr);

  RedAcc<T, S, FC> acc0, acc1;
  red_zero(acc0);
  red_zero(acc1);

  constexpr int CW = L::G >= 8 ? L::G : 8;  // CSR entries per step of a row
  constexpr int EPN = CW / L::G;            // (col, val) pairs per lane per step
  // row_ptr of one batch of R rows: (begin, end) kept raw — consuming a freshly
  // loaded register stalls the in-order warp, so lengths are formed a step later
  // (balanced row order: rp/ci/val are the length-sorted copy and the output row
  // of sorted row r is perm[r], fetched with the row pointers)
  const int* __restrict__ perm = a.perm;
  auto load_rp = [&](long long k, int (&bg)[R], int (&ln)[R], int (&pr)[R]) {
    const long long r0 = row_of(k);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const long long r = r0 + i;
      const bool in = r < n;
      bg[i] = in ? __ldg(rp + r) : 0;
      ln[i] = in ? __ldg(rp + r + 1) : 0;  // end; converted to a length by to_len
      pr[i] = (in && perm) ? __ldg(perm + r) : (int)r;
    }
  };
  auto to_len = [&](const int (&bg)[R], int (&ln)[R]) {
#pragma unroll
    for (int i = 0; i < R; ++i) ln[i] -= bg[i];
  };
  // cooperative, coalesced fetch of CW (col, val) pairs per row (streamed once with
  // evict-first loads so L2 keeps P); absent entries: column 0, value 0
  auto load_cv = [&](const int (&bg)[R], const int (&ln)[R], int j0, int (&cj)[R][EPN], T (&vj)[R][EPN]) {
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int u = 0; u < EPN; ++u) {
        const int j = j0 + g + u * L::G;
        const bool in = j < ln[i];
        cj[i][u] = in ? __ldcs(ci + bg[i] + j) : 0;
        vj[i][u] = in ? __ldcs(val + bg[i] + j) : Ar<T>::zero();
      }
  };

  // Software pipeline over the warp's row batches k = 0, 1, 2, ...: while the P
  // gathers of batch k are in flight, the (col, val) of batches up to k+PD and the
  // row pointers of batch k+PD+1 are being fetched (PD = prefetch depth).
  int bq[PD + 1][R], lq[PD + 1][R];  // row pointers (begin, length) of batches k..k+PD
  int pq[PD + 1][R];                 // output rows of batches k..k+PD
  int cq[PD][R][EPN];                // (col, val) of batches k..k+PD-1
  T vq[PD][R][EPN];
#pragma unroll
  for (int d = 0; d <= PD; ++d) {
    load_rp(d, bq[d], lq[d], pq[d]);
    to_len(bq[d], lq[d]);
  }
#pragma unroll
  for (int d = 0; d < PD; ++d) load_cv(bq[d], lq[d], 0, cq[d], vq[d]);
  for (long long k = 0; step_live(k); ++k) {  // warp-uniform loop
    const long long r0 = row_of(k);
    int (&beg)[R] = bq[0];
    int (&len)[R] = lq[0];
    int (&cj)[R][EPN] = cq[0];
    T (&vj)[R][EPN] = vq[0];
    int cjn[R][EPN];
    T vjn[R][EPN];
    int begnn[R], lennn[R], prnn[R];
    load_cv(bq[PD], lq[PD], 0, cjn, vjn);
    load_rp(k + PD + 1, begnn, lennn, prnn);
    // epilogue operand of the first reduction, requested before the gathers
    T yr0[R][L::EPL];
    T yv0[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      yv0[i] = Ar<T>::zero();
#pragma unroll
      for (int e = 0; e < L::EPL; ++e) yr0[i][e] = Ar<T>::zero();
      const long long row = pq[0][i];
      if (YPRE && r0 + i < n && mode0 != RED_NONE) {
        if (mode0 == RED_SUMVEC) yv0[i] = y0[row];
        else if (mode0 != RED_NORM2 && mode0 != RED_COLNORM2) {
          if constexpr (EX) row_load_ex_rw<T, S>(y0 + (size_t)row * S, g, yr0[i]);
          else row_load<T, S>(y0 + (size_t)row * s, g, s, a.vec, yr0[i]);
        }
      }
    }
    int maxlen = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) maxlen = max(maxlen, len[i]);
    maxlen = __reduce_max_sync(0xffffffffu, maxlen);
    T q[R][L::EPL];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int e = 0; e < L::EPL; ++e) q[i][e] = Ar<T>::zero();
    for (int j0 = 0; j0 < maxlen; j0 += CW) {
      if (j0 > 0) load_cv(beg, len, j0, cj, vj);  // rows longer than CW
      if constexpr (EX && BATCH > 0) {
        // explicit batches of BATCH entries: all gathers of a batch issued before any FMA
        static_assert(CW % BATCH == 0, "batch must divide CW");
#pragma unroll
        for (int t0 = 0; t0 < CW; t0 += BATCH) {
          T pb[R][BATCH][L::EPL];
          T vb[R][BATCH];
#pragma unroll
          for (int t = 0; t < BATCH; ++t)
#pragma unroll
            for (int i = 0; i < R; ++i) {
              const int tt = t0 + t;
              const int c = __shfl_sync(0xffffffffu, cj[i][tt / L::G], base + tt % L::G);
              vb[i][t] = Ar<T>::shfl(vj[i][tt / L::G], base + tt % L::G, 0xffffffffu);
              row_load_ex<T, S>(P + (size_t)c * S, g, pb[i][t]);
            }
#pragma unroll
          for (int t = 0; t < BATCH; ++t)
#pragma unroll
            for (int i = 0; i < R; ++i)
#pragma unroll
              for (int e = 0; e < L::EPL; ++e) q[i][e] = Ar<T>::fma(vb[i][t], pb[i][t][e], q[i][e]);
        }
        continue;
      }
#pragma unroll
      for (int t = 0; t < CW; ++t) {
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int c = __shfl_sync(0xffffffffu, cj[i][t / L::G], base + t % L::G);
          const T v = Ar<T>::shfl(vj[i][t / L::G], base + t % L::G, 0xffffffffu);
          T p[L::EPL];
          if constexpr (EX) {
            row_load_ex<T, S>(P + (size_t)c * S, g, p);
          } else {
            row_load<T, S>(P + (size_t)c * s, g, s, a.vec, p);
          }
#pragma unroll
          for (int e = 0; e < L::EPL; ++e) q[i][e] = Ar<T>::fma(v, p[e], q[i][e]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const long long row = pq[0][i];
      if (r0 + i < n) {
        if constexpr (EX) row_store_ex<T, S>(Q + (size_t)row * S, g, q[i]);
        else row_store<T, S>(Q + (size_t)row * s, g, s, a.vec, q[i]);
        // fused epilogue: reductions with X = Q
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int mode = r == 0 ? mode0 : mode1;
          if (mode == RED_NONE) continue;
          const T* yp = r == 0 ? y0 : y1;
          if (r == 0 && YPRE) {
            red_dispatch_row<T, S, FC>(mode, acc0, q[i], yr0[i], yv0[i], base, s, gmask);
          } else {
            T y[L::EPL];
            T yv = Ar<T>::zero();
#pragma unroll
            for (int e = 0; e < L::EPL; ++e) y[e] = Ar<T>::zero();
            if (mode == RED_SUMVEC) yv = yp[row];
            else if (mode != RED_NORM2 && mode != RED_COLNORM2) {
              if constexpr (EX) row_load_ex_rw<T, S>(yp + (size_t)row * S, g, y);
              else row_load<T, S>(yp + (size_t)row * s, g, s, a.vec, y);
            }
            if (r == 0) red_dispatch_row<T, S, FC>(mode, acc0, q[i], y, yv, base, s, gmask);
            else red_dispatch_row<T, S, FC>(mode, acc1, q[i], y, yv, base, s, gmask);
          }
        }
      }
    }
    // rotate the pipeline
    to_len(begnn, lennn);
#pragma unroll
    for (int i = 0; i < R; ++i) {
#pragma unroll
      for (int d = 0; d < PD; ++d) {
        bq[d][i] = bq[d + 1][i];
        lq[d][i] = lq[d + 1][i];
        pq[d][i] = pq[d + 1][i];
      }
      bq[PD][i] = begnn[i];
      lq[PD][i] = lennn[i];
      pq[PD][i] = prnn[i];
#pragma unroll
      for (int u = 0; u < EPN; ++u) {
#pragma unroll
        for (int d = 0; d + 1 < PD; ++d) {
          cq[d][i][u] = cq[d + 1][i][u];
          vq[d][i][u] = vq[d + 1][i][u];
        }
        cq[PD - 1][i][u] = cjn[i][u];
        vq[PD - 1][i][u] = vjn[i][u];
      }
    }
  }
  __syncwarp();
  if (nred > 0) red_dispatch_flush<T, S, FC>(mode0, acc0, a.partials, a.pstride, a.red[0].poff, s, smem);
  if (nred > 1) red_dispatch_flush<T, S, FC>(mode1, acc1, a.partials, a.pstride, a.red[1].poff, s, smem);
}

// ============================================================================
// Fused block update / Gram (NI = compiled input count >= nin, R rows per group)
// Every register array is indexed with compile-time indices only (sources are
// visited by unrolled loops, absent terms skipped by a uniform branch), so the
// rows stay in registers and all NI*R loads of a step are in flight together.
// ============================================================================
// MINB = 4 (<= 64 registers, 32 warps per SM) measured best for every input count on
// config-3 blocks (scripts/upd_tune.cu: 90-100% of the measured copy bandwidth)
// (the s x s-coefficient instances need more registers: 2 CTAs/SM; complex rows, one per
// lane group, fit 4 CTAs/SM with up to 2 inputs and 3 with more, without spills)
template <typename T, int S, bool FC, int NI, int R, bool EX, bool STREAM = false,
          int MINB = FC ? 2 : (sizeof(T) == 16 ? (NI <= 2 ? 4 : 3) : 4)>
__global__ void __launch_bounds__(256, MINB) upd_kernel(UpdArgs a) {
  if (a.done && *a.done) return;
  using L = Lay<T, S>;
  constexpr int ND = Ar<T>::ND;
  extern __shared__ double smem[];
  __shared__ int s_kind[MAX_OUT][MAX_SRC];
  __shared__ int s_cslot[MAX_OUT][MAX_SRC];
  const int s = a.s;
  const long long n = a.n;
  if (threadIdx.x < MAX_OUT * MAX_SRC) {
    const int o = threadIdx.x / MAX_SRC, b = threadIdx.x % MAX_SRC;
    s_kind[o][b] = (o < a.nout) ? a.cf[o][b].kind : CK_NONE;
    s_cslot[o][b] = a.cslot[o][b];
  }
  // ---- stage coefficients into shared memory (neg/conj/herm applied once),
  // padded to the lane layout's row width PW
  T* cs = reinterpret_cast<T*>(smem);
  for (int o = 0; o < a.nout; ++o)
    for (int b = 0; b < MAX_SRC; ++b) {
      const Coef& cf = a.cf[o][b];
      if (cf.kind == CK_NONE) continue;
      T* dst = cs + a.cslot[o][b];
      constexpr int PW = L::PW;
      int cnt = cf.kind == CK_FULL ? S * PW : (cf.kind == CK_DIAG ? PW : 1);
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        T v = Ar<T>::zero();
        if (cf.kind == CK_ONE) {
          if constexpr (Ar<T>::cplx) v = mk(1.0, 0.0); else v = 1.0;
        } else if (cf.kind == CK_SCALAR) {
          v = Ar<T>::ld(a.ws + cf.off);
        } else if (cf.kind == CK_DIAG) {
          if (i < s) v = Ar<T>::ld(a.ws + cf.off + i * ND);
        } else {
          const int k = i / PW, c = i % PW;
          if (k < s && c < s) v = cf.herm ? Ar<T>::conj(Ar<T>::ld(a.ws + cf.off + (c * s + k) * ND))
                                          : Ar<T>::ld(a.ws + cf.off + (k * s + c) * ND);
        }
        if (cf.conj) v = Ar<T>::conj(v);
        if (cf.neg) v = Ar<T>::sub(Ar<T>::zero(), v);
        dst[i] = v;
      }
    }
  double* rsm = reinterpret_cast<double*>(cs + a.cslot_total);
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int g = lane % L::G;
  const int base = lane - g;
  const unsigned gmask = (L::G == 32) ? 0xffffffffu : (((1u << L::G) - 1u) << base);
  const long long groups_per_cta = (blockDim.x / 32) * L::RPW;
  const long long grp0 = (long long)blockIdx.x * groups_per_cta + (threadIdx.x >> 5) * L::RPW + lane / L::G;
  const long long gstride = (long long)gridDim.x * groups_per_cta;
  const int nin = a.nin, nout = a.nout, nred = a.nred;
  // Reductions are applied at the first "stage" at which both operands exist
  // (stage 0: inputs only; stage o+1: after output o), so an output's reductions
  // consume it while it is in registers, and the common case — x is the output
  // just formed — needs no operand selection at all.
  int rmode[MAX_RED], rx[MAX_RED], ry[MAX_RED], ryk[MAX_RED];
  int st_mask[MAX_OUT + 1];
#pragma unroll
  for (int t = 0; t <= MAX_OUT; ++t) st_mask[t] = 0;
#pragma unroll
  for (int r = 0; r < MAX_RED; ++r) {
    rmode[r] = r < nred ? a.red[r].mode : RED_NONE;
    rx[r] = r < nred ? a.red[r].xsrc : -2;
    ry[r] = r < nred ? a.red[r].ysrc : -2;
    ryk[r] = red_ykind(rmode[r]);
    if (ryk[r] == 2 && ry[r] < 0) ryk[r] = 3;  // row of an external block
    if (rmode[r] == RED_FULL) ryk[r] = ry[r] < 0 ? 3 : 2;
    if (rmode[r] != RED_NONE) {
      const int sx = rx[r] >= SRC_OUT ? rx[r] - SRC_OUT + 1 : 0;
      const int sy = (ryk[r] == 2 && ry[r] >= SRC_OUT) ? ry[r] - SRC_OUT + 1 : 0;
      st_mask[sx > sy ? sx : sy] |= 1 << r;
    }
  }

  RedAcc<T, S, FC> acc0, acc1;
  RedAcc<T, S, false> acc2;
  red_zero(acc0);
  red_zero(acc1);
  red_zero(acc2);

  // apply one term: o_row += x_row * coefficient (kind uniform over the CTA)
  auto apply = [&](T (&o_row)[L::EPL], const T (&x)[L::EPL], int kind, const T* cf) {
    if constexpr (FC) {  // s x s coefficients exist only in the block-method instances
      if (kind == CK_FULL) {
#pragma unroll
        for (int k = 0; k < S; ++k) {
          if (k < s) {
            const T xk = row_get<T, S>(x, base, k, gmask);
#pragma unroll
            for (int e = 0; e < L::EPL; ++e) o_row[e] = Ar<T>::fma(xk, cf[k * L::PW + L::col(g, e)], o_row[e]);
          }
        }
        return;
      }
    }
    if (kind == CK_DIAG) {
#pragma unroll
      for (int e = 0; e < L::EPL; ++e) o_row[e] = Ar<T>::fma(x[e], cf[L::col(g, e)], o_row[e]);
    } else {
      const T c0 = cf[0];
#pragma unroll
      for (int e = 0; e < L::EPL; ++e) o_row[e] = Ar<T>::fma(x[e], c0, o_row[e]);
    }
  };

  for (long long ch = grp0; ch * R < n; ch += gstride) {
    const long long r0 = ch * R;
    // ---- issue every load of the R rows first
    T xin[NI][R][L::EPL];
#pragma unroll
    for (int b = 0; b < NI; ++b) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
#pragma unroll
        for (int e = 0; e < L::EPL; ++e) xin[b][i][e] = Ar<T>::zero();
        if (b < nin && r0 + i < n) {
          if constexpr (EX && STREAM) row_load_ex_cs<T, S>(reinterpret_cast<const T*>(a.in[b]) + (size_t)(r0 + i) * S, g, xin[b][i]);
          else if constexpr (EX) row_load_ex_rw<T, S>(reinterpret_cast<const T*>(a.in[b]) + (size_t)(r0 + i) * S, g, xin[b][i]);
          else row_load<T, S>(reinterpret_cast<const T*>(a.in[b]) + (size_t)(r0 + i) * s, g, s, a.vec, xin[b][i]);
        }
      }
    }
    // SUMVEC operands (an n-vector entry per row) requested together with the rows
    T yvp[MAX_RED][R];
#pragma unroll
    for (int r = 0; r < MAX_RED; ++r)
#pragma unroll
      for (int i = 0; i < R; ++i) {
        yvp[r][i] = Ar<T>::zero();
        if (ryk[r] == 1 && r0 + i < n) yvp[r][i] = reinterpret_cast<const T*>(a.red[r].yext)[r0 + i];
      }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const long long row = r0 + i;
      if (row < n) {
        T xo[MAX_OUT][L::EPL];
        // reductions of stage t; ONLY_X: x is output t-1 (no selection)
        auto stage = [&](int t) {
#pragma unroll
          for (int r = 0; r < MAX_RED; ++r) {
            if (!((st_mask[t] >> r) & 1)) continue;
            T x[L::EPL], y[L::EPL];
            if (t > 0 && rx[r] == SRC_OUT + t - 1) {
#pragma unroll
              for (int e = 0; e < L::EPL; ++e) x[e] = xo[t > 0 ? t - 1 : 0][e];
            } else {
#pragma unroll
              for (int e = 0; e < L::EPL; ++e) x[e] = Ar<T>::zero();
#pragma unroll
              for (int q = 0; q < NI; ++q)
#pragma unroll
                for (int e = 0; e < L::EPL; ++e) x[e] = opaque_sel(rx[r] == q, xin[q][i][e], x[e]);
#pragma unroll
              for (int q = 0; q < MAX_OUT; ++q)
                if (q < t)
#pragma unroll
                  for (int e = 0; e < L::EPL; ++e) x[e] = opaque_sel(rx[r] == SRC_OUT + q, xo[q][e], x[e]);
            }
            if (ryk[r] == 0) {
#pragma unroll
              for (int e = 0; e < L::EPL; ++e) y[e] = x[e];
            } else if (ryk[r] == 1) {
#pragma unroll
              for (int e = 0; e < L::EPL; ++e) y[e] = yvp[r][i];
            } else if (ryk[r] == 3) {
#pragma unroll
              for (int e = 0; e < L::EPL; ++e) y[e] = Ar<T>::zero();
              if constexpr (EX) row_load_ex_rw<T, S>(reinterpret_cast<const T*>(a.red[r].yext) + (size_t)row * S, g, y);
              else row_load<T, S>(reinterpret_cast<const T*>(a.red[r].yext) + (size_t)row * s, g, s, a.vec, y);
            } else {
#pragma unroll
              for (int e = 0; e < L::EPL; ++e) y[e] = Ar<T>::zero();
#pragma unroll
              for (int q = 0; q < NI; ++q)
#pragma unroll
                for (int e = 0; e < L::EPL; ++e) y[e] = opaque_sel(ry[r] == q, xin[q][i][e], y[e]);
#pragma unroll
              for (int q = 0; q < MAX_OUT; ++q)
                if (q < t)
#pragma unroll
                  for (int e = 0; e < L::EPL; ++e) y[e] = opaque_sel(ry[r] == SRC_OUT + q, xo[q][e], y[e]);
            }
            if (FC && rmode[r] == RED_FULL) {
              if (r == 0) red_full<T, S, FC>(acc0, x, y, base, s, gmask);
              else if (r == 1) red_full<T, S, FC>(acc1, x, y, base, s, gmask);
            } else {
              if (r == 0) red_acc<T, S, FC>(acc0, x, y);
              else if (r == 1) red_acc<T, S, FC>(acc1, x, y);
              else red_acc<T, S, false>(acc2, x, y);
            }
          }
        };
        if (st_mask[0]) stage(0);
#pragma unroll
        for (int o = 0; o < MAX_OUT; ++o) {
#pragma unroll
          for (int e = 0; e < L::EPL; ++e) xo[o][e] = Ar<T>::zero();
          if (o < nout) {
#pragma unroll
            for (int b = 0; b < NI; ++b) {
              const int kind = s_kind[o][b];
              if (kind != CK_NONE) apply(xo[o], xin[b][i], kind, cs + s_cslot[o][b]);
            }
#pragma unroll
            for (int b = 0; b < o; ++b) {
              const int kind = s_kind[o][MAX_IN + b];
              if (kind != CK_NONE) apply(xo[o], xo[b], kind, cs + s_cslot[o][MAX_IN + b]);
            }
            if (a.out[o]) {
              if constexpr (EX && STREAM) row_store_ex_cs<T, S>(reinterpret_cast<T*>(a.out[o]) + (size_t)row * S, g, xo[o]);
              else if constexpr (EX) row_store_ex<T, S>(reinterpret_cast<T*>(a.out[o]) + (size_t)row * S, g, xo[o]);
              else row_store<T, S>(reinterpret_cast<T*>(a.out[o]) + (size_t)row * s, g, s, a.vec, xo[o]);
            }
            if (st_mask[o + 1]) stage(o + 1);
          }
        }
      }  // row < n
    }
  }
  __syncwarp();
  if (nred > 0) red_dispatch_flush<T, S, FC>(rmode[0], acc0, a.partials, a.pstride, a.red[0].poff, s, rsm);
  if (nred > 1) red_dispatch_flush<T, S, FC>(rmode[1], acc1, a.partials, a.pstride, a.red[1].poff, s, rsm);
  if (nred > 2) red_dispatch_flush<T, S, false>(rmode[2], acc2, a.partials, a.pstride, a.red[2].poff, s, rsm);
}

// ============================================================================
// SpMM for narrow blocks (s * esz <= 32 bytes: the A^H vector product of the
// economic variants, config 5's small-s sweep): a TEAM of lanes per row, each
// lane taking every TEAM-th nonzero (coalesced (col, val) loads, TEAM gathers of
// one short P row in flight per row), R rows per team, the partial rows summed by
// a fixed xor butterfly over the team. The team leader stores the row and
// accumulates the fused reductions over its W values.
// ============================================================================
template <typename T, int W>
struct TeamRed {  // one reduction's accumulators in a team leader
  T v[W];         // DIAG / COLNORM2 (Re) per column; [0]: NORM2 (Re), TRACE, SUMVEC
  T f[W][W];      // FULL: f[k][c] += conj(y_k) q_c
};


// one finished row of a narrow-width product (team or SELL kernel): store it and add its terms to
// the fused reductions of the lane that owns it
template <typename T, int W, bool EX>
__device__ __forceinline__ void narrow_row_out(const T (&q)[W], long long row, int s, T* __restrict__ Q,
                                               const int (&rmode)[2], const T* (&ry)[2], TeamRed<T, W> (&acc)[2]) {
  T* dst = Q + (size_t)row * (EX ? W : s);
#pragma unroll
  for (int e = 0; e < W; ++e)
    if (EX || e < s) dst[e] = q[e];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int md = rmode[r];
    if (md == RED_NONE) continue;
    if (md == RED_NORM2) {
#pragma unroll
      for (int e = 0; e < W; ++e) acc[r].v[0] = Ar<T>::cfma(q[e], q[e], acc[r].v[0]);
    } else if (md == RED_COLNORM2) {
#pragma unroll
      for (int e = 0; e < W; ++e) acc[r].v[e] = Ar<T>::cfma(q[e], q[e], acc[r].v[e]);
    } else if (md == RED_SUMVEC) {
      const T y = ry[r][row];
#pragma unroll
      for (int e = 0; e < W; ++e) acc[r].v[0] = Ar<T>::cfma(y, q[e], acc[r].v[0]);
    } else {
      T y[W];
      const T* ys = ry[r] + (size_t)row * (EX ? W : s);
#pragma unroll
      for (int e = 0; e < W; ++e) y[e] = (EX || e < s) ? ys[e] : Ar<T>::zero();
      if (md == RED_FULL) {
#pragma unroll
        for (int k = 0; k < W; ++k)
#pragma unroll
          for (int c = 0; c < W; ++c) acc[r].f[k][c] = Ar<T>::cfma(y[k], q[c], acc[r].f[k][c]);
      } else if (md == RED_TRACE) {
#pragma unroll
        for (int e = 0; e < W; ++e) acc[r].v[0] = Ar<T>::cfma(y[e], q[e], acc[r].v[0]);
      } else {
#pragma unroll
        for (int e = 0; e < W; ++e) acc[r].v[e] = Ar<T>::cfma(y[e], q[e], acc[r].v[e]);
      }
    }
  }
}

// CTA partials of the narrow-width kernels: the lanes that own rows (every FIRST-th lane) are
// summed by a fixed xor butterfly, then the warps in index order
template <typename T, int W, int FIRST>
__device__ __forceinline__ void narrow_flush(const SpmmArgs& a, int s, const int (&rmode)[2], TeamRed<T, W> (&acc)[2],
                                             double* smem) {
  constexpr int ND = Ar<T>::ND;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (r >= a.nred) break;
    const int md = rmode[r];
    const int len = red_len(md, s, ND == 2);
    double* w = smem + (size_t)warp * len;
#pragma unroll
    for (int m = FIRST; m < 32; m <<= 1)
#pragma unroll
      for (int c = 0; c < W; ++c) {
        acc[r].v[c] = Ar<T>::add(acc[r].v[c], Ar<T>::shfl_xor(acc[r].v[c], m));
#pragma unroll
        for (int k = 0; k < W; ++k) acc[r].f[k][c] = Ar<T>::add(acc[r].f[k][c], Ar<T>::shfl_xor(acc[r].f[k][c], m));
      }
    if (lane == 0) {
      if (md == RED_NORM2) w[0] = re_of(acc[r].v[0]);
      else if (md == RED_TRACE || md == RED_SUMVEC) Ar<T>::st(w, acc[r].v[0]);
      else if (md == RED_COLNORM2) {
#pragma unroll
        for (int c = 0; c < W; ++c)
          if (c < s) w[c] = re_of(acc[r].v[c]);
      } else if (md == RED_DIAG) {
#pragma unroll
        for (int c = 0; c < W; ++c)
          if (c < s) Ar<T>::st(w + c * ND, acc[r].v[c]);
      } else {
#pragma unroll
        for (int k = 0; k < W; ++k)
#pragma unroll
          for (int c = 0; c < W; ++c)
            if (k < s && c < s) Ar<T>::st(w + (k * s + c) * ND, acc[r].f[k][c]);
      }
    }
    __syncthreads();
    const int nw = blockDim.x >> 5;
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
      double sum = 0.0;
      for (int q2 = 0; q2 < nw; ++q2) sum += smem[q2 * len + j];
      a.partials[(size_t)blockIdx.x * a.pstride + a.red[r].poff + j] = sum;
    }
    __syncthreads();
  }
}

template <typename T, int W, int TEAM, int R, bool EX>
__global__ void __launch_bounds__(256, W * sizeof(T) >= 32 ? 2 : 4) spmv_team_kernel(SpmmArgs a) {
  if (a.done && *a.done) return;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane % TEAM, team = lane / TEAM;
  constexpr int TPW = 32 / TEAM;  // teams per warp
  const long long n = a.n;
  const int s = a.s;
  const int* __restrict__ rp = a.row_ptr;
  const int* __restrict__ ci = a.col_idx;
  const T* __restrict__ val = reinterpret_cast<const T*>(a.val);
  const T* __restrict__ P = reinterpret_cast<const T*>(a.P);
  T* __restrict__ Q = reinterpret_cast<T*>(a.Q);
  const int* __restrict__ perm = a.perm;
  const int nred = a.nred;
  int rmode[2];
  const T* ry[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    rmode[r] = r < nred ? a.red[r].mode : RED_NONE;
    ry[r] = r < nred ? reinterpret_cast<const T*>(a.red[r].yext) : nullptr;
  }
  TeamRed<T, W> acc[2];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < W; ++c) {
      acc[r].v[c] = Ar<T>::zero();
#pragma unroll
      for (int k = 0; k < W; ++k) acc[r].f[k][c] = Ar<T>::zero();
    }
  auto load_row = [&](long long c, T (&p)[W]) {
    const T* src = P + (size_t)c * (EX ? W : s);
    if constexpr (EX && W * sizeof(T) % 16 == 0) {
#pragma unroll
      for (int q = 0; q < W * (int)sizeof(T) / 16; ++q) {
        const double2 d = __ldg(reinterpret_cast<const double2*>(src) + q);
        if constexpr (sizeof(T) == 16) {
          p[q] = *reinterpret_cast<const T*>(&d);
        } else {
          reinterpret_cast<double*>(p)[2 * q] = d.x;
          reinterpret_cast<double*>(p)[2 * q + 1] = d.y;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < W; ++e) p[e] = (EX || e < s) ? __ldg(src + e) : Ar<T>::zero();
    }
  };
  const long long nwarp = (long long)gridDim.x * (blockDim.x >> 5);
  const long long rows_per_it = (long long)TPW * R;
  for (long long wi = (long long)blockIdx.x * (blockDim.x >> 5) + warp; wi * rows_per_it < n; wi += nwarp) {
    const long long r0 = wi * rows_per_it + (long long)team * R;
    int beg[R], len[R];
    long long orow[R];
    int maxlen = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const long long r = r0 + i;
      const bool in = r < n;
      beg[i] = in ? __ldg(rp + r) : 0;
      len[i] = in ? __ldg(rp + r + 1) - beg[i] : 0;
      orow[i] = (in && perm) ? __ldg(perm + r) : r;
      maxlen = max(maxlen, len[i]);
    }
    T q[R][W];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int e = 0; e < W; ++e) q[i][e] = Ar<T>::zero();
#ifdef TEAM_UNROLL1
#pragma unroll 1
#endif
    for (int j = t; j < maxlen; j += TEAM) {
      int cj[R];
      T vj[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const bool in = j < len[i];
        cj[i] = in ? __ldcs(ci + beg[i] + j) : 0;
        vj[i] = in ? __ldcs(val + beg[i] + j) : Ar<T>::zero();
      }
      T p[R][W];
#pragma unroll
      for (int i = 0; i < R; ++i) load_row(cj[i], p[i]);
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int e = 0; e < W; ++e) q[i][e] = Ar<T>::fma(vj[i], p[i][e], q[i][e]);
    }
    // sum the team's partial rows (fixed order)
#pragma unroll
    for (int m = 1; m < TEAM; m <<= 1)
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int e = 0; e < W; ++e) q[i][e] = Ar<T>::add(q[i][e], Ar<T>::shfl_xor(q[i][e], m));
    if (t == 0) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if (r0 + i >= n) continue;
        narrow_row_out<T, W, EX>(q[i], orow[i], s, Q, rmode, ry, acc);
      }
    }
  }
  if (nred == 0) return;
  // team leaders -> warp (xor over the teams, fixed order) -> warps in index order
  narrow_flush<T, W, TEAM>(a, s, rmode, acc, smem);
}


// SELL-32-sigma product for narrow blocks (s * esz <= 32 B; SURVEY §8(a) a0 / §7.1 "SELL-C-sigma
// mapping: one row per lane, C = 32, with sigma-window sorting for the power-law rows"): a warp owns
// a chunk of 32 rows (sorted by decreasing length inside windows of sigma rows, so the chunk is
// padded only to ITS longest row); entry j of the 32 rows is contiguous (one coalesced 128-B index
// load and one value load per step for the whole warp), every lane gathers its own P row (one 16- or
// 32-byte load) and sums its row in CSR order — no team butterfly, bitwise the sequential row sum.
// Padding entries carry column -1 and are skipped. U steps are in flight per lane.
template <typename T, int W, bool EX>
__global__ void __launch_bounds__(256, 4) sell_kernel(SpmmArgs a) {
  if (a.done && *a.done) return;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int s = a.s;
  const int* __restrict__ cs = a.sell_cs;
  const int* __restrict__ ci = a.sell_ci;
  const T* __restrict__ val = reinterpret_cast<const T*>(a.sell_val);
  const int* __restrict__ srow = a.sell_row;
  const int* __restrict__ corder = a.sell_order;
  const T* __restrict__ P = reinterpret_cast<const T*>(a.P);
  T* __restrict__ Q = reinterpret_cast<T*>(a.Q);
  int rmode[2];
  const T* ry[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    rmode[r] = r < a.nred ? a.red[r].mode : RED_NONE;
    ry[r] = r < a.nred ? reinterpret_cast<const T*>(a.red[r].yext) : nullptr;
  }
  TeamRed<T, W> acc[2];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < W; ++c) {
      acc[r].v[c] = Ar<T>::zero();
#pragma unroll
      for (int k = 0; k < W; ++k) acc[r].f[k][c] = Ar<T>::zero();
    }
  auto load_row = [&](int c, T (&p)[W]) {
    const T* src = P + (size_t)c * (EX ? W : s);
    if constexpr (EX && W * sizeof(T) % 16 == 0) {
#pragma unroll
      for (int q = 0; q < W * (int)sizeof(T) / 16; ++q) {
        const double2 d = __ldg(reinterpret_cast<const double2*>(src) + q);
        if constexpr (sizeof(T) == 16) {
          p[q] = *reinterpret_cast<const T*>(&d);
        } else {
          reinterpret_cast<double*>(p)[2 * q] = d.x;
          reinterpret_cast<double*>(p)[2 * q + 1] = d.y;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < W; ++e) p[e] = (EX || e < s) ? __ldg(src + e) : Ar<T>::zero();
    }
  };
  constexpr int U = W * sizeof(T) >= 32 ? 4 : 8;  // steps in flight
  const long long nwarp = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long k = (long long)blockIdx.x * (blockDim.x >> 5) + warp; k < a.sell_nchunk; k += nwarp) {
    const int c = corder ? __ldg(corder + k) : (int)k;
    const int base = __ldg(cs + c);
    const int w = (__ldg(cs + c + 1) - base) >> 5;
    const int row = __ldg(srow + (size_t)c * 32 + lane);  // -1: no row (the last chunk's tail)
    T q[W];
#pragma unroll
    for (int e = 0; e < W; ++e) q[e] = Ar<T>::zero();
    const int* cp = ci + base + lane;
    const T* vp = val + base + lane;
    for (int j = 0; j < w; j += U) {
      int cj[U];
      T vj[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool in = j + u < w;
        cj[u] = in ? __ldcs(cp + (size_t)(j + u) * 32) : -1;
        vj[u] = in ? __ldcs(vp + (size_t)(j + u) * 32) : Ar<T>::zero();
      }
      T p[U][W];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (cj[u] >= 0) {
          load_row(cj[u], p[u]);
        } else {
#pragma unroll
          for (int e = 0; e < W; ++e) p[u][e] = Ar<T>::zero();
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (cj[u] >= 0) {
#pragma unroll
          for (int e = 0; e < W; ++e) q[e] = Ar<T>::fma(vj[u], p[u][e], q[e]);
        }
    }
    if (row >= 0) narrow_row_out<T, W, EX>(q, row, s, Q, rmode, ry, acc);
  }
  if (a.nred == 0) return;
  narrow_flush<T, W, 1>(a, s, rmode, acc, smem);
}

// rows per group in flight
// rows per lane group in flight (measured on config 3: scripts/spmm_tune.cu)
template <typename T, int S> constexpr int spmm_rows() {
  return (Lay<T, S>::G == 1 || S >= 64) ? 1 : 2;
}
// rows per lane group: 2 for real blocks with few inputs; complex rows one at a time, at
// 3-4 CTAs/SM (config 4's complex updates: 49-50% -> 65-69% of HBM against 2 rows at 2 CTAs/SM)
template <typename T, int NI> constexpr int upd_rows() { return (sizeof(T) == 16) ? 1 : (NI <= 2 ? 2 : 1); }
template <typename T, int S> constexpr bool full_ok() { return S <= 32; }

// grid < 0: return the number of resident CTAs per SM instead of launching
template <typename T, int S, bool FC, bool EX>
int launch_spmm_tx(const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  constexpr int R = spmm_rows<T, S>();
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(spmm_kernel<T, S, FC, R, EX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  if (grid < 0) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, spmm_kernel<T, S, FC, R, EX>, block, smem);
    return nb;
  }
  spmm_kernel<T, S, FC, R, EX><<<grid, block, smem, st>>>(a);
  return (int)cudaGetLastError();
}

// grid < 0: return the number of resident CTAs per SM instead of launching
template <typename T, int W, bool EX>
int launch_team(const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  // rows per team: two only for 8-byte rows. The 16-byte instance with two rows (double, W = 2: one
  // LDG.128 per row and step) is miscompiled by ptxas 12.9 at -O3 — garbage gather addresses as soon
  // as the two rows' lengths differ (the same source is correct at -Xptxas -O1, with R = 1, and for
  // W = 1 / W = 4; scripts/team_probe.cu reproduces it) — so 16-byte rows take one row per team
  constexpr int TEAM = 8, R = W * sizeof(T) >= 16 ? 1 : 2;
  if (grid < 0) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, spmv_team_kernel<T, W, TEAM, R, EX>, block, smem);
    return nb;
  }
  spmv_team_kernel<T, W, TEAM, R, EX><<<grid, block, smem, st>>>(a);
  return (int)cudaGetLastError();
}

// narrow rows (s * esz <= 32 B): team-per-row kernel
template <typename T, int S>
constexpr bool use_team() { return S * (int)sizeof(T) <= 32; }

template <typename T, int S, bool FC>
int launch_spmm_t(const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  const bool ex = a.s == S && (sizeof(T) == 16 || S % 2 == 0);
  if constexpr (use_team<T, S>()) {
    if (a.sell_cs) {
      if (grid < 0) return launch_team<T, S, true>(a, grid, block, smem, st);
      if (ex) sell_kernel<T, S, true><<<grid, block, smem, st>>>(a);
      else sell_kernel<T, S, false><<<grid, block, smem, st>>>(a);
      return (int)cudaGetLastError();
    }
    if (a.team) {
      if (grid < 0 || ex) return launch_team<T, S, true>(a, grid, block, smem, st);
      return launch_team<T, S, false>(a, grid, block, smem, st);
    }
  }
  if (grid < 0 || ex) return launch_spmm_tx<T, S, FC, true>(a, grid, block, smem, st);
  return launch_spmm_tx<T, S, FC, false>(a, grid, block, smem, st);
}

template <typename T, int S, bool FC, int NI, bool EX, int R = upd_rows<T, NI>()>
int launch_upd_nix(const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(upd_kernel<T, S, FC, NI, R, EX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  if (grid < 0) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, upd_kernel<T, S, FC, NI, R, EX>, block, smem);
    return nb;
  }
  upd_kernel<T, S, FC, NI, R, EX><<<grid, block, smem, st>>>(a);
  return (int)cudaGetLastError();
}

template <typename T, int S, bool FC, int NI>
int launch_upd_ni(const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  // exact-width variant only for the scalar/diagonal (non-block) instances
  if constexpr (!FC) {
    const bool ex = a.s == S && (sizeof(T) == 16 || S % 2 == 0);
    // two-input updates with fused reductions: one row per lane group (the reduction
    // path's registers no longer spill; config 3's V~ update 1.243 -> 1.195 ms), two
    // rows without reductions (the plain axpy keeps its 96%)
    if constexpr (NI == 2 && upd_rows<T, 2>() == 2)
      if (grid >= 0 && ex && a.nred > 0) return launch_upd_nix<T, S, FC, NI, true, 1>(a, grid, block, smem, st);
    if (grid < 0 || ex) return launch_upd_nix<T, S, FC, NI, true>(a, grid, block, smem, st);
  }
  return launch_upd_nix<T, S, FC, NI, false>(a, grid, block, smem, st);
}

template <typename T, int S, bool FC>
int launch_upd_t(const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  const int nin = a.nin;
  if constexpr (FC) {  // block-method instances: two widths only (compile time)
    if (nin <= 2) return launch_upd_ni<T, S, FC, 2>(a, grid, block, smem, st);
    return launch_upd_ni<T, S, FC, MAX_IN>(a, grid, block, smem, st);
  } else {
    if (nin == 1) return launch_upd_ni<T, S, FC, 1>(a, grid, block, smem, st);
    if (nin == 2) return launch_upd_ni<T, S, FC, 2>(a, grid, block, smem, st);
    if (nin == 3 || nin == 4) return launch_upd_ni<T, S, FC, 4>(a, grid, block, smem, st);
    return launch_upd_ni<T, S, FC, MAX_IN>(a, grid, block, smem, st);
  }
}

template <typename T, int S>
int pick_spmm(bool full, const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  if constexpr (full_ok<T, S>()) {
    if (full) return launch_spmm_t<T, S, true>(a, grid, block, smem, st);
  } else {
    if (full) return (int)cudaErrorInvalidValue;
  }
  return launch_spmm_t<T, S, false>(a, grid, block, smem, st);
}
template <typename T, int S>
int pick_upd(bool full, const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  if constexpr (full_ok<T, S>()) {
    if (full) return launch_upd_t<T, S, true>(a, grid, block, smem, st);
  } else {
    if (full) return (int)cudaErrorInvalidValue;
  }
  return launch_upd_t<T, S, false>(a, grid, block, smem, st);
}


}  // namespace srk
