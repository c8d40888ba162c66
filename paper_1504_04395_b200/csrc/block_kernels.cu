// block_kernels.cu — the hot-path kernels over row-interleaved n x s blocks.
//
//  * spmm_kernel   Q = A P, CSR, one lane group per row: each nonzero a_ij is
//                  read once and applied to the s contiguous values of P row j
//                  (SURVEY §8(a) a1/a2),
//                  with the s x s / trace / sum / diag Gram partials fused into
//                  the epilogue (P:155-158, 178, 192-195,
//                  243-249, 443-447).
//  * upd_kernel    fused multi-output block updates out = sum_t src_t*coef_t with
//                  scalar (Gl/eGl), diagonal (Li) or s x s (Bl, "BLAS3 GEMM"
//                  P:290-297) coefficients read from device memory, plus fused
//                  reductions.
//  * fin_kernel    fixed-order second-stage reduction of per-CTA partials: no
//                  floating-point atomics, so results are bitwise reproducible.
#include "kernels.cuh"

namespace srk {

// Accumulators for one reduction held by one lane (capacity S).
template <typename T, int S, bool FC>
struct RedAcc {
  using L = Lay<T, S>;
  // FULL (FC) needs S x EPL values; the other modes use the first EPL.
  static constexpr int N = FC ? S * L::EPL : L::EPL;
  T v[N];
  double r[L::EPL];  // NORM2 / COLNORM2
};

template <typename T, int S, bool FC>
__device__ __forceinline__ void red_zero(RedAcc<T, S, FC>& a) {
#pragma unroll
  for (int i = 0; i < RedAcc<T, S, FC>::N; ++i) a.v[i] = Ar<T>::zero();
#pragma unroll
  for (int i = 0; i < Lay<T, S>::EPL; ++i) a.r[i] = 0.0;
}

// Accumulate one row's contribution. x: lane elements of the X row; y: lane
// elements of the Y row (block modes) or yv the vector entry (SUMVEC).
template <typename T, int S, int MODE, bool FC>
__device__ __forceinline__ void red_row(RedAcc<T, S, FC>& a, const T (&x)[Lay<T, S>::EPL], const T (&y)[Lay<T, S>::EPL],
                                        T yv, int base, int s, unsigned gmask) {
  using L = Lay<T, S>;
  if constexpr (MODE == RED_NORM2 || MODE == RED_COLNORM2) {
#pragma unroll
    for (int e = 0; e < L::EPL; ++e) a.r[e] += Ar<T>::abs2(x[e]);
  } else if constexpr (MODE == RED_DIAG || MODE == RED_TRACE) {
#pragma unroll
    for (int e = 0; e < L::EPL; ++e) a.v[e] = Ar<T>::cfma(y[e], x[e], a.v[e]);
  } else if constexpr (MODE == RED_SUMVEC) {
#pragma unroll
    for (int e = 0; e < L::EPL; ++e) a.v[e] = Ar<T>::cfma(yv, x[e], a.v[e]);
  } else if constexpr (MODE == RED_FULL && FC) {
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

// CTA-level reduction of one RedAcc into partials[blockIdx.x*pstride + poff ...].
// Order: xor-butterfly over lane groups, then warps summed in index order by
// thread 0..len-1 — fixed for a given launch configuration.
template <typename T, int S, int MODE, bool FC>
__device__ void red_flush(RedAcc<T, S, FC>& a, double* __restrict__ partials, int pstride, int poff, int s,
                          double* smem /* >= nwarps * len doubles */) {
  using L = Lay<T, S>;
  constexpr int ND = Ar<T>::ND;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int g = lane % L::G;
  // 1) sum over the lane groups of this warp (lanes with equal g hold the same entries)
#pragma unroll
  for (int m = L::G; m < 32; m <<= 1) {
#pragma unroll
    for (int i = 0; i < RedAcc<T, S, FC>::N; ++i) a.v[i] = Ar<T>::add(a.v[i], Ar<T>::shfl_xor(a.v[i], m));
#pragma unroll
    for (int i = 0; i < L::EPL; ++i) a.r[i] += __shfl_xor_sync(0xffffffffu, a.r[i], m);
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
      rs += a.r[e];
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
          if constexpr (MODE == RED_COLNORM2) w[c] = a.r[e];
          else Ar<T>::st(w + c * ND, a.v[e]);
        }
      }
    }
  } else if constexpr (MODE == RED_FULL && FC) {
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
  __syncthreads();
  // 3) sum the warps' slices in warp order
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < nwarps; ++q) acc += smem[q * len + j];
    partials[(size_t)blockIdx.x * pstride + poff + j] = acc;
  }
  __syncthreads();
}

template <typename T, int S, bool FC>
__device__ __forceinline__ void red_dispatch_row(int mode, RedAcc<T, S, FC>& a, const T (&x)[Lay<T, S>::EPL],
                                                 const T (&y)[Lay<T, S>::EPL], T yv, int base, int s,
                                                 unsigned gmask) {
  switch (mode) {
    case RED_NORM2: red_row<T, S, RED_NORM2, FC>(a, x, y, yv, base, s, gmask); break;
    case RED_COLNORM2: red_row<T, S, RED_COLNORM2, FC>(a, x, y, yv, base, s, gmask); break;
    case RED_DIAG: red_row<T, S, RED_DIAG, FC>(a, x, y, yv, base, s, gmask); break;
    case RED_TRACE: red_row<T, S, RED_TRACE, FC>(a, x, y, yv, base, s, gmask); break;
    case RED_SUMVEC: red_row<T, S, RED_SUMVEC, FC>(a, x, y, yv, base, s, gmask); break;
    case RED_FULL: red_row<T, S, RED_FULL, FC>(a, x, y, yv, base, s, gmask); break;
    default: break;
  }
}

template <typename T, int S, bool FC>
__device__ void red_dispatch_flush(int mode, RedAcc<T, S, FC>& a, double* partials, int pstride, int poff, int s,
                                   double* smem) {
  switch (mode) {
    case RED_NORM2: red_flush<T, S, RED_NORM2, FC>(a, partials, pstride, poff, s, smem); break;
    case RED_COLNORM2: red_flush<T, S, RED_COLNORM2, FC>(a, partials, pstride, poff, s, smem); break;
    case RED_DIAG: red_flush<T, S, RED_DIAG, FC>(a, partials, pstride, poff, s, smem); break;
    case RED_TRACE: red_flush<T, S, RED_TRACE, FC>(a, partials, pstride, poff, s, smem); break;
    case RED_SUMVEC: red_flush<T, S, RED_SUMVEC, FC>(a, partials, pstride, poff, s, smem); break;
    case RED_FULL: red_flush<T, S, RED_FULL, FC>(a, partials, pstride, poff, s, smem); break;
    default: break;
  }
}

// ============================================================================
// SpMM: Q = A P
// ============================================================================
template <typename T, int S, bool FC>
__global__ void __launch_bounds__(256) spmm_kernel(SpmmArgs a) {
  if (a.done && *a.done) return;
  using L = Lay<T, S>;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int g = lane % L::G;
  const int base = lane - g;
  const unsigned gmask = (L::G == 32) ? 0xffffffffu : (((1u << L::G) - 1u) << base);
  const long long groups_per_cta = (blockDim.x / 32) * L::RPW;
  const long long grp0 = (long long)blockIdx.x * groups_per_cta + (threadIdx.x >> 5) * L::RPW + lane / L::G;
  const long long gstride = (long long)gridDim.x * groups_per_cta;
  const T* __restrict__ P = reinterpret_cast<const T*>(a.P);
  const T* __restrict__ val = reinterpret_cast<const T*>(a.val);
  T* __restrict__ Q = reinterpret_cast<T*>(a.Q);
  const int s = a.s;

  RedAcc<T, S, FC> acc0, acc1;
  red_zero(acc0);
  red_zero(acc1);

  for (long long row = grp0; row < a.n; row += gstride) {
    T q[L::EPL];
#pragma unroll
    for (int e = 0; e < L::EPL; ++e) q[e] = Ar<T>::zero();
    const int beg = __ldg(a.row_ptr + row), end = __ldg(a.row_ptr + row + 1);
    for (int j0 = beg; j0 < end; j0 += L::G) {
      // cooperative, coalesced fetch of up to G (col, val) pairs, then broadcast
      int cj = 0;
      T vj = Ar<T>::zero();
      if (j0 + g < end) {
        cj = __ldcs(a.col_idx + j0 + g);   // streamed once: evict-first, keep L2 for P
        vj = __ldcs(val + j0 + g);
      }
      const int cnt = min(L::G, end - j0);
#pragma unroll 4
      for (int t = 0; t < cnt; ++t) {
        const int c = __shfl_sync(gmask, cj, base + t);
        const T v = Ar<T>::shfl(vj, base + t, gmask);
        T p[L::EPL];
        row_load<T, S>(P + (size_t)c * s, g, s, a.vec, p);
#pragma unroll
        for (int e = 0; e < L::EPL; ++e) q[e] = Ar<T>::fma(v, p[e], q[e]);
      }
    }
    row_store<T, S>(Q + (size_t)row * s, g, s, a.vec, q);
    // fused epilogue: reductions with X = Q
    for (int r = 0; r < a.nred; ++r) {
      const Red& rd = a.red[r];
      T y[L::EPL];
      T yv = Ar<T>::zero();
      if (rd.mode == RED_SUMVEC) {
        yv = reinterpret_cast<const T*>(rd.yext)[row];
#pragma unroll
        for (int e = 0; e < L::EPL; ++e) y[e] = Ar<T>::zero();
      } else if (rd.mode == RED_NORM2 || rd.mode == RED_COLNORM2) {
#pragma unroll
        for (int e = 0; e < L::EPL; ++e) y[e] = Ar<T>::zero();
      } else {
        row_load<T, S>(reinterpret_cast<const T*>(rd.yext) + (size_t)row * s, g, s, a.vec, y);
      }
      if (r == 0) red_dispatch_row<T, S, FC>(rd.mode, acc0, q, y, yv, base, s, gmask);
      else red_dispatch_row<T, S, FC>(rd.mode, acc1, q, y, yv, base, s, gmask);
    }
  }
  __syncwarp();
  if (a.nred > 0) red_dispatch_flush<T, S, FC>(a.red[0].mode, acc0, a.partials, a.pstride, a.red[0].poff, s, smem);
  if (a.nred > 1) red_dispatch_flush<T, S, FC>(a.red[1].mode, acc1, a.partials, a.pstride, a.red[1].poff, s, smem);
}

// ============================================================================
// Fused block update / Gram
// ============================================================================
template <typename T, int S, bool FC>
__global__ void __launch_bounds__(256) upd_kernel(UpdArgs a) {
  if (a.done && *a.done) return;
  using L = Lay<T, S>;
  constexpr int ND = Ar<T>::ND;
  extern __shared__ double smem[];
  const int s = a.s;
  // ---- stage coefficients into shared memory (neg/conj/herm applied once)
  // layout: per (out, term) slot of S*S values of T
  T* cs = reinterpret_cast<T*>(smem);
  for (int o = 0; o < a.nout; ++o)
    for (int t = 0; t < a.out[o].nterm; ++t) {
      const Coef& cf = a.out[o].t[t].c;
      T* dst = cs + a.cslot[o][t];
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

  RedAcc<T, S, FC> acc0, acc1;
  RedAcc<T, S, false> acc2;
  red_zero(acc0);
  red_zero(acc1);
  red_zero(acc2);

  for (long long row = grp0; row < a.n; row += gstride) {
    T xin[MAX_IN][L::EPL];
    T xo[MAX_OUT][L::EPL];
#pragma unroll
    for (int b = 0; b < MAX_IN; ++b)
      if (b < a.nin) row_load<T, S>(reinterpret_cast<const T*>(a.in[b]) + (size_t)row * s, g, s, a.vec, xin[b]);
#pragma unroll
    for (int o = 0; o < MAX_OUT; ++o) {
      if (o < a.nout) {
#pragma unroll
        for (int e = 0; e < L::EPL; ++e) xo[o][e] = Ar<T>::zero();
        for (int t = 0; t < a.out[o].nterm; ++t) {
          const Term& tm = a.out[o].t[t];
          // resolve the source row held in registers
          T xs[L::EPL];
#pragma unroll
          for (int e = 0; e < L::EPL; ++e) {
            xs[e] = Ar<T>::zero();
#pragma unroll
            for (int b = 0; b < MAX_IN; ++b)
              if (tm.src == b) xs[e] = xin[b][e];
#pragma unroll
            for (int b = 0; b < MAX_OUT; ++b)
              if (tm.src == SRC_OUT + b) xs[e] = xo[b][e];
          }
          const T* cf = cs + a.cslot[o][t];
          if (tm.c.kind == CK_FULL) {
#pragma unroll
            for (int k = 0; k < S; ++k) {
              if (k < s) {
                const T xk = row_get<T, S>(xs, base, k, gmask);
#pragma unroll
                for (int e = 0; e < L::EPL; ++e) xo[o][e] = Ar<T>::fma(xk, cf[k * L::PW + L::col(g, e)], xo[o][e]);
              }
            }
          } else if (tm.c.kind == CK_DIAG) {
#pragma unroll
            for (int e = 0; e < L::EPL; ++e) xo[o][e] = Ar<T>::fma(xs[e], cf[L::col(g, e)], xo[o][e]);
          } else {
            const T c0 = cf[0];
#pragma unroll
            for (int e = 0; e < L::EPL; ++e) xo[o][e] = Ar<T>::fma(xs[e], c0, xo[o][e]);
          }
        }
        if (a.out[o].ptr) row_store<T, S>(reinterpret_cast<T*>(a.out[o].ptr) + (size_t)row * s, g, s, a.vec, xo[o]);
      }
    }
    // reductions
#pragma unroll
    for (int r = 0; r < MAX_RED; ++r) {
      if (r < a.nred) {
        const Red& rd = a.red[r];
        T x[L::EPL], y[L::EPL];
        T yv = Ar<T>::zero();
#pragma unroll
        for (int e = 0; e < L::EPL; ++e) {
          x[e] = Ar<T>::zero();
          y[e] = Ar<T>::zero();
#pragma unroll
          for (int b = 0; b < MAX_IN; ++b) {
            if (rd.xsrc == b) x[e] = xin[b][e];
            if (rd.ysrc == b) y[e] = xin[b][e];
          }
#pragma unroll
          for (int b = 0; b < MAX_OUT; ++b) {
            if (rd.xsrc == SRC_OUT + b) x[e] = xo[b][e];
            if (rd.ysrc == SRC_OUT + b) y[e] = xo[b][e];
          }
        }
        if (rd.ysrc < 0 && rd.yext) {
          if (rd.mode == RED_SUMVEC) yv = reinterpret_cast<const T*>(rd.yext)[row];
          else row_load<T, S>(reinterpret_cast<const T*>(rd.yext) + (size_t)row * s, g, s, a.vec, y);
        }
        if (r == 0) red_dispatch_row<T, S, FC>(rd.mode, acc0, x, y, yv, base, s, gmask);
        else if (r == 1) red_dispatch_row<T, S, FC>(rd.mode, acc1, x, y, yv, base, s, gmask);
        else red_dispatch_row<T, S, false>(rd.mode, acc2, x, y, yv, base, s, gmask);
      }
    }
  }
  __syncwarp();
  if (a.nred > 0) red_dispatch_flush<T, S, FC>(a.red[0].mode, acc0, a.partials, a.pstride, a.red[0].poff, s, rsm);
  if (a.nred > 1) red_dispatch_flush<T, S, FC>(a.red[1].mode, acc1, a.partials, a.pstride, a.red[1].poff, s, rsm);
  if (a.nred > 2) red_dispatch_flush<T, S, false>(a.red[2].mode, acc2, a.partials, a.pstride, a.red[2].poff, s, rsm);
}

// ============================================================================
// Deterministic second stage: ws[woff + j] = sum_b partials[b*pstride + poff + j]
// One warp per output value; lanes stride over CTAs; fixed xor tree.
// ============================================================================
__global__ void fin_kernel(FinArgs a) {
  if (a.done && *a.done) return;
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int j = wid;
  for (int q = 0; q < a.nseg; ++q) {
    if (j < a.seg[q].len) {
      double acc = 0.0;
      for (int b = lane; b < a.nblk; b += 32) acc += a.partials[(size_t)b * a.pstride + a.seg[q].poff + j];
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
      if (lane == 0) a.ws[a.seg[q].woff + j] = acc;
      return;
    }
    j -= a.seg[q].len;
  }
}

// ============================================================================
// Host-side launchers (explicit instantiation per capacity S)
// ============================================================================
// grid < 0: return the number of resident CTAs per SM instead of launching
template <typename T, int S, bool FC>
static int launch_spmm_t(const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(spmm_kernel<T, S, FC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  if (grid < 0) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, spmm_kernel<T, S, FC>, block, smem);
    return nb;
  }
  spmm_kernel<T, S, FC><<<grid, block, smem, st>>>(a);
  return (int)cudaGetLastError();
}
template <typename T, int S, bool FC>
static int launch_upd_t(const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(upd_kernel<T, S, FC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  if (grid < 0) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, upd_kernel<T, S, FC>, block, smem);
    return nb;
  }
  upd_kernel<T, S, FC><<<grid, block, smem, st>>>(a);
  return (int)cudaGetLastError();
}
// FULL Gram epilogues are instantiated only where the accumulators fit in registers
template <typename T, int S> constexpr bool full_ok() { return (sizeof(T) == 8) ? (S <= 32) : (S <= 16); }

#define SRK_CAPS(X) X(1) X(2) X(4) X(8) X(12) X(16) X(32) X(64)

int cap_for(int s) {
  const int caps[] = {1, 2, 4, 8, 12, 16, 32, 64};
  for (int c : caps)
    if (s <= c) return c;
  return -1;
}

// rows handled by one 256-thread CTA per grid-stride step
int rows_per_cta(int cap, bool cplx) {
  int esz = cplx ? 16 : 8;
  int epc = (esz == 16) ? 1 : ((cap % 2 == 0) ? 2 : 1);
  int nch = (cap + epc - 1) / epc;
  int G = pow2ceil(nch);
  if (G > 32) G = 32;
  return 8 * (32 / G);
}

template <typename T, int S>
static int pick_spmm(bool full, const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  if constexpr (full_ok<T, S>()) {
    if (full) return launch_spmm_t<T, S, true>(a, grid, block, smem, st);
  } else {
    if (full) return (int)cudaErrorInvalidValue;
  }
  return launch_spmm_t<T, S, false>(a, grid, block, smem, st);
}
template <typename T, int S>
static int pick_upd(bool full, const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  if constexpr (full_ok<T, S>()) {
    if (full) return launch_upd_t<T, S, true>(a, grid, block, smem, st);
  } else {
    if (full) return (int)cudaErrorInvalidValue;
  }
  return launch_upd_t<T, S, false>(a, grid, block, smem, st);
}

int launch_spmm(bool cplx, int cap, bool full, const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
#define CASE(C)                                                                  \
  case C:                                                                        \
    return cplx ? pick_spmm<double2, C>(full, a, grid, block, smem, st)         \
                : pick_spmm<double, C>(full, a, grid, block, smem, st);
  switch (cap) { SRK_CAPS(CASE) }
#undef CASE
  return (int)cudaErrorInvalidValue;
}

int launch_upd(bool cplx, int cap, bool full, const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
#define CASE(C)                                                                 \
  case C:                                                                       \
    return cplx ? pick_upd<double2, C>(full, a, grid, block, smem, st)         \
                : pick_upd<double, C>(full, a, grid, block, smem, st);
  switch (cap) { SRK_CAPS(CASE) }
#undef CASE
  return (int)cudaErrorInvalidValue;
}

bool full_supported(bool cplx, int cap) { return cplx ? cap <= 16 : cap <= 32; }

int padded_width(int cap, bool cplx) {
  const int esz = cplx ? 16 : 8;
  const int epc = (esz == 16) ? 1 : ((cap % 2 == 0) ? 2 : 1);
  const int nch = (cap + epc - 1) / epc;
  int G = pow2ceil(nch);
  if (G > 32) G = 32;
  const int cpl = (nch + G - 1) / G;
  return G * epc * cpl;
}

int launch_fin(const FinArgs& a, cudaStream_t st) {
  int total = 0;
  for (int q = 0; q < a.nseg; ++q) total += a.seg[q].len;
  if (total == 0) return 0;
  const int warps_per_cta = 8;
  int grid = (total + warps_per_cta - 1) / warps_per_cta;
  fin_kernel<<<grid, warps_per_cta * 32, 0, st>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace srk
