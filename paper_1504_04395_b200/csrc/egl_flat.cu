// eGl-BiCG (Alg. 4) on large operators: the two block updates of an iteration as
// lean flat kernels that also carry the economic variant's n-vectors (the shape of qmr_tail.cu).
//
//   egl_bicg_xr_kernel:  X <- X + alpha P ;  R <- R - alpha Q  with  sum(r̂^H R)  and  ||R||^2
//                        for the NEW shadow vector r̂ = r̂ - conj(alpha) q̂, formed per row in
//                        registers from its two operands and not stored (no thread reads an entry
//                        another one rewrites);
//   egl_bicg_p_kernel:   P <- R + beta P ; the thread that owns the first 16-byte unit of a row
//                        stores that r̂ and forms p̂ <- r̂ + conj(beta) p̂.
//
// Per iteration: 2 + 1 launches (kernels + finalisation) instead of 4 + 1, the same bytes; the
// per-element FMA order is upd_kernel's (out = 0; out = fma(src, coef, out) in source order), so
// iterates differ from the generic path only through the summation order of the two reductions.
#include <cuda_runtime.h>

#include "block_kernels.cuh"
#include "engine.h"

namespace srk {

template <typename T>
__device__ __forceinline__ T one_v() {
  if constexpr (Ar<T>::cplx) return mk(1.0, 0.0);
  else return 1.0;
}

template <typename T>
__global__ void __launch_bounds__(256, 4) egl_bicg_xr_kernel(EglFlatArgs a) {
  if (a.done && *a.done) return;
  constexpr int W = 128 / (int)sizeof(T);
  using L = Lay<T, W>;
  constexpr int E = L::EPL;
  __shared__ double rsm[16];
  const T zero = Ar<T>::zero(), one = one_v<T>();
  const T al = Ar<T>::ld(a.ws + a.off_alpha);
  const T nal = Ar<T>::sub(zero, al);
  const T ncal = Ar<T>::sub(zero, Ar<T>::conj(al));
  RedAcc<T, W, false> arho, ar2;
  red_zero(arho);
  red_zero(ar2);
  const long long stride = (long long)gridDim.x * 256;
  for (long long u = (long long)blockIdx.x * 256 + threadIdx.x; u < a.units; u += stride) {
    const long long row = a.sh >= 0 ? (u >> a.sh) : (u / a.upr);
    const double2 tx = reinterpret_cast<const double2*>(a.X)[u];
    const double2 tp = reinterpret_cast<const double2*>(a.P)[u];
    const double2 tr = reinterpret_cast<const double2*>(a.R)[u];
    const double2 tq = reinterpret_cast<const double2*>(a.Q)[u];
    const T rhv = reinterpret_cast<const T*>(a.rh)[row];
    const T qhv = reinterpret_cast<const T*>(a.qh)[row];
    T x[E], p[E], r[E], q[E], xn[E], rn[E];
    if constexpr (E == 2) {
      x[0] = tx.x; x[1] = tx.y; p[0] = tp.x; p[1] = tp.y; r[0] = tr.x; r[1] = tr.y; q[0] = tq.x; q[1] = tq.y;
    } else {
      x[0] = tx; p[0] = tp; r[0] = tr; q[0] = tq;
    }
    const T rhn = Ar<T>::fma(qhv, ncal, Ar<T>::fma(rhv, one, zero));
#pragma unroll
    for (int e = 0; e < E; ++e) {
      xn[e] = Ar<T>::fma(p[e], al, Ar<T>::fma(x[e], one, zero));
      rn[e] = Ar<T>::fma(q[e], nal, Ar<T>::fma(r[e], one, zero));
      arho.v[e] = Ar<T>::cfma(rhn, rn[e], arho.v[e]);
      ar2.v[e] = Ar<T>::cfma(rn[e], rn[e], ar2.v[e]);
    }
    if constexpr (E == 2) {
      reinterpret_cast<double2*>(a.X)[u] = make_double2(xn[0], xn[1]);
      reinterpret_cast<double2*>(a.R)[u] = make_double2(rn[0], rn[1]);
    } else {
      reinterpret_cast<double2*>(a.X)[u] = xn[0];
      reinterpret_cast<double2*>(a.R)[u] = rn[0];
    }
  }
  __syncwarp();
  red_flush<T, W, RED_SUMVEC, false>(arho, a.partials, a.pstride, 0, W, rsm);
  red_flush<T, W, RED_NORM2, false>(ar2, a.partials, a.pstride, Ar<T>::ND, W, rsm);
}

template <typename T>
__global__ void __launch_bounds__(256, 4) egl_bicg_p_kernel(EglFlatArgs a) {
  if (a.done && *a.done) return;
  constexpr int E = Lay<T, 128 / (int)sizeof(T)>::EPL;
  const T zero = Ar<T>::zero(), one = one_v<T>();
  const T be = Ar<T>::ld(a.ws + a.off_beta);
  const T cbe = Ar<T>::conj(be);
  const T ncal = Ar<T>::sub(zero, Ar<T>::conj(Ar<T>::ld(a.ws + a.off_alpha)));
  const long long stride = (long long)gridDim.x * 256;
  for (long long u = (long long)blockIdx.x * 256 + threadIdx.x; u < a.units; u += stride) {
    // the row's n-vector entries are requested with the block loads (by the thread that owns the
    // row's first unit)
    const long long row = a.sh >= 0 ? (u >> a.sh) : (u / a.upr);
    const bool lead = u == (a.sh >= 0 ? (row << a.sh) : row * a.upr);
    T ro = zero, qo = zero, po = zero;
    if (lead) {
      ro = reinterpret_cast<const T*>(a.rh)[row];
      qo = reinterpret_cast<const T*>(a.qh)[row];
      po = reinterpret_cast<const T*>(a.ph)[row];
    }
    const double2 tr = reinterpret_cast<const double2*>(a.R)[u];
    const double2 tp = reinterpret_cast<const double2*>(a.P)[u];
    if constexpr (E == 2) {
      reinterpret_cast<double2*>(a.P)[u] = make_double2(Ar<T>::fma(tp.x, be, Ar<T>::fma(tr.x, one, zero)),
                                                         Ar<T>::fma(tp.y, be, Ar<T>::fma(tr.y, one, zero)));
    } else {
      reinterpret_cast<double2*>(a.P)[u] = Ar<T>::fma(tp, be, Ar<T>::fma(tr, one, zero));
    }
    if (lead) {
      const T rhn = Ar<T>::fma(qo, ncal, Ar<T>::fma(ro, one, zero));
      reinterpret_cast<T*>(a.rh)[row] = rhn;
      reinterpret_cast<T*>(a.ph)[row] = Ar<T>::fma(po, cbe, Ar<T>::fma(rhn, one, zero));
    }
  }
}

// which: 0 = the (X, R) kernel, 1 = the P kernel; grid < 0: resident CTAs per SM
int launch_egl_flat(int which, bool cplx, const EglFlatArgs& a, int grid, cudaStream_t st) {
  if (grid < 0) {
    int nb = 0;
    if (which == 0) {
      if (cplx) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, egl_bicg_xr_kernel<double2>, 256, 0);
      else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, egl_bicg_xr_kernel<double>, 256, 0);
    } else {
      if (cplx) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, egl_bicg_p_kernel<double2>, 256, 0);
      else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, egl_bicg_p_kernel<double>, 256, 0);
    }
    return nb;
  }
  if (which == 0) {
    if (cplx) egl_bicg_xr_kernel<double2><<<grid, 256, 0, st>>>(a);
    else egl_bicg_xr_kernel<double><<<grid, 256, 0, st>>>(a);
  } else {
    if (cplx) egl_bicg_p_kernel<double2><<<grid, 256, 0, st>>>(a);
    else egl_bicg_p_kernel<double><<<grid, 256, 0, st>>>(a);
  }
  return (int)cudaGetLastError();
}

}  // namespace srk
