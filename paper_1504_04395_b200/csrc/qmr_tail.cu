// Gl / eGl-QMR: the last update of iteration k fused with the first update of
// iteration k+1.
//
//   D <- eta P + f D ;  S <- eta P~ + f S ;  X <- X + D ;  R <- R - S ;  ||R||^2   (iteration k)
//   P <- Ṽ/rho' - c1' P                                                        (iteration k+1)
//
// The second line needs only rho' = ||Ṽ_{k+1}||, xi', delta' = <Ṽ, W̃>/(rho' xi') and this
// iteration's eps, all known once Ṽ_{k+1} has been formed — before theta, gamma, eta — so
// coefficient phase 4 also writes 1/rho' and c1' (SL_INVRHO_N, SL_C1_N; the same arithmetic
// as next iteration's phases 1-2, which still run and own the breakdown tests). P is
// read once for D and for its own successor: 7 blocks in, 5 out = 12 block passes
// against 10 + 3 for the two separate updates (the iteration: 17 instead of 18).
//
// All coefficients are scalars, so the n x s blocks are flat arrays: one 16-byte
// unit per thread and step, the seven loads of a step issued before any arithmetic,
// one wave of 256-thread CTAs striding the array (the shape of upd_kernel's NI = 6
// instance, whose FMA order per element and whose reduction order this kernel keeps:
// iterates are bitwise those of the separate updates).
#include <cuda_runtime.h>

#include <atomic>

#include "block_kernels.cuh"
#include "engine.h"

namespace srk {

template <typename T>
__global__ void __launch_bounds__(256, sizeof(T) == 16 ? 3 : 4) qmr_tail_kernel(QmrTailArgs a) {
  if (a.done && *a.done) return;
  constexpr int W = 128 / (int)sizeof(T);  // 128-byte rows: the lane layout of upd_kernel at s = 16 (real) / 8 (complex)
  using L = Lay<T, W>;
  constexpr int E = L::EPL;  // 2 reals or 1 complex value per 16-byte unit
  __shared__ double rsm[8];
  const T zero = Ar<T>::zero();
  T one;
  if constexpr (Ar<T>::cplx) one = mk(1.0, 0.0); else one = 1.0;
  const T neg1 = Ar<T>::sub(zero, one);
  const T eta = Ar<T>::ld(a.ws + a.off_eta);
  const T f = Ar<T>::ld(a.ws + a.off_f);
  const T ir = Ar<T>::ld(a.ws + a.off_invrho);
  const T nc1 = Ar<T>::sub(zero, Ar<T>::ld(a.ws + a.off_c1));
  RedAcc<T, W, false> acc;
  red_zero(acc);
  auto ld = [&](const void* base, long long u, T (&v)[E]) {
    const double2 t = reinterpret_cast<const double2*>(base)[u];
    if constexpr (E == 2) { v[0] = t.x; v[1] = t.y; } else { v[0] = t; }
  };
  auto st = [&](void* base, long long u, const T (&v)[E]) {
    if constexpr (E == 2) reinterpret_cast<double2*>(base)[u] = make_double2(v[0], v[1]);
    else reinterpret_cast<double2*>(base)[u] = v[0];
  };
  const long long stride = (long long)gridDim.x * 256;
  for (long long u = (long long)blockIdx.x * 256 + threadIdx.x; u < a.units; u += stride) {
    T p[E], d[E], pt[E], s[E], x[E], r[E], vt[E];
    ld(a.P, u, p);
    ld(a.D, u, d);
    ld(a.Pt, u, pt);
    ld(a.S, u, s);
    ld(a.X, u, x);
    ld(a.R, u, r);
    ld(a.Vt, u, vt);
    T dn[E], sn[E], xn[E], rn[E], pn[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      dn[e] = Ar<T>::fma(d[e], f, Ar<T>::fma(p[e], eta, zero));
      sn[e] = Ar<T>::fma(s[e], f, Ar<T>::fma(pt[e], eta, zero));
      xn[e] = Ar<T>::fma(dn[e], one, Ar<T>::fma(x[e], one, zero));
      rn[e] = Ar<T>::fma(sn[e], neg1, Ar<T>::fma(r[e], one, zero));
      pn[e] = Ar<T>::fma(p[e], nc1, Ar<T>::fma(vt[e], ir, zero));
    }
    st(a.D, u, dn);
    st(a.S, u, sn);
    st(a.X, u, xn);
    st(a.R, u, rn);
    st(a.P, u, pn);
    red_acc<T, W, false>(acc, rn, rn);
  }
  __syncwarp();
  red_flush<T, W, RED_NORM2, false>(acc, a.partials, a.pstride, a.poff, W, rsm);
}

// grid < 0: resident CTAs per SM of this instance
int launch_qmr_tail(bool cplx, const QmrTailArgs& a, int grid, cudaStream_t st) {
  if (grid < 0) {
    int nb = 0;
    if (cplx) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, qmr_tail_kernel<double2>, 256, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, qmr_tail_kernel<double>, 256, 0);
    return nb;
  }
  if (cplx) qmr_tail_kernel<double2><<<grid, 256, 0, st>>>(a);
  else qmr_tail_kernel<double><<<grid, 256, 0, st>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace srk
