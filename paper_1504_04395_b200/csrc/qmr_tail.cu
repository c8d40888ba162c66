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
  T nbx = zero, ix = zero, nc2 = zero;
  if (a.upr > 0) {
    nbx = Ar<T>::sub(zero, Ar<T>::ld(a.ws + a.off_bx));
    ix = Ar<T>::ld(a.ws + a.off_invxi);
    nc2 = Ar<T>::sub(zero, Ar<T>::ld(a.ws + a.off_c2));
  }
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
    // eGl: the thread that owns the first unit of a row also carries the row's n-vector entries;
    // their loads are issued with the block loads
    bool lead = false;
    long long row = 0;
    T wo = zero, ah = zero, qo = zero;
    if (a.upr > 0) {
      row = a.sh >= 0 ? (u >> a.sh) : (u / a.upr);
      lead = u == (a.sh >= 0 ? (row << a.sh) : row * a.upr);
      if (lead) {
        wo = reinterpret_cast<const T*>(a.Wt)[row];
        ah = reinterpret_cast<const T*>(a.AHQ)[row];
        qo = reinterpret_cast<const T*>(a.Qv)[row];
      }
    }
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
    // eGl: the left Lanczos vectors of the next iteration, by the thread that owns the first unit of
    // a row (nobody else touches them): w̃ <- A^H q - (conj(beta)/xi) w̃ (deferred from qmr_vt_kernel,
    // which only reduced it) and q <- w̃/xi' - c2' q
    if (lead) {
      const T wn = Ar<T>::fma(wo, nbx, Ar<T>::fma(ah, one, zero));
      reinterpret_cast<T*>(a.Wt)[row] = wn;
      reinterpret_cast<T*>(a.Qv)[row] = Ar<T>::fma(qo, nc2, Ar<T>::fma(wn, ix, zero));
    }
  }
  __syncwarp();
  red_flush<T, W, RED_NORM2, false>(acc, a.partials, a.pstride, a.poff, W, rsm);
}

// eGl-QMR: Ṽ <- P~ - (beta/rho) Ṽ with ||Ṽ||^2 and sum(w̃^H Ṽ) for the NEW left vector
// w̃ = A^H q - (conj(beta)/xi) w̃, formed per row in registers from its two operands and reduced
// (||w̃||^2, by the first unit of each row) but not stored: the fused tail stores it (see above),
// so no thread reads an entry another one rewrites. One launch and one finalisation instead of
// the n-vector update, the block update and their two finalisations; flat 16-byte units as above.
template <typename T>
__global__ void __launch_bounds__(256, 4) qmr_vt_kernel(QmrVtArgs a) {
  if (a.done && *a.done) return;
  constexpr int W = 128 / (int)sizeof(T);
  using L = Lay<T, W>;
  constexpr int E = L::EPL;
  __shared__ double rsm[16];
  const T zero = Ar<T>::zero();
  T one;
  if constexpr (Ar<T>::cplx) one = mk(1.0, 0.0); else one = 1.0;
  const T nbr = Ar<T>::sub(zero, Ar<T>::ld(a.ws + a.off_br));
  const T nbx = Ar<T>::sub(zero, Ar<T>::ld(a.ws + a.off_bx));
  RedAcc<T, W, false> arho, ak1, axi;
  red_zero(arho);
  red_zero(ak1);
  red_zero(axi);
  const long long stride = (long long)gridDim.x * 256;
  for (long long u = (long long)blockIdx.x * 256 + threadIdx.x; u < a.units; u += stride) {
    const long long row = a.sh >= 0 ? (u >> a.sh) : (u / a.upr);
    const double2 tp = reinterpret_cast<const double2*>(a.Pt)[u];
    const double2 tv = reinterpret_cast<const double2*>(a.Vt)[u];
    const T ah = reinterpret_cast<const T*>(a.AHQ)[row];
    const T wo = reinterpret_cast<const T*>(a.Wt)[row];
    T pt[E], vt[E], vn[E];
    if constexpr (E == 2) { pt[0] = tp.x; pt[1] = tp.y; vt[0] = tv.x; vt[1] = tv.y; } else { pt[0] = tp; vt[0] = tv; }
    const T wn = Ar<T>::fma(wo, nbx, Ar<T>::fma(ah, one, zero));
#pragma unroll
    for (int e = 0; e < E; ++e) {
      vn[e] = Ar<T>::fma(vt[e], nbr, Ar<T>::fma(pt[e], one, zero));
      arho.v[e] = Ar<T>::cfma(vn[e], vn[e], arho.v[e]);
      ak1.v[e] = Ar<T>::cfma(wn, vn[e], ak1.v[e]);
    }
    if constexpr (E == 2) reinterpret_cast<double2*>(a.Vt)[u] = make_double2(vn[0], vn[1]);
    else reinterpret_cast<double2*>(a.Vt)[u] = vn[0];
    if (u == (a.sh >= 0 ? (row << a.sh) : row * a.upr)) axi.v[0] = Ar<T>::cfma(wn, wn, axi.v[0]);
  }
  __syncwarp();
  red_flush<T, W, RED_NORM2, false>(arho, a.partials, a.pstride, 0, W, rsm);
  red_flush<T, W, RED_SUMVEC, false>(ak1, a.partials, a.pstride, 1, W, rsm);
  red_flush<T, W, RED_NORM2, false>(axi, a.partials, a.pstride, 1 + Ar<T>::ND, W, rsm);
}

int launch_qmr_vt(bool cplx, const QmrVtArgs& a, int grid, cudaStream_t st) {
  if (grid < 0) {
    int nb = 0;
    if (cplx) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, qmr_vt_kernel<double2>, 256, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, qmr_vt_kernel<double>, 256, 0);
    return nb;
  }
  if (cplx) qmr_vt_kernel<double2><<<grid, 256, 0, st>>>(a);
  else qmr_vt_kernel<double><<<grid, 256, 0, st>>>(a);
  return (int)cudaGetLastError();
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
