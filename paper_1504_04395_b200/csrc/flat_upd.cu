// Block updates whose coefficients are all scalars (the global methods) do not
// depend on the row structure of the n x s blocks: they are flat array updates. This file
// holds them as compile-time plans of one lean kernel — one 16-byte unit per thread and step,
// every load of a step issued before any arithmetic, coefficients in registers, one wave of
// 256-thread CTAs striding the array — the shape of qmr_tail.cu's kernels (97-99% of the
// measured HBM peak against 81-85% for the same updates on the generic upd_kernel, whose
// term table, coefficient staging and reduction dispatch are decoded at run time).
//
// A plan states its inputs, outputs, coefficients (offsets into the coefficient workspace, with
// an optional negation), the per-element arithmetic in the FMA order of upd_kernel (out = 0;
// out = fma(src, coef, out) over the sources in index order — iterates differ from the generic
// path only through the summation order of the reductions) and its reductions
// (NORM2: sum |x|^2; TRACE: sum conj(y) x).
//
// Plans: Gl-BiCGStab (SURVEY App. A.4 with scalar coefficients; the method of config 4 and
// config 3's second method): S = R - alpha V with ||S||^2; (X, R) = (X + alpha P + omega S,
// S - omega T) with <R, R~> and ||R||^2; P = R + beta P - beta omega V. Gl-BiCG (Alg. 2): the (X, R, R^)
// update with <R, R^> and ||R||^2, and the (P, P^) update. Gl-QMR: the (V~, W~) update with its three
// reductions.
#include <cuda_runtime.h>

#include "block_kernels.cuh"
#include "engine.h"

namespace srk {

template <typename T>
__device__ __forceinline__ T one_of() {
  if constexpr (Ar<T>::cplx) return mk(1.0, 0.0);
  else return 1.0;
}

// S = R - alpha V ; ||S||^2                      in: R, V ; coef: alpha (negated)
struct PlanStabS {
  static constexpr int NI = 2, NO = 1, NC = 1, NR = 1;
  __host__ __device__ static constexpr bool cj(int) { return false; }
  __host__ __device__ static constexpr bool neg(int) { return true; }
  __host__ __device__ static constexpr int rmode(int) { return RED_NORM2; }
  template <typename T>
  __device__ __forceinline__ static void elem(const T (&x)[NI], const T (&c)[NC], T (&y)[NO], T (&ra)[NR]) {
    const T z = Ar<T>::zero();
    y[0] = Ar<T>::fma(x[1], c[0], Ar<T>::fma(x[0], one_of<T>(), z));
    ra[0] = Ar<T>::cfma(y[0], y[0], ra[0]);
  }
};
// X = X + alpha P + omega S ; R = S - omega T ; <R, R~>, ||R||^2      in: X, P, S, T, R~ ; coef: alpha, omega, -omega
struct PlanStabXR {
  static constexpr int NI = 5, NO = 2, NC = 3, NR = 2;
  __host__ __device__ static constexpr bool cj(int) { return false; }
  __host__ __device__ static constexpr bool neg(int i) { return i == 2; }
  __host__ __device__ static constexpr int rmode(int r) { return r == 0 ? RED_TRACE : RED_NORM2; }
  template <typename T>
  __device__ __forceinline__ static void elem(const T (&x)[NI], const T (&c)[NC], T (&y)[NO], T (&ra)[NR]) {
    const T z = Ar<T>::zero();
    y[0] = Ar<T>::fma(x[2], c[1], Ar<T>::fma(x[1], c[0], Ar<T>::fma(x[0], one_of<T>(), z)));
    y[1] = Ar<T>::fma(x[3], c[2], Ar<T>::fma(x[2], one_of<T>(), z));
    ra[0] = Ar<T>::cfma(x[4], y[1], ra[0]);
    ra[1] = Ar<T>::cfma(y[1], y[1], ra[1]);
  }
};
// P = R + beta P - (beta omega) V                in: R, P, V ; coef: beta, beta omega (negated)
struct PlanStabP {
  static constexpr int NI = 3, NO = 1, NC = 2, NR = 0;
  __host__ __device__ static constexpr bool cj(int) { return false; }
  __host__ __device__ static constexpr bool neg(int i) { return i == 1; }
  __host__ __device__ static constexpr int rmode(int) { return RED_NONE; }
  template <typename T>
  __device__ __forceinline__ static void elem(const T (&x)[NI], const T (&c)[NC], T (&y)[NO], T (&)[1]) {
    const T z = Ar<T>::zero();
    y[0] = Ar<T>::fma(x[2], c[1], Ar<T>::fma(x[1], c[0], Ar<T>::fma(x[0], one_of<T>(), z)));
  }
};

// Gl-BiCG (Alg. 2): X = X + alpha P ; R = R - alpha Q ; R^ = R^ - conj(alpha) Q^ ; <R, R^>, ||R||^2
//                                in: X, P, R, Q, R^, Q^ ; coef: alpha, -alpha, -conj(alpha)
struct PlanBicgXR {
  static constexpr int NI = 6, NO = 3, NC = 3, NR = 2;
  __host__ __device__ static constexpr bool cj(int i) { return i == 2; }
  __host__ __device__ static constexpr bool neg(int i) { return i >= 1; }
  __host__ __device__ static constexpr int rmode(int r) { return r == 0 ? RED_TRACE : RED_NORM2; }
  template <typename T>
  __device__ __forceinline__ static void elem(const T (&x)[NI], const T (&c)[NC], T (&y)[NO], T (&ra)[NR]) {
    const T z = Ar<T>::zero();
    y[0] = Ar<T>::fma(x[1], c[0], Ar<T>::fma(x[0], one_of<T>(), z));
    y[1] = Ar<T>::fma(x[3], c[1], Ar<T>::fma(x[2], one_of<T>(), z));
    y[2] = Ar<T>::fma(x[5], c[2], Ar<T>::fma(x[4], one_of<T>(), z));
    ra[0] = Ar<T>::cfma(y[2], y[1], ra[0]);
    ra[1] = Ar<T>::cfma(y[1], y[1], ra[1]);
  }
};
// P = R + beta P ; P^ = R^ + conj(beta) P^        in: R, P, R^, P^ ; coef: beta, conj(beta)
struct PlanBicgP {
  static constexpr int NI = 4, NO = 2, NC = 2, NR = 0;
  __host__ __device__ static constexpr bool cj(int i) { return i == 1; }
  __host__ __device__ static constexpr bool neg(int) { return false; }
  __host__ __device__ static constexpr int rmode(int) { return RED_NONE; }
  template <typename T>
  __device__ __forceinline__ static void elem(const T (&x)[NI], const T (&c)[NC], T (&y)[NO], T (&)[1]) {
    const T z = Ar<T>::zero();
    y[0] = Ar<T>::fma(x[1], c[0], Ar<T>::fma(x[0], one_of<T>(), z));
    y[1] = Ar<T>::fma(x[3], c[1], Ar<T>::fma(x[2], one_of<T>(), z));
  }
};

// Gl-QMR: V~ = P~ - (beta/rho) V~ ; W~ = A^H Q - (conj(beta)/xi) W~ ; ||V~||^2, <V~, W~>, ||W~||^2
//                            in: P~, V~, A^H Q, W~ ; coef: beta/rho (negated), conj(beta)/xi (negated)
struct PlanQmrVW {
  static constexpr int NI = 4, NO = 2, NC = 2, NR = 3;
  __host__ __device__ static constexpr bool cj(int) { return false; }
  __host__ __device__ static constexpr bool neg(int) { return true; }
  __host__ __device__ static constexpr int rmode(int r) { return r == 1 ? RED_TRACE : RED_NORM2; }
  template <typename T>
  __device__ __forceinline__ static void elem(const T (&x)[NI], const T (&c)[NC], T (&y)[NO], T (&ra)[NR]) {
    const T z = Ar<T>::zero();
    y[0] = Ar<T>::fma(x[1], c[0], Ar<T>::fma(x[0], one_of<T>(), z));
    y[1] = Ar<T>::fma(x[3], c[1], Ar<T>::fma(x[2], one_of<T>(), z));
    ra[0] = Ar<T>::cfma(y[0], y[0], ra[0]);
    ra[1] = Ar<T>::cfma(y[1], y[0], ra[1]);
    ra[2] = Ar<T>::cfma(y[1], y[1], ra[2]);
  }
};

template <typename T, typename P>
__global__ void __launch_bounds__(256, (sizeof(T) == 16 && P::NI > 3) ? (P::NI > 5 ? 2 : 3) : (P::NI > 5 ? 3 : 4)) flat_kernel(FlatArgs a) {
  if (a.done && *a.done) return;
  constexpr int W = 128 / (int)sizeof(T);
  using L = Lay<T, W>;
  constexpr int E = L::EPL;
  constexpr int NRA = P::NR > 0 ? P::NR : 1;
  __shared__ double rsm[16];
  T c[P::NC];
#pragma unroll
  for (int i = 0; i < P::NC; ++i) {
    c[i] = Ar<T>::ld(a.ws + a.coff[i]);
    if (P::cj(i)) c[i] = Ar<T>::conj(c[i]);
    if (P::neg(i)) c[i] = Ar<T>::sub(Ar<T>::zero(), c[i]);
  }
  RedAcc<T, W, false> acc[NRA];
#pragma unroll
  for (int r = 0; r < NRA; ++r) red_zero(acc[r]);
  const long long stride = (long long)gridDim.x * 256;
  for (long long u = (long long)blockIdx.x * 256 + threadIdx.x; u < a.units; u += stride) {
    double2 t[P::NI];
#pragma unroll
    for (int b = 0; b < P::NI; ++b) t[b] = reinterpret_cast<const double2*>(a.in[b])[u];
    T y[P::NO][E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      T xe[P::NI], ye[P::NO], ra[NRA];
#pragma unroll
      for (int b = 0; b < P::NI; ++b) {
        if constexpr (E == 2) xe[b] = e == 0 ? t[b].x : t[b].y;
        else xe[b] = t[b];
      }
#pragma unroll
      for (int r = 0; r < NRA; ++r) ra[r] = acc[r].v[e];
      P::template elem<T>(xe, c, ye, ra);
#pragma unroll
      for (int r = 0; r < NRA; ++r) acc[r].v[e] = ra[r];
#pragma unroll
      for (int o = 0; o < P::NO; ++o) y[o][e] = ye[o];
    }
#pragma unroll
    for (int o = 0; o < P::NO; ++o) {
      if constexpr (E == 2) reinterpret_cast<double2*>(a.out[o])[u] = make_double2(y[o][0], y[o][1]);
      else reinterpret_cast<double2*>(a.out[o])[u] = y[o][0];
    }
  }
  __syncwarp();
  int poff = 0;
  if constexpr (P::NR > 0) {
    red_flush<T, W, P::rmode(0), false>(acc[0], a.partials, a.pstride, poff, W, rsm);
    poff += red_len(P::rmode(0), W, Ar<T>::cplx);
  }
  if constexpr (P::NR > 1) {
    red_flush<T, W, P::rmode(1), false>(acc[1], a.partials, a.pstride, poff, W, rsm);
    poff += red_len(P::rmode(1), W, Ar<T>::cplx);
  }
  if constexpr (P::NR > 2) {
    red_flush<T, W, P::rmode(2), false>(acc[2], a.partials, a.pstride, poff, W, rsm);
    poff += red_len(P::rmode(2), W, Ar<T>::cplx);
  }
  static_assert(P::NR <= 3, "three reductions per plan");
}

template <typename P>
static int launch_plan(bool cplx, const FlatArgs& a, int grid, cudaStream_t st) {
  if (grid < 0) {
    int nb = 0;
    if (cplx) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, flat_kernel<double2, P>, 256, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, flat_kernel<double, P>, 256, 0);
    return nb;
  }
  if (cplx) flat_kernel<double2, P><<<grid, 256, 0, st>>>(a);
  else flat_kernel<double, P><<<grid, 256, 0, st>>>(a);
  return (int)cudaGetLastError();
}

template <typename P>
static FlatPlanInfo info_of() {
  FlatPlanInfo f{};
  f.ni = P::NI; f.no = P::NO; f.nc = P::NC; f.nr = P::NR;
  for (int r = 0; r < P::NR && r < 3; ++r) f.rmode[r] = P::rmode(r);
  return f;
}

FlatPlanInfo flat_plan_info(int plan) {
  switch (plan) {
    case FP_STAB_S: return info_of<PlanStabS>();
    case FP_STAB_XR: return info_of<PlanStabXR>();
    case FP_STAB_P: return info_of<PlanStabP>();
    case FP_BICG_XR: return info_of<PlanBicgXR>();
    case FP_BICG_P: return info_of<PlanBicgP>();
    case FP_QMR_VW: return info_of<PlanQmrVW>();
    default: return FlatPlanInfo{};
  }
}

// grid < 0: resident CTAs per SM of the plan's instance
int launch_flat(int plan, bool cplx, const FlatArgs& a, int grid, cudaStream_t st) {
  switch (plan) {
    case FP_STAB_S: return launch_plan<PlanStabS>(cplx, a, grid, st);
    case FP_STAB_XR: return launch_plan<PlanStabXR>(cplx, a, grid, st);
    case FP_STAB_P: return launch_plan<PlanStabP>(cplx, a, grid, st);
    case FP_BICG_XR: return launch_plan<PlanBicgXR>(cplx, a, grid, st);
    case FP_BICG_P: return launch_plan<PlanBicgP>(cplx, a, grid, st);
    case FP_QMR_VW: return launch_plan<PlanQmrVW>(cplx, a, grid, st);
    default: return grid < 0 ? 0 : (int)cudaErrorInvalidValue;
  }
}

}  // namespace srk
