// common.cuh — shared device types for the srk CUDA path (sm_100a).
//
// Block vectors (n x s, "block vector denoting a matrix of
// size n x s") are stored ROW-MAJOR ("row-interleaved"): element (i, j) at
// i*s + j, so one nonzero a_ij of A is applied to the s contiguous values of
// row j of P ("reading and storing A only once while updating ... all
// s"). Complex values are interleaved (re, im) doubles (double2).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace srk {

// True the first time it is called for the current device with this mask: launch
// attributes (cudaFuncSetAttribute) are per device context, so a per-kernel cache
// must be keyed by device ordinal, and thread-safe (virtual ranks run on threads).
inline bool first_on_device(std::atomic<unsigned long long>& seen) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  return (seen.fetch_or(bit) & bit) == 0;
}

// ---------------------------------------------------------------- scalars
struct cplx { double x, y; };

__host__ __device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }

// Arithmetic traits: T = double (SRK_F64) or double2 (SRK_C128).
template <typename T> struct Ar;
template <> struct Ar<double> {
  static constexpr bool cplx = false;
  static constexpr int ND = 1;  // doubles per value
  __device__ __forceinline__ static double zero() { return 0.0; }
  __device__ __forceinline__ static double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
  // conj(a)*b + c
  __device__ __forceinline__ static double cfma(double a, double b, double c) { return __fma_rn(a, b, c); }
  __device__ __forceinline__ static double mul(double a, double b) { return a * b; }
  __device__ __forceinline__ static double add(double a, double b) { return a + b; }
  __device__ __forceinline__ static double sub(double a, double b) { return a - b; }
  __device__ __forceinline__ static double conj(double a) { return a; }
  __device__ __forceinline__ static double abs2(double a) { return a * a; }
  __device__ __forceinline__ static double ld(const double* w) { return w[0]; }
  __device__ __forceinline__ static void st(double* w, double v) { w[0] = v; }
  __device__ __forceinline__ static double shfl(double v, int src, unsigned mask = 0xffffffffu) {
    return __shfl_sync(mask, v, src);
  }
  __device__ __forceinline__ static double shfl_xor(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
};
template <> struct Ar<double2> {
  static constexpr bool cplx = true;
  static constexpr int ND = 2;
  __device__ __forceinline__ static double2 zero() { return mk(0.0, 0.0); }
  // a*b + c
  __device__ __forceinline__ static double2 fma(double2 a, double2 b, double2 c) {
    return mk(__fma_rn(a.x, b.x, __fma_rn(-a.y, b.y, c.x)), __fma_rn(a.x, b.y, __fma_rn(a.y, b.x, c.y)));
  }
  // conj(a)*b + c
  __device__ __forceinline__ static double2 cfma(double2 a, double2 b, double2 c) {
    return mk(__fma_rn(a.x, b.x, __fma_rn(a.y, b.y, c.x)), __fma_rn(a.x, b.y, __fma_rn(-a.y, b.x, c.y)));
  }
  __device__ __forceinline__ static double2 mul(double2 a, double2 b) {
    return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
  __device__ __forceinline__ static double2 add(double2 a, double2 b) { return mk(a.x + b.x, a.y + b.y); }
  __device__ __forceinline__ static double2 sub(double2 a, double2 b) { return mk(a.x - b.x, a.y - b.y); }
  __device__ __forceinline__ static double2 conj(double2 a) { return mk(a.x, -a.y); }
  __device__ __forceinline__ static double abs2(double2 a) { return a.x * a.x + a.y * a.y; }
  __device__ __forceinline__ static double2 ld(const double* w) { return mk(w[0], w[1]); }
  __device__ __forceinline__ static void st(double* w, double2 v) { w[0] = v.x; w[1] = v.y; }
  __device__ __forceinline__ static double2 shfl(double2 v, int src, unsigned mask = 0xffffffffu) {
    return mk(__shfl_sync(mask, v.x, src), __shfl_sync(mask, v.y, src));
  }
  __device__ __forceinline__ static double2 shfl_xor(double2 v, int m) {
    return mk(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
  }
};

// ------------------------------------------------------------- row layout
// A lane group of G lanes owns one row of an n x s block with capacity S >= s.
// Each lane holds CPL "chunks" of EPC elements; chunk c of lane g covers
// row-local columns [(g + c*G)*EPC, ... + EPC).  With a 16-byte chunk every
// lane issues one coalesced 16-byte load per chunk.
__host__ __device__ constexpr int pow2ceil(int x) { return x <= 1 ? 1 : 2 * pow2ceil((x + 1) / 2); }

template <typename T, int S>
struct Lay {
  static constexpr int ESZ = (int)sizeof(T);
  static constexpr int EPC = (ESZ == 16) ? 1 : ((S % 2 == 0) ? 2 : 1);  // elements per chunk
  static constexpr int NCH = (S + EPC - 1) / EPC;                         // chunks per row
  static constexpr int G = (pow2ceil(NCH) > 32) ? 32 : pow2ceil(NCH);     // lanes per row
  static constexpr int CPL = (NCH + G - 1) / G;                           // chunks per lane
  static constexpr int EPL = CPL * EPC;                                   // elements per lane
  static constexpr int RPW = 32 / G;                                      // rows per warp
  static constexpr int PW = G * EPC * CPL;                                // padded row width (>= S)
  // row-local column of element e (0..EPL-1) of lane g
  __device__ __forceinline__ static int col(int g, int e) { return ((g + (e / EPC) * G) * EPC) + (e % EPC); }
};

// Load / store the lane's elements of one row (row pointer p, runtime width s <= S,
// vec = row base is 16-byte aligned and s*ESZ % 16 == 0).
template <typename T, int S>
__device__ __forceinline__ void row_load(const T* __restrict__ p, int g, int s, bool vec, T (&v)[Lay<T, S>::EPL]) {
  using L = Lay<T, S>;
#pragma unroll
  for (int c = 0; c < L::CPL; ++c) {
    const int c0 = (g + c * L::G) * L::EPC;
    if constexpr (L::EPC == 2) {
      if (vec && c0 + 1 < s) {
        double2 t = *reinterpret_cast<const double2*>(p + c0);
        v[c * 2] = t.x;
        v[c * 2 + 1] = t.y;
      } else {
        v[c * 2] = (c0 < s) ? p[c0] : Ar<T>::zero();
        v[c * 2 + 1] = (c0 + 1 < s) ? p[c0 + 1] : Ar<T>::zero();
      }
    } else {
      v[c] = (c0 < s) ? p[c0] : Ar<T>::zero();
    }
  }
}

// Exact-width variants (s == S, rows 16-byte aligned): no data-dependent
// branches, so a batch of loads can be issued back to back. Lanes beyond the
// chunk count (G > NCH) are masked by a lane predicate only.
template <typename T, int S>
__device__ __forceinline__ void row_load_ex(const T* __restrict__ p, int g, T (&v)[Lay<T, S>::EPL]) {
  using L = Lay<T, S>;
#pragma unroll
  for (int c = 0; c < L::CPL; ++c) {
    const int ch = g + c * L::G;
    const bool ok = (L::NCH % L::G == 0) || ch < L::NCH;
    if constexpr (L::EPC == 2) {
      double2 t = make_double2(0.0, 0.0);
      if (ok) t = __ldg(reinterpret_cast<const double2*>(p) + ch);
      v[c * 2] = t.x;
      v[c * 2 + 1] = t.y;
    } else {
      T t = Ar<T>::zero();
      if (ok) t = __ldg(p + ch);
      v[c] = t;
    }
  }
}
template <typename T, int S>
__device__ __forceinline__ void row_store_ex(T* __restrict__ p, int g, const T (&v)[Lay<T, S>::EPL]) {
  using L = Lay<T, S>;
#pragma unroll
  for (int c = 0; c < L::CPL; ++c) {
    const int ch = g + c * L::G;
    const bool ok = (L::NCH % L::G == 0) || ch < L::NCH;
    if (ok) {
      if constexpr (L::EPC == 2) reinterpret_cast<double2*>(p)[ch] = make_double2(v[c * 2], v[c * 2 + 1]);
      else p[ch] = v[c];
    }
  }
}
// streaming (evict-first) variants: data touched once per kernel
template <typename T, int S>
__device__ __forceinline__ void row_load_ex_cs(const T* p, int g, T (&v)[Lay<T, S>::EPL]) {
  using L = Lay<T, S>;
#pragma unroll
  for (int c = 0; c < L::CPL; ++c) {
    const int ch = g + c * L::G;
    const bool ok = (L::NCH % L::G == 0) || ch < L::NCH;
    if constexpr (L::EPC == 2) {
      double2 t = make_double2(0.0, 0.0);
      if (ok) t = __ldcs(reinterpret_cast<const double2*>(p) + ch);
      v[c * 2] = t.x;
      v[c * 2 + 1] = t.y;
    } else {
      T t = Ar<T>::zero();
      if (ok) t = __ldcs(p + ch);
      v[c] = t;
    }
  }
}
template <typename T, int S>
__device__ __forceinline__ void row_store_ex_cs(T* p, int g, const T (&v)[Lay<T, S>::EPL]) {
  using L = Lay<T, S>;
#pragma unroll
  for (int c = 0; c < L::CPL; ++c) {
    const int ch = g + c * L::G;
    const bool ok = (L::NCH % L::G == 0) || ch < L::NCH;
    if (ok) {
      if constexpr (L::EPC == 2) __stcs(reinterpret_cast<double2*>(p) + ch, make_double2(v[c * 2], v[c * 2 + 1]));
      else __stcs(p + ch, v[c]);
    }
  }
}
// row-local loads with a plain ld.global (data written earlier in the same kernel sequence)
template <typename T, int S>
__device__ __forceinline__ void row_load_ex_rw(const T* p, int g, T (&v)[Lay<T, S>::EPL]) {
  using L = Lay<T, S>;
#pragma unroll
  for (int c = 0; c < L::CPL; ++c) {
    const int ch = g + c * L::G;
    const bool ok = (L::NCH % L::G == 0) || ch < L::NCH;
    if constexpr (L::EPC == 2) {
      double2 t = make_double2(0.0, 0.0);
      if (ok) t = reinterpret_cast<const double2*>(p)[ch];
      v[c * 2] = t.x;
      v[c * 2 + 1] = t.y;
    } else {
      T t = Ar<T>::zero();
      if (ok) t = p[ch];
      v[c] = t;
    }
  }
}

template <typename T, int S>
__device__ __forceinline__ void row_store(T* __restrict__ p, int g, int s, bool vec, const T (&v)[Lay<T, S>::EPL]) {
  using L = Lay<T, S>;
#pragma unroll
  for (int c = 0; c < L::CPL; ++c) {
    const int c0 = (g + c * L::G) * L::EPC;
    if constexpr (L::EPC == 2) {
      if (vec && c0 + 1 < s) {
        *reinterpret_cast<double2*>(p + c0) = make_double2(v[c * 2], v[c * 2 + 1]);
      } else {
        if (c0 < s) p[c0] = v[c * 2];
        if (c0 + 1 < s) p[c0 + 1] = v[c * 2 + 1];
      }
    } else {
      if (c0 < s) p[c0] = v[c];
    }
  }
}

// Opaque select (inline PTX selp): keeps "pick one of several register rows by a
// runtime index" from being turned into an indexed local-memory array.
__device__ __forceinline__ double opaque_sel(int p, double a, double b) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}" : "=d"(r) : "d"(a), "d"(b), "r"(p));
  return r;
}
__device__ __forceinline__ double2 opaque_sel(int p, double2 a, double2 b) {
  return make_double2(opaque_sel(p, a.x, b.x), opaque_sel(p, a.y, b.y));
}

// Fetch element k (row-local column) of the row held by the lane group whose
// first lane is `base` (k must be a compile-time-unrolled index).
template <typename T, int S>
__device__ __forceinline__ T row_get(const T (&v)[Lay<T, S>::EPL], int base, int k, unsigned mask) {
  using L = Lay<T, S>;
  const int chunk = k / L::EPC, e = k % L::EPC;
  const int owner = chunk % L::G, c = chunk / L::G;
  return Ar<T>::shfl(v[c * L::EPC + e], base + owner, mask);
}

}  // namespace srk
