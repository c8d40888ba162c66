// small.cuh — s x s coefficient algebra on the device, executed by ONE CTA
// ("on device, in one warp/CTA: LU-with-pivoting solves
// G^-1 M, adjoint reuse G^-H M^H, products with C/Sigma, Cholesky (CholQR),
// 2s x s Householder QR (Bl-QMR), scalars, breakdown tests").
//
// Matrices are row-major arrays of T (double or double2) in global memory
// (the coefficient workspace) or shared memory. Every routine is called by all
// threads of the CTA and ends with __syncthreads().
#pragma once
#include "common.cuh"

namespace srk {

constexpr double EPS_BRK = 1e-14;   // reading G12: LU pivot <= EPS_BRK * max|G| -> singular Gram
constexpr double EPS_DEFL = 1e-12;  // reading G11: R_jj <= EPS_DEFL * ||Z||_F -> rank deficient (MGS2)
// CholQR works on the Gram G = Z^H Z, whose pivots carry an absolute rounding error ~ eps * tr(G):
// it flags rank deficiency when a pivot d_j <= EPS_CHOL * tr(G), i.e. a column norm below ~1e-7
// relative — the resolution limit of CholQR (reading R5 in DESIGN.md).
constexpr double EPS_CHOL = 1e-14;

template <typename T> __device__ __forceinline__ T one();
template <> __device__ __forceinline__ double one<double>() { return 1.0; }
template <> __device__ __forceinline__ double2 one<double2>() { return mk(1.0, 0.0); }

__device__ __forceinline__ double cabs1(double a) { return fabs(a); }
__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }
__device__ __forceinline__ double cabs(double a) { return fabs(a); }
__device__ __forceinline__ double cabs(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ double re(double a) { return a; }
__device__ __forceinline__ double re(double2 a) { return a.x; }
__device__ __forceinline__ bool fin(double a) { return isfinite(a); }
__device__ __forceinline__ bool fin(double2 a) { return isfinite(a.x) && isfinite(a.y); }
__device__ __forceinline__ double scal(double a, double r) { return a * r; }
__device__ __forceinline__ double2 scal(double2 a, double r) { return mk(a.x * r, a.y * r); }
__device__ __forceinline__ double mkT(double r, double, double) { return r; }
__device__ __forceinline__ double2 mkT(double r, double i, double2) { return mk(r, i); }

// complex division a / b (plain formula: a * conj(b) / |b|^2)
__device__ __forceinline__ double cdiv(double a, double b) { return a / b; }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double d = b.x * b.x + b.y * b.y;
  return mk((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
template <typename T> __device__ __forceinline__ bool is_zero(T a);
template <> __device__ __forceinline__ bool is_zero<double>(double a) { return a == 0.0; }
template <> __device__ __forceinline__ bool is_zero<double2>(double2 a) { return a.x == 0.0 && a.y == 0.0; }

template <typename T>
__device__ __forceinline__ T neg(T a) { return Ar<T>::sub(Ar<T>::zero(), a); }

// C (n x m) = alpha * op(A) (n x k) * op(B) (k x m); op: 0 = N, 1 = H. C must not alias A or B.
template <typename T>
__device__ void sm_gemm(T* C, const T* A, const T* B, int n, int k, int m, int opA, int opB, T alpha) {
  for (int idx = threadIdx.x; idx < n * m; idx += blockDim.x) {
    const int i = idx / m, j = idx % m;
    T acc = Ar<T>::zero();
    for (int l = 0; l < k; ++l) {
      T a = opA ? Ar<T>::conj(A[l * n + i]) : A[i * k + l];
      T b = opB ? Ar<T>::conj(B[j * k + l]) : B[l * m + j];
      acc = Ar<T>::fma(a, b, acc);
    }
    C[idx] = Ar<T>::mul(alpha, acc);
  }
  __syncthreads();
}

// dst = op(src) (n x m source, H gives m x n)
template <typename T>
__device__ void sm_copy(T* dst, const T* src, int n, int m, int herm) {
  for (int idx = threadIdx.x; idx < n * m; idx += blockDim.x) {
    const int i = idx / m, j = idx % m;
    if (herm) dst[j * n + i] = Ar<T>::conj(src[idx]);
    else dst[idx] = src[idx];
  }
  __syncthreads();
}

template <typename T>
__device__ void sm_scale(T* dst, const T* src, int cnt, T alpha) {
  for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) dst[idx] = Ar<T>::mul(alpha, src[idx]);
  __syncthreads();
}

// Frobenius norm^2 of an n x m matrix (thread 0 sums in index order; broadcast through smem)
template <typename T>
__device__ double sm_fro2(const T* A, int cnt, double* red) {
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int i = 0; i < cnt; ++i) acc += Ar<T>::abs2(A[i]);
    red[0] = acc;
  }
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

// X (n x m) = G^{-1} M (herm = 0) or G^{-H} M (herm = 1) by LU with partial pivoting
// (SPEC small_solve S:106-114; reading G29: pivot = first max |re|+|im|, as LAPACK's
// i?amax). Returns 1 (breakdown) if a pivot <= EPS_BRK * max|G_ij| (reading G12)
// or any entry is not finite. Scratch: (n*n + n*m) T + 2 doubles in `sh`.
template <typename T>
__device__ int sm_solve(T* X, const T* G, const T* M, int n, int m, int herm, T* sh, double eps = EPS_BRK) {
  T* L = sh;
  T* B = sh + n * n;
  __shared__ int s_piv;
  __shared__ int s_bad;
  __shared__ double s_gmax;
  if (threadIdx.x == 0) { s_bad = 0; s_gmax = 0.0; }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int i = idx / n, j = idx % n;
    L[idx] = herm ? Ar<T>::conj(G[j * n + i]) : G[idx];
  }
  for (int idx = threadIdx.x; idx < n * m; idx += blockDim.x) B[idx] = M[idx];
  __syncthreads();
  if (threadIdx.x == 0) {
    double gm = 0.0;
    int bad = 0;
    for (int i = 0; i < n * n; ++i) {
      if (!fin(L[i])) bad = 1;
      gm = fmax(gm, cabs(L[i]));
    }
    for (int i = 0; i < n * m; ++i)
      if (!fin(B[i])) bad = 1;
    if (gm == 0.0) bad = 1;
    s_gmax = gm;
    s_bad = bad;
  }
  __syncthreads();
  if (s_bad) return 1;
  for (int k = 0; k < n; ++k) {
    if (threadIdx.x == 0) {
      int p = k;
      double best = cabs1(L[k * n + k]);
      for (int i = k + 1; i < n; ++i) {
        const double v = cabs1(L[i * n + k]);
        if (v > best) { best = v; p = i; }
      }
      s_piv = p;
      if (cabs(L[p * n + k]) <= eps * s_gmax) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) return 1;
    const int p = s_piv;
    if (p != k) {
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        T t = L[k * n + j]; L[k * n + j] = L[p * n + j]; L[p * n + j] = t;
      }
      for (int j = threadIdx.x; j < m; j += blockDim.x) {
        T t = B[k * m + j]; B[k * m + j] = B[p * m + j]; B[p * m + j] = t;
      }
    }
    __syncthreads();
    // multipliers l_ik = L_ik / L_kk (stored in place)
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) L[i * n + k] = cdiv(L[i * n + k], L[k * n + k]);
    __syncthreads();
    // trailing update of L and forward elimination of B
    const int wl = n - k - 1;
    for (int idx = threadIdx.x; idx < wl * (wl + m); idx += blockDim.x) {
      const int i = k + 1 + idx / (wl + m);
      const int j = idx % (wl + m);
      const T lik = L[i * n + k];
      if (j < wl) {
        const int jj = k + 1 + j;
        L[i * n + jj] = Ar<T>::sub(L[i * n + jj], Ar<T>::mul(lik, L[k * n + jj]));
      } else {
        const int jj = j - wl;
        B[i * m + jj] = Ar<T>::sub(B[i * m + jj], Ar<T>::mul(lik, B[k * m + jj]));
      }
    }
    __syncthreads();
  }
  // back substitution, one thread per right-hand-side column
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    for (int k = n - 1; k >= 0; --k) {
      T acc = B[k * m + j];
      for (int l = k + 1; l < n; ++l) acc = Ar<T>::sub(acc, Ar<T>::mul(L[k * n + l], B[l * m + j]));
      B[k * m + j] = cdiv(acc, L[k * n + k]);
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * m; idx += blockDim.x) X[idx] = B[idx];
  __syncthreads();
  return 0;
}

// Upper Cholesky G = R^H R (n x n Hermitian positive definite). Rank test
// (reading R5): pivot d_j <= EPS_CHOL * tr(G) -> return 1. Row j: thread 0 forms the
// pivot, then one thread per entry R_jk (each entry's sum in the same order as a
// serial loop, so the result does not depend on the thread count).
template <typename T>
__device__ int sm_chol(T* R, const T* G, int n, int check_rank, double eps = EPS_CHOL) {
  __shared__ int s_bad;
  __shared__ double s_rjj;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) R[i] = Ar<T>::zero();
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      double tr = 0.0;
      for (int i = 0; i < n; ++i) tr += re(G[i * n + i]);
      const double thr = eps * tr;
      // R_jj^2 = G_jj - sum_i |R_ij|^2
      double d = re(G[j * n + j]);
      for (int i = 0; i < j; ++i) d -= Ar<T>::abs2(R[i * n + j]);
      if (!(d > 0.0) || !isfinite(d) || (check_rank && d <= thr) || tr == 0.0) {
        s_bad = 1;
      } else {
        s_rjj = sqrt(d);
        R[j * n + j] = mkT(s_rjj, 0.0, T());
      }
    }
    __syncthreads();
    if (s_bad) break;
    const double rjj = s_rjj;
    // R_jk = (G_jk - sum_i conj(R_ij) R_ik) / R_jj, k > j
    for (int k = j + 1 + threadIdx.x; k < n; k += blockDim.x) {
      T acc = G[j * n + k];
      for (int i = 0; i < j; ++i) acc = Ar<T>::sub(acc, Ar<T>::mul(Ar<T>::conj(R[i * n + j]), R[i * n + k]));
      R[j * n + k] = scal(acc, 1.0 / rjj);
    }
    __syncthreads();
  }
  int b = s_bad;
  __syncthreads();
  return b;
}

// Cholesky with the deficient pivots skipped (rank-deficiency continuation, SURVEY §8(f)
// f4): a pivot d_j <= eps * tr(G) sets bit j of the returned mask and leaves row j of R
// zero (column j is dependent on the earlier ones, so the later pivots are those of the
// block without it); ~0 on a non-finite value or a zero Gram. Same order of operations
// as sm_chol otherwise.
template <typename T>
__device__ unsigned long long sm_chol_mask(T* R, const T* G, int n, double eps) {
  __shared__ unsigned long long s_mask;
  __shared__ int s_skip;
  __shared__ double s_rjj;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) R[i] = Ar<T>::zero();
  if (threadIdx.x == 0) s_mask = 0ull;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      double tr = 0.0;
      for (int i = 0; i < n; ++i) tr += re(G[i * n + i]);
      double d = re(G[j * n + j]);
      for (int i = 0; i < j; ++i) d -= Ar<T>::abs2(R[i * n + j]);
      s_skip = 0;
      if (!isfinite(d) || !(tr > 0.0) || !isfinite(tr)) {
        s_mask = ~0ull;
      } else if (d <= eps * tr) {
        s_mask |= 1ull << j;
        s_skip = 1;
      } else {
        s_rjj = sqrt(d);
        R[j * n + j] = mkT(s_rjj, 0.0, T());
      }
    }
    __syncthreads();
    if (s_mask == ~0ull) break;
    if (!s_skip) {
      const double rjj = s_rjj;
      for (int k = j + 1 + threadIdx.x; k < n; k += blockDim.x) {
        T acc = G[j * n + k];
        for (int i = 0; i < j; ++i) acc = Ar<T>::sub(acc, Ar<T>::mul(Ar<T>::conj(R[i * n + j]), R[i * n + k]));
        R[j * n + k] = scal(acc, 1.0 / rjj);
      }
    }
    __syncthreads();
  }
  const unsigned long long m = s_mask;
  __syncthreads();
  return m;
}

// Ri = R^{-1} for upper-triangular R; one thread per column (back substitution).
template <typename T>
__device__ void sm_trinv(T* Ri, const T* R, int n) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    for (int i = 0; i < n; ++i) Ri[i * n + j] = Ar<T>::zero();
    for (int i = j; i >= 0; --i) {
      T acc = (i == j) ? one<T>() : Ar<T>::zero();
      for (int l = i + 1; l <= j; ++l) acc = Ar<T>::sub(acc, Ar<T>::mul(R[i * n + l], Ri[l * n + j]));
      Ri[i * n + j] = cdiv(acc, R[i * n + i]);
    }
  }
  __syncthreads();
}

// Full QR of a (2n x n) stack M = Om [R; 0] by Householder reflections in LAPACK's
// convention (?larfg: beta = -sign(Re alpha) * norm, real), then phase-normalised so
// diag(R) is real non-negative. Om: 2n x 2n; R: n x n. Thread 0
// forms each reflector; its application runs one thread per column (every entry
// updated by the same serial sums as a one-thread loop).
template <typename T>
__device__ void sm_qr_stack(T* Om, T* R, const T* M, int n, T* work /* 2n*n + 2n*n */) {
  const int m2 = 2 * n;
  T* A = work;           // 2n x n working copy
  T* V = work + m2 * n;  // reflectors, column j stored in V[:, j] (2n x n)
  __shared__ double tau_r[64];
  __shared__ double tau_i[64];
  __shared__ int s_skip[2];  // double-buffered: thread 0 may write j + 1's before all read j's
  __shared__ T s_d;
  for (int i = threadIdx.x; i < m2 * n; i += blockDim.x) {
    A[i] = M[i];
    V[i] = Ar<T>::zero();
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      T alpha = A[j * n + j];
      double xn2 = 0.0;
      for (int i = j + 1; i < m2; ++i) xn2 += Ar<T>::abs2(A[i * n + j]);
      double ar = re(alpha);
      double ai = 0.0;
      if constexpr (Ar<T>::cplx) ai = reinterpret_cast<double2&>(alpha).y;
      V[j * n + j] = one<T>();
      if (xn2 == 0.0 && ai == 0.0) {
        tau_r[j] = 0.0;
        tau_i[j] = 0.0;
        s_skip[j & 1] = 1;
      } else {
        double nrm = sqrt(ar * ar + ai * ai + xn2);
        double beta = (ar >= 0.0) ? -nrm : nrm;
        tau_r[j] = (beta - ar) / beta;
        tau_i[j] = -ai / beta;
        s_d = Ar<T>::sub(alpha, mkT(beta, 0.0, T()));  // alpha - beta
        s_skip[j & 1] = 0;
      }
    }
    __syncthreads();
    if (s_skip[j & 1]) continue;
    const T d = s_d;
    for (int i = j + 1 + threadIdx.x; i < m2; i += blockDim.x) V[i * n + j] = cdiv(A[i * n + j], d);
    __syncthreads();
    // apply H^H = I - conj(tau) v v^H to A[:, j:]  (geqrf applies H^H on the left)
    const T tc = mkT(tau_r[j], -tau_i[j], T());
    for (int c = j + threadIdx.x; c < n; c += blockDim.x) {
      T w = Ar<T>::zero();
      for (int i = j; i < m2; ++i) w = Ar<T>::cfma(V[i * n + j], A[i * n + c], w);  // v^H a
      w = Ar<T>::mul(tc, w);
      for (int i = j; i < m2; ++i) A[i * n + c] = Ar<T>::sub(A[i * n + c], Ar<T>::mul(V[i * n + j], w));
    }
    __syncthreads();
  }
  // Om = H_1 H_2 ... H_n applied to I (H_j = I - tau_j v_j v_j^H): columns in parallel
  for (int i = threadIdx.x; i < m2 * m2; i += blockDim.x) Om[i] = (i / m2 == i % m2) ? one<T>() : Ar<T>::zero();
  __syncthreads();
  for (int c = threadIdx.x; c < m2; c += blockDim.x)
    for (int j = n - 1; j >= 0; --j) {
      const T t = mkT(tau_r[j], tau_i[j], T());
      T w = Ar<T>::zero();
      for (int i = j; i < m2; ++i) w = Ar<T>::cfma(V[i * n + j], Om[i * m2 + c], w);
      w = Ar<T>::mul(t, w);
      for (int i = j; i < m2; ++i) Om[i * m2 + c] = Ar<T>::sub(Om[i * m2 + c], Ar<T>::mul(V[i * n + j], w));
    }
  __syncthreads();
  // R = upper n x n of A, then phase normalisation (column j of Om, row j of R)
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) R[i] = ((i % n) >= (i / n)) ? A[i] : Ar<T>::zero();
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const T d = R[j * n + j];
    const double a = cabs(d);
    if (a > 0.0) {
      const T ph = scal(d, 1.0 / a);  // phase
      for (int i = 0; i < m2; ++i) Om[i * m2 + j] = Ar<T>::mul(Om[i * m2 + j], ph);
      for (int c = 0; c < n; ++c) R[j * n + c] = Ar<T>::mul(Ar<T>::conj(ph), R[j * n + c]);
    }
  }
  __syncthreads();
}

}  // namespace srk
