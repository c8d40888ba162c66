// trsv.cu — the level-scheduled triangular solves of the right ILU(0)
// preconditioner on n x s row-major blocks:
//   z_i = (r_i - sum_{j in T_i} t_ij z_j) * dinv_i        (dinv = 1 for a unit factor)
// One launch per level (ilu.cu's schedule): every row of a level depends only on rows
// of earlier levels, so a warp takes one row and its lanes the s columns (coalesced
// row-major accesses, s <= 64 in two lane passes). Deterministic: each z_i is one
// fixed-order sum.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "engine.h"

namespace srk {

namespace {

template <typename T>
__global__ void trsv_level_kernel(const int* __restrict__ order, int lo, int hi, const int* __restrict__ rp,
                                  const int* __restrict__ ci, const T* __restrict__ val, const T* __restrict__ dinv,
                                  const T* R, T* Z, int s, const int* done) {
  if (done && *done) return;
  const int w = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int k = lo + w;
  if (k >= hi) return;
  const int i = __ldg(order + k);
  const int b = __ldg(rp + i), e = __ldg(rp + i + 1);
  for (int c = lane; c < s; c += 32) {
    T acc = R[(size_t)i * s + c];
    for (int p = b; p < e; ++p) {
      const T t = __ldg(val + p);
      const T z = Z[(size_t)__ldg(ci + p) * s + c];
      acc = Ar<T>::sub(acc, Ar<T>::mul(t, z));
    }
    if (dinv) acc = Ar<T>::mul(acc, __ldg(dinv + i));
    Z[(size_t)i * s + c] = acc;
  }
}

template <typename T>
__global__ void trimul_kernel(long long n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ val,
                              const T* __restrict__ diag, const T* __restrict__ R, T* __restrict__ Z, int s) {
  const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int b = __ldg(rp + i), e = __ldg(rp + i + 1);
  for (int c = lane; c < s; c += 32) {
    T acc = R[(size_t)i * s + c];
    if (diag) acc = Ar<T>::mul(__ldg(diag + i), acc);
    for (int p = b; p < e; ++p) acc = Ar<T>::add(acc, Ar<T>::mul(__ldg(val + p), R[(size_t)__ldg(ci + p) * s + c]));
    Z[(size_t)i * s + c] = acc;
  }
}

template <typename T>
__device__ __forceinline__ T nan_of();
template <>
__device__ __forceinline__ double nan_of<double>() { return __longlong_as_double(0x7ff8000000000000LL); }
template <>
__device__ __forceinline__ double2 nan_of<double2>() {
  return make_double2(__longlong_as_double(0x7ff8000000000000LL), __longlong_as_double(0x7ff8000000000000LL));
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Sync-free variant (one launch per solve): warps take rows in level order from an atomic
// work counter, so every row a warp waits on was taken earlier by a running warp (no
// deadlock whatever the residency). A row waits for its dependencies' done flags
// (acquire loads), reads their Z rows through L2 (ld.global.cg: L1 is not coherent across
// SMs), writes its own row, and one lane fences and raises the row's flag. Same fixed-order sums as the
// level kernel (bitwise-identical results). A spin that outlives ~2^26 polls (a broken
// schedule) writes NaN instead of hanging, so the solver reports a non-finite breakdown.
template <typename T>
__global__ void trsv_syncfree_kernel(const int* __restrict__ order, int nrows, const int* __restrict__ rp,
                                     const int* __restrict__ ci, const T* __restrict__ val,
                                     const T* __restrict__ dinv, const T* R, T* Z, int s, int* flags,
                                     const int* done) {
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  int* counter = flags + nrows;
  volatile int* vflags = flags;
  while (true) {
    int k = 0;
    if (lane == 0) k = atomicAdd(counter, 1);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= nrows) break;
    const int i = __ldg(order + k);
    const int b = __ldg(rp + i), e = __ldg(rp + i + 1);
    bool bad = false;
    for (int p = b + lane; p < e; p += 32) {
      const int j = __ldg(ci + p);
      long long spin = 0;
      while (ld_acquire(flags + j) == 0) {  // acquire: the row's Z was written before its flag
        if (++spin > (1LL << 26)) {
          bad = true;
          break;
        }
      }
    }
    // __syncwarp orders every lane's acquire loads before any lane's reads of the
    // dependencies' Z rows below (vote intrinsics alone carry no memory ordering)
    __syncwarp();
    bad = __any_sync(0xffffffffu, bad);
    for (int c = lane; c < s; c += 32) {
      T acc = R[(size_t)i * s + c];
      for (int p = b; p < e; ++p) {
        const T tv = __ldg(val + p);
        const T z = __ldcg(Z + (size_t)__ldg(ci + p) * s + c);
        acc = Ar<T>::sub(acc, Ar<T>::mul(tv, z));
      }
      if (dinv) acc = Ar<T>::mul(acc, __ldg(dinv + i));
      if (bad) acc = nan_of<T>();
      Z[(size_t)i * s + c] = acc;
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();  // release, cumulative over the warp's writes ordered by the barrier
      vflags[i] = 1;
    }
  }
}

template <typename T>
int run_syncfree(const DevTri& t, long long n, int s, const void* R, void* Z, const int* done, cudaStream_t st) {
  const int nrows = t.lvl.empty() ? 0 : t.lvl.back();
  if (nrows == 0) return 0;
  DevTri& tm = const_cast<DevTri&>(t);  // the flag array is scratch owned by the factor
  if (!tm.flags) {  // first use runs eagerly (never inside a graph capture)
    if (cudaMalloc(&tm.flags, sizeof(int) * ((size_t)n + 1)) != cudaSuccess) return -(int)cudaErrorMemoryAllocation;
  }
  cudaMemsetAsync(tm.flags, 0, sizeof(int) * ((size_t)n + 1), st);
  static std::atomic<int> grids[64];  // per device ordinal (occupancy x SM count)
  int dev = 0;
  cudaGetDevice(&dev);
  int grid = grids[dev & 63].load();
  if (!grid) {
    int nsm = 0, occ = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, trsv_syncfree_kernel<T>, 256, 0);
    grid = nsm * std::max(1, occ);
    grids[dev & 63].store(grid);
  }
  const int g = (int)std::min<long long>(grid, ((long long)nrows + 7) / 8);
  trsv_syncfree_kernel<T><<<g, 256, 0, st>>>(t.order, nrows, t.rp, t.ci, reinterpret_cast<const T*>(t.val),
                                             reinterpret_cast<const T*>(t.dinv), reinterpret_cast<const T*>(R),
                                             reinterpret_cast<T*>(Z), s, tm.flags, done);
  const int e = (int)cudaGetLastError();
  return e ? -e : 1;
}

template <typename T>
int run(const DevTri& t, long long n, int s, const void* R, void* Z, const int* done, cudaStream_t st) {
  static const bool levels = getenv("SRK_TRSV_LEVELS") != nullptr;  // A/B: one launch per level
  if (!levels) return run_syncfree<T>(t, n, s, R, Z, done, st);
  const int nlev = (int)t.lvl.size() - 1;
  for (int l = 0; l < nlev; ++l) {
    const int lo = t.lvl[l], hi = t.lvl[l + 1];
    const int rows = hi - lo;
    if (rows <= 0) continue;
    const int warps_per_cta = 8;
    const int grid = (rows + warps_per_cta - 1) / warps_per_cta;
    // level 0 rows have no dependencies but still need Z = R * dinv: same kernel
    trsv_level_kernel<T><<<grid, warps_per_cta * 32, 0, st>>>(
        t.order, lo, hi, t.rp, t.ci, reinterpret_cast<const T*>(t.val), reinterpret_cast<const T*>(t.dinv),
        reinterpret_cast<const T*>(R), reinterpret_cast<T*>(Z), s, done);
  }
  const int e = (int)cudaGetLastError();
  return e ? -e : nlev;
}

}  // namespace

int launch_trsv(const DevTri& t, bool cplx, long long n, int s, const void* R, void* Z, const int* done, cudaStream_t st) {
  return cplx ? run<double2>(t, n, s, R, Z, done, st) : run<double>(t, n, s, R, Z, done, st);
}

// ILUTP row permutation of an n x s block (rows of w doubles): gather dst[k] = src[perm[k]]
// (Pi P, before the L solve) or scatter dst[perm[k]] = src[k] (Pi^T, after the L^H solve)
__global__ static void permute_kernel(const int* __restrict__ perm, int gather, long long n, int w,
                                      const double* __restrict__ src, double* __restrict__ dst) {
  const long long tot = n * (long long)w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long k = e / w, c = e % w;
    const long long r = perm[k];
    if (gather) dst[k * w + c] = src[r * w + c];
    else dst[r * w + c] = src[k * w + c];
  }
}

int launch_permute(const int* perm, bool gather, bool cplx, long long n, int s, const void* src, void* dst,
                   cudaStream_t st) {
  const int w = s * (cplx ? 2 : 1);
  const long long tot = n * (long long)w;
  const int grid = (int)std::max<long long>(1, std::min<long long>((tot + 255) / 256, 148LL * 16));
  permute_kernel<<<grid, 256, 0, st>>>(perm, gather ? 1 : 0, n, w, reinterpret_cast<const double*>(src),
                                       reinterpret_cast<double*>(dst));
  return (int)cudaGetLastError();
}

int launch_trimul(const DevTri& t, bool cplx, long long n, int s, const void* R, void* Z, cudaStream_t st) {
  const int grid = (int)((n + 7) / 8);
  if (cplx)
    trimul_kernel<double2><<<grid, 256, 0, st>>>(n, t.rp, t.ci, reinterpret_cast<const double2*>(t.val),
                                                  reinterpret_cast<const double2*>(t.diag),
                                                  reinterpret_cast<const double2*>(R), reinterpret_cast<double2*>(Z), s);
  else
    trimul_kernel<double><<<grid, 256, 0, st>>>(n, t.rp, t.ci, reinterpret_cast<const double*>(t.val),
                                                reinterpret_cast<const double*>(t.diag), reinterpret_cast<const double*>(R),
                                                reinterpret_cast<double*>(Z), s);
  return (int)cudaGetLastError();
}

}  // namespace srk
