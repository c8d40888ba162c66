// gram_mma.cu — the s x s block Gram G = Y^H X over n rows (the
// "2s^2 inner products" of the block variants) on the FP64
// tensor cores, for widths where the contraction is dense enough to be compute
// bound (s >= 16: 2ns^2 flops against 16ns bytes, e.g. config 5 at s = 64:
// 34 GFLOP per Gram; at s = 16 the FMA epilogue costs more than this pass). mma.sync.m8n8k4.f64 (DMMA) measured 37.1 TFLOP/s on this
// B200 against 33.9 for DFMA (scripts/fp64_probe.cu), with 8x fewer instructions.
//
// A complex n x s block in interleaved storage is the real n x 2s matrix
// Z = [re_0, im_0, re_1, ...]; with B = Z_Y^T Z_X (2s x 2s real),
//   G[j][k] = (B[2j][2k] + B[2j+1][2k+1]) + i (B[2j][2k+1] - B[2j+1][2k]),
// so one real kernel serves both dtypes (real width w = s or 2s <= 128).
//
// Each CTA (8 warps, 2 per SM) streams chunks of KC consecutive
// rows of Y and X (contiguous in the row-major layout) into an NBUF-deep
// shared-memory ring with cp.async, and every warp accumulates its TM x TN
// grid of 8 x 8 output tiles in registers over the CTA's rows (k = 4 rows per
// DMMA). The CTA's W x W partial goes through shared memory into the partials
// array in the layout of the fused FULL reductions, and fin_kernel sums the CTAs
// in fixed order (deterministic, no atomics).
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.cuh"

namespace srk {

namespace {

constexpr int KCMIN = 32;  // rows per chunk (at least; narrow blocks take longer chunks)
constexpr int PADW = 8;  // smem row padding (doubles): rows k and k+1 land 16 banks apart

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int W>
struct GCfg {
  static constexpr int NT = W / 8;            // 8 x 8 tiles per dimension
  static constexpr int WM = NT < 2 ? NT : 2;  // warp grid (warps >= WM * WN only stage data)
  static constexpr int WN = NT < 4 ? NT : 4;
  static constexpr int TM = NT / WM, TN = NT / WN;
  static constexpr int LDS = W + PADW;        // smem row stride (doubles)
  static constexpr int KC = W <= 16 ? 2 * KCMIN : KCMIN;  // rows per chunk: >= 24 KB in flight per stage
  static constexpr int BUF = 2 * KC * LDS;    // Y chunk + X chunk (doubles)
  static constexpr int NBUF = W <= 64 ? 3 : 2;
  static constexpr int SMEM = NBUF * BUF * 8;
};

template <int W>
__global__ void __launch_bounds__(256, W <= 64 ? 2 : 1) gram_mma_kernel(GramArgs g) {
  if (g.done && *g.done) return;
  using C = GCfg<W>;
  extern __shared__ __align__(16) double gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp / C::WN, wn = warp % C::WN;
  const long long n = g.n;
  const int w = g.w;
  const long long nchunk = (n + C::KC - 1) / C::KC;
  const bool vec = (w % 2) == 0;  // 16-byte rows
  const bool same = g.X == g.Y;   // a block's own Gram (CholQR): one copy serves both operands
  const int nops = same ? 1 : 2;

  // stage chunk c of Y and X into buffer b (columns >= w and rows >= n are zero)
  auto stage = [&](long long c, int b) {
    double* ys = gsm + (size_t)b * C::BUF;
    double* xs = ys + C::KC * C::LDS;
    const long long r0 = c * C::KC;
    if (vec) {
      const int pairs = W / 2;
      for (int t = threadIdx.x; t < nops * C::KC * pairs; t += blockDim.x) {
        const int which = t / (C::KC * pairs);
        const int rem = t % (C::KC * pairs);
        const int k = rem / pairs, cp = rem % pairs;
        double* dst = (which ? xs : ys) + k * C::LDS + 2 * cp;
        const long long r = r0 + k;
        if (r < n && 2 * cp < w) {
          cp_async16(dst, (which ? g.X : g.Y) + (size_t)r * w + 2 * cp);
        } else {
          dst[0] = 0.0;
          dst[1] = 0.0;
        }
      }
    } else {
      for (int t = threadIdx.x; t < nops * C::KC * W; t += blockDim.x) {
        const int which = t / (C::KC * W);
        const int rem = t % (C::KC * W);
        const int k = rem / W, col = rem % W;
        double* dst = (which ? xs : ys) + k * C::LDS + col;
        const long long r = r0 + k;
        if (r < n && col < w) cp_async8(dst, (which ? g.X : g.Y) + (size_t)r * w + col);
        else dst[0] = 0.0;
      }
    }
  };

  double acc[C::TM][C::TN][2];
#pragma unroll
  for (int i = 0; i < C::TM; ++i)
#pragma unroll
    for (int j = 0; j < C::TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // fragment coordinates (m8n8k4, .row A / .col B): lane -> (row l/4, k l%4)
  const int fr = lane >> 2, fk = lane & 3;
  long long c0 = blockIdx.x;
  // prologue: NBUF - 1 chunks in flight
#pragma unroll
  for (int p = 0; p < C::NBUF - 1; ++p) {
    const long long c = c0 + (long long)p * gridDim.x;
    if (c < nchunk) stage(c, p);
    cp_commit();
  }
  int it = 0;
  for (long long c = c0; c < nchunk; c += gridDim.x, ++it) {
    {  // keep NBUF - 1 chunks ahead
      const long long cn = c + (long long)(C::NBUF - 1) * gridDim.x;
      if (cn < nchunk) stage(cn, (it + C::NBUF - 1) % C::NBUF);
      cp_commit();
    }
    cp_wait<C::NBUF - 1>();
    __syncthreads();
    const double* ys = gsm + (size_t)(it % C::NBUF) * C::BUF;
    const double* xs = same ? ys : ys + C::KC * C::LDS;
#pragma unroll
    for (int k0 = 0; k0 < C::KC; k0 += 4) {
      if (warp >= C::WM * C::WN) break;
      double a[C::TM], bb[C::TN];
#pragma unroll
      for (int i = 0; i < C::TM; ++i) a[i] = ys[(k0 + fk) * C::LDS + (wm * C::TM + i) * 8 + fr];
#pragma unroll
      for (int j = 0; j < C::TN; ++j) bb[j] = xs[(k0 + fk) * C::LDS + (wn * C::TN + j) * 8 + fr];
#pragma unroll
      for (int i = 0; i < C::TM; ++i)
#pragma unroll
        for (int j = 0; j < C::TN; ++j) dmma(acc[i][j], a[i], bb[j]);
    }
    __syncthreads();  // buffer it % NBUF is refilled next iteration
  }
  cp_wait<0>();
  __syncthreads();
  // CTA partial: B (W x W real) through shared memory, then the FULL layout
  double* bsm = gsm;  // W * W doubles <= the ring
  if (warp < C::WM * C::WN)
#pragma unroll
  for (int i = 0; i < C::TM; ++i)
#pragma unroll
    for (int j = 0; j < C::TN; ++j) {
      const int row = (wm * C::TM + i) * 8 + fr;
      const int col = (wn * C::TN + j) * 8 + 2 * fk;
      bsm[row * W + col] = acc[i][j][0];
      bsm[row * W + col + 1] = acc[i][j][1];
    }
  __syncthreads();
  double* out = g.partials + (size_t)blockIdx.x * g.pstride;
  const int s = g.s;
  if (!g.cplx) {
    for (int t = threadIdx.x; t < s * s; t += blockDim.x) out[t] = bsm[(t / s) * W + (t % s)];
  } else {
    for (int t = threadIdx.x; t < s * s; t += blockDim.x) {
      const int j = t / s, k = t % s;
      out[2 * t] = bsm[(2 * j) * W + 2 * k] + bsm[(2 * j + 1) * W + 2 * k + 1];
      out[2 * t + 1] = bsm[(2 * j) * W + 2 * k + 1] - bsm[(2 * j + 1) * W + 2 * k];
    }
  }
}

template <int W>
int launch_w(const GramArgs& g, int grid, cudaStream_t st) {
  using C = GCfg<W>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gram_mma_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  if (grid < 0) {  // resident CTAs per SM
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gram_mma_kernel<W>, 256, C::SMEM);
    return occ;
  }
  gram_mma_kernel<W><<<grid, 256, C::SMEM, st>>>(g);
  return (int)cudaGetLastError();
}

}  // namespace

// real width w <= 128; grid < 0: returns the resident CTAs per SM
int launch_gram_mma(const GramArgs& g, int grid, cudaStream_t st) {
  if (g.w <= 16) return launch_w<16>(g, grid, st);
  if (g.w <= 32) return launch_w<32>(g, grid, st);
  if (g.w <= 64) return launch_w<64>(g, grid, st);
  if (g.w <= 128) return launch_w<128>(g, grid, st);
  return (int)cudaErrorInvalidValue;
}

int gram_mma_chunks(long long n) { return (int)std::min<long long>((n + KCMIN - 1) / KCMIN, 1LL << 30); }

}  // namespace srk
