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
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// narrow Grams (real width w <= 32): every warp owns the whole W x W accumulator and
// a private ring of RT-row stages filled by cp.async (no CTA barriers in the loop).
// Smem rows are padded to LDS = W + 2 doubles (row r starts 16-byte group r mod 8 later)
// and lane (fr, fk) reads, per k-step (4 rows), the 16-byte column pairs
// cpair(fr, h) = 8h + (fr even ? fr/2 : fr/2 + 4): the 8 lanes of each quarter-warp then
// hit 8 distinct bank groups, and one 16-byte load feeds two 8 x 8 output tiles
// (tile 2h + e takes column 2 cpair + e for m = fr). The same layout serves the B
// fragments, so X == Y needs one load per k-step.
// ---------------------------------------------------------------------------
constexpr int RT = 16;  // rows per stage

__device__ __forceinline__ int cpair(int f, int h) { return 8 * h + ((f & 1) ? (f >> 1) + 4 : (f >> 1)); }

template <int W>
__global__ void __launch_bounds__(256, 2) gram_warp_kernel(GramArgs g, int stg) {
  if (g.done && *g.done) return;
  constexpr int NT = W / 8, NH = W / 16, LDS = W + 2;
  extern __shared__ __align__(16) double gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 2, fk = lane & 3;
  const long long n = g.n;
  const int w = g.w;
  const bool vec = (w % 2) == 0;
  const bool same = g.X == g.Y;
  const int nops = same ? 1 : 2;
  const int slen = nops * RT * LDS;
  double* ring = gsm + (size_t)warp * stg * slen;
  // zero the ring once: the padding columns (>= w) are never written by the copies
  for (int i = lane; i < stg * slen; i += 32) ring[i] = 0.0;
  __syncwarp();
  const long long ntile = (n + RT - 1) / RT;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long first = (long long)blockIdx.x * (blockDim.x >> 5) + warp;

  auto stage = [&](long long tile, int q) {
    double* dst0 = ring + (size_t)q * slen;
    const long long r0 = tile * RT;
    for (int op = 0; op < nops; ++op) {
      const double* src = op ? g.X : g.Y;
      double* dst = dst0 + op * RT * LDS;
      if (vec) {
        const int pairs = w / 2;
        for (int t = lane; t < RT * pairs; t += 32) {
          const int k = t / pairs, cp = t % pairs;
          const long long r = r0 + k;
          if (r < n) cp_async16(dst + k * LDS + 2 * cp, src + (size_t)r * w + 2 * cp);
          else *reinterpret_cast<double2*>(dst + k * LDS + 2 * cp) = make_double2(0.0, 0.0);
        }
      } else {
        for (int t = lane; t < RT * w; t += 32) {
          const int k = t / w, c = t % w;
          const long long r = r0 + k;
          if (r < n) cp_async8(dst + k * LDS + c, src + (size_t)r * w + c);
          else dst[k * LDS + c] = 0.0;
        }
      }
    }
  };

  double acc[NT][NT][2];
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int q = 0; q < stg - 1; ++q) {
    const long long t = first + q * nwarps;
    if (t < ntile) stage(t, q);
    cp_commit();
  }
  long long k = 0;
  for (long long tile = first; tile < ntile; tile += nwarps, ++k) {
    {
      const long long tn = tile + (long long)(stg - 1) * nwarps;
      if (tn < ntile) stage(tn, (int)((k + stg - 1) % stg));
      cp_commit();
    }
    // all but the newest stg - 1 groups complete (runtime depth: stg is 2..4)
    if (stg == 2) cp_wait<1>();
    else if (stg == 3) cp_wait<2>();
    else cp_wait<3>();
    __syncwarp();
    const double* ys = ring + (size_t)(k % stg) * slen;
    const double* xs = same ? ys : ys + RT * LDS;
#pragma unroll
    for (int ks = 0; ks < RT / 4; ++ks) {
      const int rr = (ks * 4 + fk) * LDS;
      double2 ya[NH], xa[NH];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        ya[h] = *reinterpret_cast<const double2*>(ys + rr + 2 * cpair(fr, h));
        xa[h] = same ? ya[h] : *reinterpret_cast<const double2*>(xs + rr + 2 * cpair(fr, h));
      }
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
          dmma(acc[i][j], (i & 1) ? ya[i >> 1].y : ya[i >> 1].x, (j & 1) ? xa[j >> 1].y : xa[j >> 1].x);
    }
    __syncwarp();  // this stage is refilled next iteration
  }
  cp_wait<0>();
  __syncthreads();
  // warps' W x W partials (real, natural column order) -> shared memory -> fixed-order sum
  double* bsm = gsm;  // 8 * W * W doubles <= the ring
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = 2 * cpair(fr, i >> 1) + (i & 1);        // column of Y (m = fr of tile i)
        const int col = 2 * cpair(2 * fk + e, j >> 1) + (j & 1);  // column of X (n = 2fk + e of tile j)
        bsm[(size_t)warp * W * W + row * W + col] = acc[i][j][e];
      }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  auto bval = [&](int r, int c) {
    double v = 0.0;
    for (int q = 0; q < nw; ++q) v += bsm[(size_t)q * W * W + r * W + c];
    return v;
  };
  double* out = g.partials + (size_t)blockIdx.x * g.pstride;
  const int s = g.s;
  if (!g.cplx) {
    for (int t = threadIdx.x; t < s * s; t += blockDim.x) out[t] = bval(t / s, t % s);
  } else {
    for (int t = threadIdx.x; t < s * s; t += blockDim.x) {
      const int j = t / s, kk = t % s;
      out[2 * t] = bval(2 * j, 2 * kk) + bval(2 * j + 1, 2 * kk + 1);
      out[2 * t + 1] = bval(2 * j, 2 * kk + 1) - bval(2 * j + 1, 2 * kk);
    }
  }
}

template <int W>
int stages_w(const GramArgs& g) {
  const int nops = g.X == g.Y ? 1 : 2;
  const size_t per = (size_t)8 * nops * RT * (W + 2) * 8;  // one stage for each of 8 warps
  int stg = (int)std::min<size_t>(4, (size_t)(110 * 1024) / per);
  return std::max(2, stg);
}

template <int W>
int launch_warp_w(const GramArgs& g, int grid, cudaStream_t st) {
  const int stg = stages_w<W>(g);
  const int nops = g.X == g.Y ? 1 : 2;
  const size_t smem = std::max<size_t>((size_t)8 * stg * nops * RT * (W + 2) * 8, (size_t)8 * W * W * 8);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(gram_warp_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  if (grid < 0) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gram_warp_kernel<W>, 256, smem);
    return occ;
  }
  gram_warp_kernel<W><<<grid, 256, smem, st>>>(g, stg);
  return (int)cudaGetLastError();
}

template <int W>
int launch_w(const GramArgs& g, int grid, cudaStream_t st) {
  using C = GCfg<W>;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(gram_mma_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
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
  // a block's own Gram (X == Y) on the per-warp kernel: one staged copy, no CTA barriers
  // (n = 2^21: 3.5 / 3.1 TB/s at w = 16 / 32 against 2.8 / 2.3 for the CTA-tiled kernel);
  // distinct operands stay CTA-tiled (4.8 / 4.0 TB/s against 4.6 / 3.4: twice the bytes
  // per stage leave the per-warp ring one stage deep). SRK_GRAM_CTA=1: always CTA-tiled.
  static const bool cta = getenv("SRK_GRAM_CTA") != nullptr;
  const bool warp = !cta && g.X == g.Y;
  if (g.w <= 16) return warp ? launch_warp_w<16>(g, grid, st) : launch_w<16>(g, grid, st);
  if (g.w <= 32) return warp ? launch_warp_w<32>(g, grid, st) : launch_w<32>(g, grid, st);
  if (g.w <= 64) return launch_w<64>(g, grid, st);
  if (g.w <= 128) return launch_w<128>(g, grid, st);
  return (int)cudaErrorInvalidValue;
}

int gram_mma_chunks(long long n) { return (int)std::min<long long>((n + KCMIN - 1) / KCMIN, 1LL << 30); }

}  // namespace srk
