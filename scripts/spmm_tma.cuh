// spmm_tma.cuh — Q = A P with the P-row gathers done by the Tensor Memory
// Accelerator (sm_100a `cp.async.bulk.tensor.2d ... tile::gather4`): a producer
// warp reads the column indices of a tile of TR rows and issues one gather4 per 4
// nonzeros (4 rows of P, S*esz bytes each, landing back to back in shared memory
// in CSR order), plus bulk copies of the tile's values, row pointers and epilogue
// operand; the consumer warps wait
// on the stage's mbarrier and form the rows from shared memory. The gathers are
// asynchronous, so NSTAGE tiles of P rows are in flight per SM without holding
// registers (the register-gather kernel is latency bound at ~50% of HBM). Same
// arithmetic and fused epilogue as spmm_kernel (
// SURVEY §8(a) a1/a2/a3).
#pragma once
#include "block_kernels.cuh"

namespace srk {

struct alignas(64) TmaDesc {
  unsigned char bytes[128];  // CUtensorMap (opaque, 128 bytes)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx_arrive(unsigned long long* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const TmaDesc* map, int c0, int r0, int r1, int r2, int r3,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Compile-time shape of the TMA SpMM for (T, S): NP producer warps, NC consumer
// warps, tile rows TR (one row per consumer lane group), NSTAGE stages of EMAX
// gathered rows each. Each producer warp issues a contiguous chunk of the tile's
// gather4 groups (one TMA instruction is issued per warp at a time, so the issue
// rate scales with NP) from its own ring of column indices.
template <typename T, int S, bool FC, int EMAX_, int NSTAGE_, int NP_ = 4>
struct TmaCfg {
  using L = Lay<T, S>;
  static constexpr int NP = NP_;
  static constexpr int NC = 8;
  static constexpr int NT = 32 * (NP + NC);
  static constexpr int TR = NC * L::RPW;
  static constexpr int RB = S * (int)sizeof(T);
  static constexpr int EMAX = EMAX_;  // multiple of 4, >= TR * max row length + 3
  static constexpr int NSTAGE = NSTAGE_;
  static constexpr int PBYTES = EMAX * RB;
  static constexpr int VBYTES = ((EMAX * (int)sizeof(T) + 127) / 128) * 128;
  static constexpr int RPBYTES = ((TR + 1) * 4 + 15) / 16 * 16 + 64;  // row pointers of the tile
  static constexpr int YBYTES = TR * RB;                              // epilogue operand of reduction 0
  static constexpr int STAGE_BYTES = PBYTES + VBYTES + ((RPBYTES + 127) / 128) * 128 + YBYTES;
  static constexpr int RSM = NC * (FC ? S * S * 2 : 2 * S) * 8;  // red_flush scratch
  static constexpr int YOFF = PBYTES + VBYTES + ((RPBYTES + 127) / 128) * 128;
  static constexpr int DM = 7;                            // column indices fetched DM tiles ahead
  static constexpr int MR = DM + 1;                       // ring slots per producer warp
  static constexpr int CIW = (EMAX / 4 / NP + 1) * 4;     // ints per slot (one chunk)
  static constexpr int SMEM = NSTAGE * STAGE_BYTES + NP * MR * CIW * 4 + (2 * NSTAGE + NP * MR) * 8 + RSM;
};

// a.P must be the base of the tensor map; the value array is padded by 2 elements,
// the column-index and row-pointer arrays by 4 (zeros) — 16-byte bulk copies round
// the ranges up, and a tile's entries are taken from e0 & ~3; rows
// of P must be >= 32 bytes (gather4 destinations 128-byte aligned); an n-vector
// epilogue operand (SUMVEC) needs n * esz to be a multiple of 16.
template <typename T, int S, bool FC, int EMAX, int NSTAGE, int NP = 4>
__global__ void __launch_bounds__(32 * (NP + 8), 1) spmm_tma_kernel(SpmmArgs a, const __grid_constant__ TmaDesc pmap) {
  if (a.done && *a.done) return;
  using L = Lay<T, S>;
  using C = TmaCfg<T, S, FC, EMAX, NSTAGE, NP>;
  constexpr int TR = C::TR, RB = C::RB;
  extern __shared__ __align__(128) unsigned char tsm[];
  unsigned char* stage_base = tsm;
  int* ciring = reinterpret_cast<int*>(tsm + NSTAGE * C::STAGE_BYTES);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(tsm + NSTAGE * C::STAGE_BYTES + NP * C::MR * C::CIW * 4);
  unsigned long long* empty = full + NSTAGE;
  unsigned long long* cifull = empty + NSTAGE;  // [NP][MR]
  double* rsm = reinterpret_cast<double*>(cifull + NP * C::MR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long n = a.n;
  const int* __restrict__ rp = a.row_ptr;
  const int* __restrict__ ci = a.col_idx;
  const long long ntiles = (n + TR - 1) / TR;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&full[i], NP);
      mbar_init(&empty[i], C::NC);
    }
    for (int i = 0; i < NP * C::MR; ++i) mbar_init(&cifull[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int nred = a.nred;
  const int mode0 = nred > 0 ? a.red[0].mode : RED_NONE;
  const int mode1 = nred > 1 ? a.red[1].mode : RED_NONE;
  const T* y0 = reinterpret_cast<const T*>(nred > 0 ? a.red[0].yext : nullptr);
  const T* y1 = reinterpret_cast<const T*>(nred > 1 ? a.red[1].yext : nullptr);
  // bytes per row of reduction 0's operand staged with the tile (0: none)
  const int yrow = (mode0 == RED_NONE || mode0 == RED_NORM2 || mode0 == RED_COLNORM2 || !y0)
                       ? 0 : (mode0 == RED_SUMVEC ? (int)sizeof(T) : RB);
  if (warp < NP) {
    // ---------------- producers ----------------
    // Local tile k is global tile blockIdx.x + k * gridDim.x. Entry bounds of 32
    // tiles are fetched per lane-parallel load, 32 tiles ahead; the column indices
    // of this warp's chunk of tile k + DM are bulk-copied into its ring while tile
    // k is issued, so no register ever waits on a fresh global load.
    const int pw = warp;
    int* ring = ciring + (size_t)pw * C::MR * C::CIW;
    unsigned long long* cif = cifull + pw * C::MR;
    const long long nloc = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto load_batch = [&](long long kb, int& E0, int& E1) {
      const long long kk = kb + lane;
      E0 = E1 = 0;
      if (kk < nloc) {
        const long long t0 = ((long long)blockIdx.x + kk * gridDim.x) * TR;
        E0 = __ldg(rp + t0);
        E1 = __ldg(rp + min(n, t0 + TR));
      }
    };
    int B0c, B1c, B0n, B1n;
    long long kbc = 0;
    load_batch(0, B0c, B1c);
    load_batch(32, B0n, B1n);
    auto bnd = [&](long long kk, int& e0, int& e1) {  // kbc <= kk < kbc + 64
      const int src = (int)(kk - kbc);
      const int a0 = __shfl_sync(0xffffffffu, B0c, src & 31), a1 = __shfl_sync(0xffffffffu, B1c, src & 31);
      const int b0 = __shfl_sync(0xffffffffu, B0n, src & 31), b1 = __shfl_sync(0xffffffffu, B1n, src & 31);
      e0 = src < 32 ? a0 : b0;
      e1 = src < 32 ? a1 : b1;
    };
    // this warp's chunk [g0, g1) of the ngr gather4 groups of a tile
    auto chunk = [&](int ngr, int& g0, int& g1) {
      g0 = pw * ngr / NP;
      g1 = (pw + 1) * ngr / NP;
    };
    auto issue_ci = [&](long long kk) {
      if (kk >= nloc) return;
      int e0, e1;
      bnd(kk, e0, e1);
      const int e0q = e0 & ~3;
      int g0, g1;
      chunk((e1 - e0q + 3) >> 2, g0, g1);
      const unsigned bytes = (unsigned)(g1 - g0) * 16u;
      const int slot = (int)(kk % C::MR);
      if (lane == 0) {
        mbar_expect_tx_arrive(&cif[slot], bytes);
        if (bytes) bulk_g2s(ring + (size_t)slot * C::CIW, ci + e0q + 4 * g0, bytes, &cif[slot]);
      }
    };
    for (int d = 0; d < C::DM; ++d) issue_ci(d);
    for (long long k = 0; k < nloc; ++k) {
      if (k == kbc + 32) {  // slide the bound batches (the next one was loaded 32 tiles ago)
        B0c = B0n;
        B1c = B1n;
        kbc += 32;
        load_batch(kbc + 32, B0n, B1n);
      }
      issue_ci(k + C::DM);
      const long long tile = (long long)blockIdx.x + k * gridDim.x;
      const int st = (int)(k % NSTAGE);
      const unsigned ph = (unsigned)(k / NSTAGE) & 1u;
      int e0, e1;
      bnd(k, e0, e1);
      const int e0q = e0 & ~3;
      const int cnt = e1 - e0q;
      int g0, g1;
      chunk((cnt + 3) >> 2, g0, g1);
      const long long t0 = tile * TR;
      unsigned extra = 0, vbytes = 0, rpbytes = 0, ybytes = 0;
      if (pw == 0) {  // warp 0 also stages the values, row pointers and epilogue operand
        const int rows = (int)min((long long)TR, n - t0);
        vbytes = cnt > 0 ? (unsigned)((cnt * (int)sizeof(T) + 15) & ~15) : 0u;
        rpbytes = (unsigned)(((rows + 1) * 4 + 15) & ~15);
        ybytes = yrow ? (unsigned)((rows * yrow + 15) & ~15) : 0u;
        extra = vbytes + rpbytes + ybytes;
      }
      const int slot = (int)(k % C::MR);
      unsigned char* sp = stage_base + (size_t)st * C::STAGE_BYTES;
      mbar_wait(&empty[st], ph ^ 1u);
      if (lane == 0) {
        mbar_wait(&cif[slot], (unsigned)(k / C::MR) & 1u);  // this chunk's column indices landed
        mbar_expect_tx_arrive(&full[st], (unsigned)(g1 - g0) * 4u * RB + extra);
        const int4* cring = reinterpret_cast<const int4*>(ring + (size_t)slot * C::CIW);
        for (int gi = g0; gi < g1; ++gi) {
          const int4 c = cring[gi - g0];
          tma_gather4(sp + (size_t)gi * 4 * RB, &pmap, 0, c.x, c.y, c.z, c.w, &full[st]);
        }
        if (pw == 0) {
          if (vbytes) bulk_g2s(sp + C::PBYTES, reinterpret_cast<const T*>(a.val) + e0q, vbytes, &full[st]);
          bulk_g2s(sp + C::PBYTES + C::VBYTES, rp + t0, rpbytes, &full[st]);
          if (ybytes) bulk_g2s(sp + C::YOFF, reinterpret_cast<const char*>(y0) + (size_t)t0 * yrow, ybytes, &full[st]);
        }
      }
      __syncwarp();
    }
    return;  // the producer holds no reduction state
  }

  // ---------------- consumers ----------------
  const int cw = warp - NP;
  const int g = lane % L::G;
  const int base = lane - g;
  const unsigned gmask = (L::G == 32) ? 0xffffffffu : (((1u << L::G) - 1u) << base);
  const int rl = cw * L::RPW + lane / L::G;  // row of the tile handled by this lane group
  T* __restrict__ Q = reinterpret_cast<T*>(a.Q);
  const int s = a.s;
  RedAcc<T, S, FC> acc0, acc1;
  red_zero(acc0);
  red_zero(acc1);
  long long tile = blockIdx.x;
  for (int k = 0; tile < ntiles; ++k, tile += gridDim.x) {
    const int st = k % NSTAGE;
    const unsigned ph = (unsigned)(k / NSTAGE) & 1u;
    const long long t0 = tile * TR;
    const long long row = t0 + rl;
    const bool live = row < n;
    const unsigned char* sp = stage_base + (size_t)st * C::STAGE_BYTES;
    const T* vals = reinterpret_cast<const T*>(sp + C::PBYTES);
    const int* rps = reinterpret_cast<const int*>(sp + C::PBYTES + C::VBYTES);
    mbar_wait(&full[st], ph);
    const int e0q = rps[0] & ~3;
    const int b = live ? rps[rl] - e0q : 0;
    const int e = live ? rps[rl + 1] - e0q : 0;
    T yr0[L::EPL];
    T yv0 = Ar<T>::zero();
#pragma unroll
    for (int q = 0; q < L::EPL; ++q) yr0[q] = Ar<T>::zero();
    if (live && yrow) {
      if (mode0 == RED_SUMVEC) yv0 = reinterpret_cast<const T*>(sp + C::YOFF)[rl];
      else row_load_ex_rw<T, S>(reinterpret_cast<const T*>(sp + C::YOFF + (size_t)rl * RB), g, yr0);
    }
    T acc[L::EPL];
#pragma unroll
    for (int q = 0; q < L::EPL; ++q) acc[q] = Ar<T>::zero();
    for (int j = b; j < e; ++j) {
      const T v = vals[j];
      T p[L::EPL];
      row_load_ex_rw<T, S>(reinterpret_cast<const T*>(sp + (size_t)j * RB), g, p);  // shared memory
#pragma unroll
      for (int q = 0; q < L::EPL; ++q) acc[q] = Ar<T>::fma(v, p[q], acc[q]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // every smem read of this stage is done
    if (live) {
      row_store_ex<T, S>(Q + (size_t)row * S, g, acc);
      if (mode0 != RED_NONE) red_dispatch_row<T, S, FC>(mode0, acc0, acc, yr0, yv0, base, s, gmask);
      if (mode1 != RED_NONE) {
        T y[L::EPL];
        T yv = Ar<T>::zero();
#pragma unroll
        for (int q = 0; q < L::EPL; ++q) y[q] = Ar<T>::zero();
        if (mode1 == RED_SUMVEC) yv = y1[row];
        else if (mode1 != RED_NORM2 && mode1 != RED_COLNORM2) row_load_ex_rw<T, S>(y1 + (size_t)row * S, g, y);
        red_dispatch_row<T, S, FC>(mode1, acc1, acc, y, yv, base, s, gmask);
      }
    }
  }
  // reductions over the consumer warps only (named barrier 1)
  __syncwarp();
  if (nred > 0) red_dispatch_flush<T, S, FC>(mode0, acc0, a.partials, a.pstride, a.red[0].poff, s, rsm, NP, C::NC, 1);
  if (nred > 1) red_dispatch_flush<T, S, FC>(mode1, acc1, a.partials, a.pstride, a.red[1].poff, s, rsm, NP, C::NC, 1);
}

}  // namespace srk
