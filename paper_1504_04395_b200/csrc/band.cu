// band.cu — block SpMM Q = A P for banded operators (the stencils of configs 1-3),
// the "SELL-C-σ slot" of operator preparation for regular operators.
//
// a0 detects operators whose nonzeros lie on K <= 8 diagonals j - i = d_k (the 5- and
// 7-point convection-diffusion stencils) and stores them as K diagonals of n
// values each (zero where a row has no entry on that diagonal; summation order = the CSR
// order, ascending column). The product then needs, for a tile of TR consecutive rows,
// only K CONTIGUOUS windows of P (rows r + d_k .. r + d_k + TR): each nonzero a_ij is
// still applied to the s contiguous values of P row j, but the rows arrive as
// bulk copies instead of 7 scattered 128-byte gathers per row — the SpMM's limit on
// config 3 was the L2->SM gather latency, not DRAM bytes.
//
// Layout per CTA (1 CTA / SM, persistent): one producer warp (lane 0 issues
// cp.async.bulk copies into a D-stage mbarrier ring) and NW consumer warps.
//   * near diagonals (|d| <= H): a shared-memory RING of P rows indexed by row mod CAP
//     (CAP = D TR + 2H). A CTA walks a chunk of consecutive tiles, so consecutive tiles
//     share all but TR rows of their near windows: each tile loads TR new rows.
//   * far diagonals (|d| > H, e.g. +-n^(2/3) on the 3D grid): one TR-row window per tile.
//   * the K diagonal slices of the tile (TR values each).
// Chunks (CT tiles) are dealt round-robin over the CTAs, so all SMs sweep the rows
// together: a P row's near and far uses happen within one sweep front (~grid*CT*TR rows)
// and its re-reads are L2 hits.
// Epilogue: the fused non-FULL reductions of block_kernels.cuh (red_acc / red_flush).
#include <climits>
#include <vector>

#include "block_kernels.cuh"
#include "engine.h"

namespace srk {

constexpr int BAND_KMAX = 8;
constexpr int BAND_FMAX = 3;  // far diagonals staged per tile
constexpr int BAND_DMAX = 8;  // pipeline stages (runtime D <= DMAX)
constexpr int BAND_NWMAX = 16;  // consumer warps: 16 (1 CTA / SM) or 8 (2 CTAs / SM)

struct BandOffs {
  long long d[8];
};

struct BandArgs {
  const void* dia;  // the K diagonals row-major: [npad][K] (zero-padded)
  long long npad;
  int K;
  int off[BAND_KMAX];   // ascending diagonal offsets d_k
  int far_slot[BAND_KMAX];  // -1: near (ring), else far window index
  int H;                // near half-width (rows)
  int cap;              // ring capacity (rows)
  int D;                // pipeline stages
  int tr;               // rows per tile (<= BandCfg::TR)
  int ct;               // tiles per chunk
  const void* P;
  void* Q;
  long long n;
  Red red[2];
  int nred;
  int ystage[2];        // reduction q's Y operand staged per tile: 0 none, 1 vector (SUMVEC), 2 rows
  double* partials;
  int pstride;
  const int* done;
  int xflags;  // measurement knobs: 1 skip the arithmetic, 2 skip the P windows
};

__device__ __forceinline__ unsigned bsmem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bwait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "BW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra BW_%=;\n\t}" ::"r"(bsmem(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bcopy(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   bsmem(dst)),
               "l"(src), "r"(bytes), "r"(bsmem(bar))
               : "memory");
}

template <typename T, int S>
struct BandCfg {
  static constexpr int RB = S * (int)sizeof(T);                // bytes per row (multiple of 16)
  static constexpr int TR = (8192 / RB < 256) ? 8192 / RB : 256;  // rows per tile: <= 8 KB windows
};
// near half-width for a row size: the 2H-row ring margin stays within ~96 KB
inline int band_hcap(int rb) { return 49152 / rb; }

template <typename T, int S>
size_t band_smem(int K, int nfar, int cap, int ny, int D, int tr) {
  using C = BandCfg<T, S>;
  return 128 + (size_t)D * K * tr * sizeof(T) + (size_t)D * nfar * tr * C::RB + (size_t)cap * C::RB +
         (size_t)D * ny * tr * C::RB;
}

template <typename T, int S, int KK, int BAND_NW>
__global__ void __launch_bounds__(32 * (BAND_NW + 1), 16 / BAND_NW) band_kernel(BandArgs a) {
  if (a.done && *a.done) return;
  using L = Lay<T, S>;
  using C = BandCfg<T, S>;
  const int TR = a.tr;
  const int BAND_D = a.D;
  extern __shared__ __align__(128) unsigned char bsm[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(bsm);
  unsigned long long* empty = full + BAND_DMAX;
  int nfar = 0;
  for (int k = 0; k < a.K; ++k) nfar += a.far_slot[k] >= 0 ? 1 : 0;
  T* vals = reinterpret_cast<T*>(bsm + 128);                                  // [D][K][TR]
  T* farb = vals + (size_t)BAND_D * a.K * TR;                               // [D][nfar][TR][S]
  T* ring = farb + (size_t)BAND_D * nfar * TR * S;                          // [cap][S]
  T* ybuf = ring + (size_t)a.cap * S;  // [D][2 slots][TR][S]: staged Y rows / vector entries of the reductions
  int ny = 0;
  int yslot[2] = {-1, -1};
  for (int q = 0; q < a.nred && q < 2; ++q)
    if (a.ystage[q]) yslot[q] = ny++;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long n = a.n;
  const long long ntiles = (n + TR - 1) / TR;
  const long long nchunks = (ntiles + a.ct - 1) / a.ct;
  // zero the staged P rows once (rows outside [0, n) are never loaded; their diagonal
  // values are zero, so only finiteness matters)
  {
    double* z = reinterpret_cast<double*>(farb);
    const size_t nd = ((size_t)BAND_D * nfar * TR * S + (size_t)a.cap * S) * sizeof(T) / 8;
    for (size_t i = threadIdx.x; i < nd; i += blockDim.x) z[i] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the bulk copies into the same smem
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < BAND_D; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bsmem(full + q)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bsmem(empty + q)), "r"(BAND_NW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // Lane roles (a handful of instructions per tile per lane, no divisions in the tile
    // loop): lanes 0-1 the new near rows (two pieces at the ring wrap), lanes 2.. the far
    // windows, lane 8 the tile's diagonal values, lanes 9-10 the staged Y operands. The
    // expected byte count is a warp sum of the lanes' jobs.
    const char* P = reinterpret_cast<const char*>(a.P);
    const char* dia = reinterpret_cast<const char*>(a.dia);
    long long foff = 0;  // far window offset of this lane (lanes 2 .. 2 + nfar - 1)
    int fslot = -1;
    if (lane >= 2 && lane < 2 + nfar)
      for (int k = 0; k < a.K; ++k)
        if (a.far_slot[k] == lane - 2) {
          foff = a.off[k];
          fslot = lane - 2;
        }
    const int yq = lane - 9;
    const bool ylane = (yq == 0 || yq == 1) && yslot[yq < 0 ? 0 : (yq > 1 ? 1 : yq)] >= 0;
    long long g = 0;
    int st = 0;
    unsigned ph = 0;  // parity of stage st's current use
    long long nnext = 0;  // near rows: next row to load and its ring position
    int npos = 0;
    for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
      const long long t0 = ch * a.ct;
      const long long t1 = (t0 + a.ct < ntiles) ? t0 + a.ct : ntiles;
      for (long long t = t0; t < t1; ++t, ++g) {
        if (g >= BAND_D) bwait(empty + st, ph ^ 1u);  // the previous use of this stage was consumed
        if (t == t0)  // a new chunk rewrites arbitrary ring positions: drain every tile in flight
          for (int j = 1; j < BAND_D && j <= g; ++j) {
            const int sj = (st - j + BAND_D) % BAND_D;
            const unsigned pj = (sj < st) ? ph : (ph ^ 1u);  // tile g - j's use parity
            bwait(empty + sj, pj);
          }
        const long long r = t * TR;
        unsigned myb = 0;
        const void* src = nullptr;
        void* dst = nullptr;
        if (lane < 2) {
          if (t == t0) {
            nnext = r - a.H < 0 ? 0 : r - a.H;
            npos = (int)(nnext % a.cap);
          }
          long long hi = r + TR + a.H;
          if (hi > n) hi = n;
          const long long lo = nnext;
          if (hi > lo) {
            const int first = (int)((hi - lo) < (long long)(a.cap - npos) ? (hi - lo) : (long long)(a.cap - npos));
            if (lane == 0) {
              myb = (unsigned)(first * C::RB);
              dst = ring + (size_t)npos * S;
              src = P + (size_t)lo * C::RB;
            } else if (hi - lo > first) {
              myb = (unsigned)((hi - lo - first) * C::RB);
              dst = ring;
              src = P + (size_t)(lo + first) * C::RB;
            }
            npos += (int)(hi - lo);
            if (npos >= a.cap) npos -= a.cap;
            nnext = hi;
          }
        } else if (fslot >= 0) {
          long long flo = r + foff, fhi = r + foff + TR;
          if (flo < 0) flo = 0;
          if (fhi > n) fhi = n;
          if (fhi > flo) {
            myb = (unsigned)((fhi - flo) * C::RB);
            dst = farb + (((size_t)st * nfar + fslot) * TR + (flo - (r + foff))) * S;
            src = P + (size_t)flo * C::RB;
          }
        } else if (lane == 8) {
          myb = (unsigned)(TR * a.K * sizeof(T));
          dst = vals + (size_t)st * a.K * TR;
          src = dia + (size_t)r * a.K * sizeof(T);
        } else if (ylane) {
          const long long rows = (n - r < TR) ? n - r : TR;
          T* yd = ybuf + ((size_t)st * ny + yslot[yq]) * TR * S;
          const T* ys = reinterpret_cast<const T*>(a.red[yq].yext);
          dst = yd;
          if (a.ystage[yq] == 2) {
            myb = (unsigned)(rows * C::RB);
            src = ys + (size_t)r * S;
          } else {  // vector entries: the 16-byte part by the copy engine, an odd tail entry here
            const long long even = (rows * (long long)sizeof(T)) / 16 * 16 / (long long)sizeof(T);
            myb = (unsigned)(even * sizeof(T));
            src = ys + r;
            if (even < rows) yd[even] = ys[r + even];
          }
        }
        if (a.xflags & 2) {
          if (lane < 2 + nfar) myb = 0;
        }
        const unsigned bytes = __reduce_add_sync(0xffffffffu, myb);
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bsmem(full + st)), "r"(bytes)
                       : "memory");
        __syncwarp();
        if (myb) bcopy(dst, src, myb, full + st);
        if (++st == BAND_D) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  // Every staged P row is addressed as a row slot of `farb`: far window f of stage st at
  // st*nfar*TR + f*TR + rr, the ring row of position pos at D*nfar*TR + pos. Per tile and
  // diagonal one base slot (and, for the ring, the wrap point) is formed incrementally —
  // no divisions inside the tile loop.
  const int cw = warp - 1;
  const int g = lane % L::G;
  const int rr0 = cw * L::RPW + lane / L::G;
  RedAcc<T, S, false> acc0, acc1;
  red_zero<T, S, false>(acc0);
  red_zero<T, S, false>(acc1);
  const int m0 = a.nred > 0 ? a.red[0].mode : RED_NONE;
  const int m1 = a.nred > 1 ? a.red[1].mode : RED_NONE;
  const int ringbase = BAND_D * nfar * TR;
  int dmod[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dmod[k] = k < a.K ? (int)(((long long)a.off[k] % a.cap + a.cap) % a.cap) : 0;
  int st = 0;
  unsigned ph = 0;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long t0 = ch * a.ct;
    const long long t1 = (t0 + a.ct < ntiles) ? t0 + a.ct : ntiles;
    int rpos = (int)((t0 * TR) % a.cap);
    for (long long t = t0; t < t1; ++t) {
      bwait(full + st, ph);
      const long long r = t * TR;
      const T* sv = vals + (size_t)st * a.K * TR;
      int kb[KK], ke[KK];
#pragma unroll
      for (int k = 0; k < KK; ++k) {
        if (k < a.K && a.far_slot[k] < 0) {
          int p0 = rpos + dmod[k];
          if (p0 >= a.cap) p0 -= a.cap;
          kb[k] = ringbase + p0;
          ke[k] = ringbase + a.cap;
        } else {
          kb[k] = (st * nfar + (k < a.K ? a.far_slot[k] : 0)) * TR;
          ke[k] = INT_MAX;
        }
      }
      const T* sy = ybuf + (size_t)st * ny * TR * S;
      for (int rr = rr0; rr < TR; rr += BAND_NW * L::RPW) {
        const long long i = r + rr;
        T x[L::EPL];
#pragma unroll
        for (int e = 0; e < L::EPL; ++e) x[e] = Ar<T>::zero();
#pragma unroll
        for (int k = 0; k < KK; ++k) {
          if (KK == BAND_KMAX && k >= a.K) break;
          if (a.xflags & 1) break;
          const T v = sv[rr * a.K + k];
          int pos = kb[k] + rr;
          if (pos >= ke[k]) pos -= a.cap;
          T p[L::EPL];
          row_load_ex_rw<T, S>(farb + (size_t)pos * S, g, p);
#pragma unroll
          for (int e = 0; e < L::EPL; ++e) x[e] = Ar<T>::fma(v, p[e], x[e]);
        }
        if (i < n) {
          row_store_ex_cs<T, S>(reinterpret_cast<T*>(a.Q) + (size_t)i * S, g, x);
          if (m0 != RED_NONE || m1 != RED_NONE) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int m = q ? m1 : m0;
              if (m == RED_NONE) continue;
              const int yk = red_ykind(m);
              T y[L::EPL];
              T yv = Ar<T>::zero();
              if (yk == 1) yv = sy[(size_t)yslot[q] * TR * S + rr];
              if (yk == 2) row_load_ex_rw<T, S>(sy + ((size_t)yslot[q] * TR + rr) * S, g, y);
              T yy[L::EPL];
#pragma unroll
              for (int e = 0; e < L::EPL; ++e) yy[e] = yk == 0 ? x[e] : (yk == 1 ? yv : y[e]);
              if (q == 0) red_acc<T, S, false>(acc0, x, yy);
              else red_acc<T, S, false>(acc1, x, yy);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bsmem(empty + st)) : "memory");
      if (++st == BAND_D) {
        st = 0;
        ph ^= 1u;
      }
      rpos += TR;
      if (rpos >= a.cap) rpos -= a.cap;
    }
  }
  if (a.nred > 0) {
    double* red_smem = reinterpret_cast<double*>(vals);  // the stages are no longer read
    asm volatile("bar.sync 1, %0;" ::"r"(BAND_NW * 32) : "memory");
    red_dispatch_flush<T, S, false>(m0, acc0, a.partials, a.pstride, a.red[0].poff, S, red_smem, 1, BAND_NW, 1);
    if (a.nred > 1)
      red_dispatch_flush<T, S, false>(m1, acc1, a.partials, a.pstride, a.red[1].poff, S, red_smem, 1, BAND_NW, 1);
  }
}

// ---------------------------------------------------------------------------
// Variant fed by cp.async (LDGSTS, 16 B per lane) from all warps instead of the bulk-copy
// engine: measured on B200, the per-SM bulk-copy path sustained only ~12 B/clk here
// (time per tile independent of the pipeline depth and of the CTA count per SM), while
// the LSU path carries the CSR kernel's 21 B/clk. Same smem layout and arithmetic; per
// tile: all threads issue the 16-byte pieces of tile g + D - 1, one commit group per tile,
// wait for tile g's group, barrier, compute, barrier. The pipeline is re-primed per chunk.
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(bsmem(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_dyn(int pending) {
  switch (pending) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
    case 4: asm volatile("cp.async.wait_group 4;\n" ::: "memory"); break;
    case 5: asm volatile("cp.async.wait_group 5;\n" ::: "memory"); break;
    case 6: asm volatile("cp.async.wait_group 6;\n" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 7;\n" ::: "memory"); break;
  }
}

template <typename T, int S, int KK, int NWT>
__global__ void __launch_bounds__(32 * NWT, 1) band_cp_kernel(BandArgs a) {
  if (a.done && *a.done) return;
  using L = Lay<T, S>;
  using C = BandCfg<T, S>;
  constexpr int U = C::RB / 16;  // 16-byte pieces per row
  const int TR = a.tr;
  const int D = a.D;
  extern __shared__ __align__(128) unsigned char bsm[];
  int nfar = 0;
  for (int k = 0; k < a.K; ++k) nfar += a.far_slot[k] >= 0 ? 1 : 0;
  T* vals = reinterpret_cast<T*>(bsm + 128);
  T* farb = vals + (size_t)D * a.K * TR;
  T* ring = farb + (size_t)D * nfar * TR * S;
  T* ybuf = ring + (size_t)a.cap * S;
  int ny = 0;
  int yslot[2] = {-1, -1};
  for (int q = 0; q < a.nred && q < 2; ++q)
    if (a.ystage[q]) yslot[q] = ny++;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const long long n = a.n;
  const long long ntiles = (n + TR - 1) / TR;
  const long long nchunks = (ntiles + a.ct - 1) / a.ct;
  {
    double* z = reinterpret_cast<double*>(farb);
    const size_t nd = ((size_t)D * nfar * TR * S + (size_t)a.cap * S) * sizeof(T) / 8;
    for (size_t i = tid; i < nd; i += nth) z[i] = 0.0;
  }
  __syncthreads();
  const char* P = reinterpret_cast<const char*>(a.P);
  const char* dia = reinterpret_cast<const char*>(a.dia);
  // the 16-byte pieces of tile t (first = chunk's first tile) into stage st; this thread's share
  auto issue = [&](long long t, bool first, int st) {
    const long long r = t * TR;
    const long long rows = (n - r < TR) ? n - r : TR;
    long long lo = first ? r - a.H : r + a.H;
    long long hi = r + TR + a.H;
    if (lo < 0) lo = 0;
    if (hi > n) hi = n;
    if (hi > lo) {
      const int p0 = (int)(lo % a.cap);
      const long long cnt = (hi - lo) * U;
      for (long long u = tid; u < cnt; u += nth) {
        const long long rw = u / U;
        int pos = p0 + (int)rw;
        if (pos >= a.cap) pos -= a.cap;
        cpa16(reinterpret_cast<char*>(ring + (size_t)pos * S) + (u % U) * 16, P + (size_t)(lo + rw) * C::RB + (u % U) * 16);
      }
    }
    for (int k = 0; k < a.K; ++k)
      if (a.far_slot[k] >= 0) {
        long long flo = r + a.off[k], fhi = r + a.off[k] + TR;
        if (flo < 0) flo = 0;
        if (fhi > n) fhi = n;
        if (fhi <= flo) continue;
        char* d0 = reinterpret_cast<char*>(farb + (((size_t)st * nfar + a.far_slot[k]) * TR + (flo - (r + a.off[k]))) * S);
        const char* s0 = P + (size_t)flo * C::RB;
        const long long cnt = (fhi - flo) * U;
        for (long long u = tid; u < cnt; u += nth) cpa16(d0 + u * 16, s0 + u * 16);
      }
    {
      char* d0 = reinterpret_cast<char*>(vals + (size_t)st * a.K * TR);
      const char* s0 = dia + (size_t)r * a.K * sizeof(T);
      const int cnt = TR * a.K * (int)sizeof(T) / 16;
      for (int u = tid; u < cnt; u += nth) cpa16(d0 + u * 16, s0 + u * 16);
    }
    for (int q = 0; q < 2; ++q)
      if (yslot[q] >= 0) {
        T* yd = ybuf + ((size_t)st * ny + yslot[q]) * TR * S;
        const T* ys = reinterpret_cast<const T*>(a.red[q].yext);
        if (a.ystage[q] == 2) {
          const long long cnt = rows * U;
          for (long long u = tid; u < cnt; u += nth)
            cpa16(reinterpret_cast<char*>(yd) + u * 16, reinterpret_cast<const char*>(ys + (size_t)r * S) + u * 16);
        } else {
          const long long even = (rows * (long long)sizeof(T)) / 16 * 16 / (long long)sizeof(T);
          const long long cnt = even * (long long)sizeof(T) / 16;
          for (long long u = tid; u < cnt; u += nth)
            cpa16(reinterpret_cast<char*>(yd) + u * 16, reinterpret_cast<const char*>(ys + r) + u * 16);
          if (even < rows && tid == 0) yd[even] = ys[r + even];
        }
      }
  };

  const int g = lane % L::G;
  const int rr0 = warp * L::RPW + lane / L::G;
  RedAcc<T, S, false> acc0, acc1;
  red_zero<T, S, false>(acc0);
  red_zero<T, S, false>(acc1);
  const int m0 = a.nred > 0 ? a.red[0].mode : RED_NONE;
  const int m1 = a.nred > 1 ? a.red[1].mode : RED_NONE;
  const int ringbase = D * nfar * TR;
  int dmod[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dmod[k] = k < a.K ? (int)(((long long)a.off[k] % a.cap + a.cap) % a.cap) : 0;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long t0 = ch * a.ct;
    const long long t1 = (t0 + a.ct < ntiles) ? t0 + a.ct : ntiles;
    const int nt = (int)(t1 - t0);
    // prologue: tiles 0 .. D-2 of the chunk (one commit group each)
    for (int j = 0; j < D - 1; ++j) {
      if (j < nt) issue(t0 + j, j == 0, j % D);
      cpa_commit();
    }
    int rpos = (int)((t0 * TR) % a.cap);
    for (int j = 0; j < nt; ++j) {
      const int st = j % D;
      if (j + D - 1 < nt) issue(t0 + j + D - 1, false, (j + D - 1) % D);
      cpa_commit();
      cpa_wait_dyn(D - 1);  // tile j's group (the D - 1 younger ones may still fly)
      __syncthreads();
      const long long r = (t0 + j) * TR;
      const T* sv = vals + (size_t)st * a.K * TR;
      int kb[KK], ke[KK];
#pragma unroll
      for (int k = 0; k < KK; ++k) {
        if (k < a.K && a.far_slot[k] < 0) {
          int p0 = rpos + dmod[k];
          if (p0 >= a.cap) p0 -= a.cap;
          kb[k] = ringbase + p0;
          ke[k] = ringbase + a.cap;
        } else {
          kb[k] = (st * nfar + (k < a.K ? a.far_slot[k] : 0)) * TR;
          ke[k] = INT_MAX;
        }
      }
      const T* sy = ybuf + (size_t)st * ny * TR * S;
      for (int rr = rr0; rr < TR; rr += NWT * L::RPW) {
        const long long i = r + rr;
        T x[L::EPL];
#pragma unroll
        for (int e = 0; e < L::EPL; ++e) x[e] = Ar<T>::zero();
#pragma unroll
        for (int k = 0; k < KK; ++k) {
          if (KK == BAND_KMAX && k >= a.K) break;
          const T v = sv[rr * a.K + k];
          int pos = kb[k] + rr;
          if (pos >= ke[k]) pos -= a.cap;
          T p[L::EPL];
          row_load_ex_rw<T, S>(farb + (size_t)pos * S, g, p);
#pragma unroll
          for (int e = 0; e < L::EPL; ++e) x[e] = Ar<T>::fma(v, p[e], x[e]);
        }
        if (i < n) {
          row_store_ex_cs<T, S>(reinterpret_cast<T*>(a.Q) + (size_t)i * S, g, x);
          if (m0 != RED_NONE || m1 != RED_NONE) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int m = q ? m1 : m0;
              if (m == RED_NONE) continue;
              const int yk = red_ykind(m);
              T y[L::EPL];
              T yv = Ar<T>::zero();
              if (yk == 1) yv = sy[(size_t)yslot[q] * TR * S + rr];
              if (yk == 2) row_load_ex_rw<T, S>(sy + ((size_t)yslot[q] * TR + rr) * S, g, y);
              T yy[L::EPL];
#pragma unroll
              for (int e = 0; e < L::EPL; ++e) yy[e] = yk == 0 ? x[e] : (yk == 1 ? yv : y[e]);
              if (q == 0) red_acc<T, S, false>(acc0, x, yy);
              else red_acc<T, S, false>(acc1, x, yy);
            }
          }
        }
      }
      __syncthreads();  // stage st and the oldest ring rows may be refilled now
      rpos += TR;
      if (rpos >= a.cap) rpos -= a.cap;
    }
    cpa_wait_dyn(0);
  }
  if (a.nred > 0) {
    double* red_smem = reinterpret_cast<double*>(vals);
    __syncthreads();
    red_dispatch_flush<T, S, false>(m0, acc0, a.partials, a.pstride, a.red[0].poff, S, red_smem);
    if (a.nred > 1) red_dispatch_flush<T, S, false>(m1, acc1, a.partials, a.pstride, a.red[1].poff, S, red_smem);
  }
}

// ---------------------------------------------------------------------------
// Plane-marching SpMM for the 7-point pattern (round 2, session 3). Operators whose
// diagonals are exactly {-F, -m, -1, 0, +1, +m, +F} with F a multiple of m (the 3D
// convection-diffusion stencils of configs 2 / 3, and their adjoints) are
// multiplied as a 2.5D sweep: row i = z F + y m + x is point (x, y) of plane z. A work item
// is a TX x TY tile of (x, y) points and a segment of ZL planes; the CTA marches z through
// the segment keeping a ring of NB plane WINDOWS in shared memory, each window = the
// (TX + 2) x (TY + 2) rows around the tile (rows addressed by index, so the +-1 / +-m
// neighbours of every tile row lie inside the window whatever the matrix's values at the
// grid edges), filled by TY + 2 bulk copies of TX + 2 consecutive rows. The -F neighbour of
// a row is the centre row of the previous plane, held in registers from the previous step;
// the +F neighbour is the centre row of the next window. So every P row is copied into shared
// memory (TX+2)(TY+2)/(TX TY) ~ 1.4 times instead of the band kernel's three times (ring +
// two far windows) — the far windows' L2 -> SM traffic was the band kernel's limit on
// config 3. Concurrent items are neighbouring tiles of one plane segment, so the halo rows
// a tile shares with its neighbours are L2 hits. Summation order per row = ascending offset
// (= ascending column, the CSR order), as in band_kernel.
constexpr int PL_NBMAX = 4;   // plane windows in flight (runtime NB <= 4)
constexpr int PL_TX = 32;     // tile width (points along x)
constexpr int PL_TY = 6;      // tile height (lines along y)
constexpr int PL_K = 7;

struct PlaneArgs {
  const void* dia;  // [npad][7] diagonal values, row-major
  const void* P;
  void* Q;
  long long n, F;
  int m, ny;        // points per line, lines per plane (F = m ny)
  long long nz;     // planes (ceil(n / F))
  int ntx, nty;     // tiles per plane along x / y
  int zl, nzs;      // planes per segment, segments
  long long nitems; // ntx * nty * nzs
  int NB;           // ring depth
  Red red[2];
  int nred;
  int ystage[2];    // 1: SUMVEC vector staged per plane
  double* partials;
  int pstride;
  const int* done;
};

template <typename T, int S>
struct PlaneCfg {
  static constexpr int RB = S * (int)sizeof(T);
  static constexpr int WX = PL_TX + 2, WY = PL_TY + 2;
  static constexpr int WR = WX * WY;                       // rows per window
  static constexpr int VL = (PL_TX + 2) * PL_K;            // values per line slot (+2: alignment shift)
  static constexpr int YL = PL_TX + 2;                     // vector entries per line slot
  static constexpr size_t WIN = (size_t)WR * RB;           // bytes per window
  static constexpr size_t VAL = (size_t)PL_TY * VL * sizeof(T);
  static constexpr size_t YV = (size_t)PL_TY * YL * sizeof(T);
};

template <typename T, int S>
size_t plane_smem(int NB, int ny) {
  using C = PlaneCfg<T, S>;
  return 128 + (size_t)NB * (C::WIN + C::VAL + (size_t)ny * C::YV);
}

// YROW: instance with row-operand reductions (TRACE / DIAG); the plain / NORM2 / SUMVEC instance
// keeps its register budget (config 3's SpMM + eGl sum: 92 registers, 0.87 ms; with the row-operand
// code compiled in: 96 registers, 0.90 ms)
template <typename T, int S, int NW, bool YROW>
__global__ void __launch_bounds__(32 * (NW + 1), 1) band_plane_kernel(PlaneArgs a) {
  if (a.done && *a.done) return;
  using L = Lay<T, S>;
  using C = PlaneCfg<T, S>;
  constexpr int TROWS = PL_TX * PL_TY;
  constexpr int SLOTS = NW * L::RPW;
  constexpr int RPL = (TROWS + SLOTS - 1) / SLOTS;  // tile rows per lane group
  const int NB = a.NB;
  extern __shared__ __align__(128) unsigned char bsm[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(bsm);
  unsigned long long* empty = full + PL_NBMAX;
  T* win = reinterpret_cast<T*>(bsm + 128);                      // [NB][WY][WX][S]
  T* vals = win + (size_t)NB * C::WR * S;                        // [NB][TY][VL]
  T* ybuf = vals + (size_t)NB * PL_TY * C::VL;                   // [NB][ny][TY][YL]
  int ny = 0;
  int yslot[2] = {-1, -1};
  for (int q = 0; q < a.nred && q < 2; ++q)
    if (a.ystage[q]) yslot[q] = ny++;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long n = a.n, F = a.F;
  const int m = a.m;
  const long long ntile = (long long)a.ntx * a.nty;
  {  // windows start finite (clamped rows are never copied; their diagonal values are zero)
    double* z = reinterpret_cast<double*>(win);
    const size_t nd = (size_t)NB * C::WIN / 8;
    for (size_t i = threadIdx.x; i < nd; i += blockDim.x) z[i] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < NB; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bsmem(full + q)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bsmem(empty + q)), "r"(NW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // per window: TY + 2 P line segments; for computed planes also TY value segments and TY
    // vector segments per staged reduction — one copy per lane (looping for wide tiles)
    const char* P = reinterpret_cast<const char*>(a.P);
    const char* dia = reinterpret_cast<const char*>(a.dia);
    constexpr int ESZ = (int)sizeof(T);
    long long g = 0;
    int st = 0;
    unsigned ph = 0;
    for (long long it = blockIdx.x; it < a.nitems; it += gridDim.x) {
      const long long zs0 = (it / ntile) * a.zl;
      const int tile = (int)(it % ntile);
      const int y0 = (tile / a.ntx) * PL_TY, x0 = (tile % a.ntx) * PL_TX;
      const long long ze = (zs0 + a.zl < a.nz) ? zs0 + a.zl : a.nz;
      for (long long p = zs0 - 1; p <= ze; ++p, ++g) {
        if (g >= NB) bwait(empty + st, ph ^ 1u);
        const bool comp = p >= zs0 && p < ze;
        const int ncp = (PL_TY + 2) + (comp ? PL_TY * (1 + ny) : 0);
        unsigned myb = 0;
        // descriptors (at most two per lane for the tile sizes used)
        const void* src[2] = {nullptr, nullptr};
        void* dst[2] = {nullptr, nullptr};
        unsigned by[2] = {0, 0};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = lane + 32 * u;
          if (c >= ncp) break;
          if (c < PL_TY + 2) {  // P line segment j = c of plane p
            const long long lo = p * F + (long long)(y0 - 1 + c) * m + x0 - 1;
            long long clo = lo < 0 ? 0 : lo, chi = lo + C::WX;
            if (chi > n) chi = n;
            if (chi > clo) {
              by[u] = (unsigned)((chi - clo) * C::RB);
              src[u] = P + (size_t)clo * C::RB;
              dst[u] = win + ((size_t)st * C::WR + (size_t)c * C::WX + (size_t)(clo - lo)) * S;
            }
          } else {
            const int c2 = c - (PL_TY + 2);
            const int yl = c2 % PL_TY, kind = c2 / PL_TY;  // 0 values, 1.. staged vectors
            if (y0 + yl < a.ny) {
              const long long i0 = p * F + (long long)(y0 + yl) * m + x0;
              long long cnt = m - x0 < PL_TX ? m - x0 : PL_TX;
              if (i0 + cnt > n) cnt = n - i0;
              if (cnt > 0) {
                const long long a0 = (ESZ == 8) ? (i0 & ~1LL) : i0;  // 16-byte aligned source row
                const long long rows = cnt + (i0 - a0);
                if (kind == 0) {
                  by[u] = (unsigned)(((rows * PL_K * ESZ) + 15) / 16 * 16);
                  src[u] = dia + (size_t)a0 * PL_K * ESZ;
                  dst[u] = vals + ((size_t)st * PL_TY + yl) * C::VL;
                } else {
                  int q = 0;
                  for (int qq = 0; qq < 2; ++qq)
                    if (yslot[qq] == kind - 1) q = qq;
                  by[u] = (unsigned)(((rows * ESZ) + 15) / 16 * 16);
                  src[u] = reinterpret_cast<const char*>(a.red[q].yext) + (size_t)a0 * ESZ;
                  dst[u] = ybuf + (((size_t)st * ny + (kind - 1)) * PL_TY + yl) * C::YL;
                }
              }
            }
          }
          myb += by[u];
        }
        const unsigned bytes = __reduce_add_sync(0xffffffffu, myb);
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bsmem(full + st)), "r"(bytes)
                       : "memory");
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (by[u]) bcopy(dst[u], src[u], by[u], full + st);
        if (++st == NB) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int cw = warp - 1;
  const int g = lane % L::G;
  const int slot = cw * L::RPW + lane / L::G;
  RedAcc<T, S, false> acc0, acc1;
  red_zero<T, S, false>(acc0);
  red_zero<T, S, false>(acc1);
  const int m0 = a.nred > 0 ? a.red[0].mode : RED_NONE;
  const int m1 = a.nred > 1 ? a.red[1].mode : RED_NONE;
  // row operands (TRACE / DIAG: acc += conj(y_row) .* q_row): the product's own input row is the
  // centre row already in registers (Gl-BiCGStab's <A S, S>); the rows of one external block
  // (<A P, R~>) are requested at the top of each plane step, ahead of the window wait
  int qext = -1;
  if constexpr (YROW) {
    if (m0 != RED_NONE && red_ykind(m0) == 2 && a.red[0].yext != a.P) qext = 0;
    if (m1 != RED_NONE && red_ykind(m1) == 2 && a.red[1].yext != a.P) qext = 1;
  }
  const T* yext = qext >= 0 ? reinterpret_cast<const T*>(a.red[qext].yext) : nullptr;
  int st = 0;
  unsigned ph = 0;
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bsmem(empty + st)) : "memory");
    if (++st == NB) {
      st = 0;
      ph ^= 1u;
    }
  };
  for (long long it = blockIdx.x; it < a.nitems; it += gridDim.x) {
    const long long zs0 = (it / ntile) * a.zl;
    const int tile = (int)(it % ntile);
    const int y0 = (tile / a.ntx) * PL_TY, x0 = (tile % a.ntx) * PL_TX;
    const long long ze = (zs0 + a.zl < a.nz) ? zs0 + a.zl : a.nz;
    // this lane group's tile rows: (yl, xl) and the window offset of their centre row
    int woff[RPL];
    bool live[RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int rr = slot + k * SLOTS;
      const int yl = rr / PL_TX, xl = rr % PL_TX;
      live[k] = rr < TROWS && y0 + yl < a.ny && x0 + xl < m;
      woff[k] = rr < TROWS ? ((yl + 1) * C::WX + xl + 1) * S : (C::WX + 1) * S;  // (idle slots read row 0)
    }
    T prev[RPL][L::EPL], cur[RPL][L::EPL];
    // window zs0 - 1: its centre rows are the -F neighbours of plane zs0
    bwait(full + st, ph);
    {
      const T* w = win + (size_t)st * C::WR * S;
#pragma unroll
      for (int k = 0; k < RPL; ++k) row_load_ex_rw<T, S>(w + woff[k], g, prev[k]);
    }
    release();
    bwait(full + st, ph);  // window zs0: centre rows
    {
      const T* w = win + (size_t)st * C::WR * S;
#pragma unroll
      for (int k = 0; k < RPL; ++k) row_load_ex_rw<T, S>(w + woff[k], g, cur[k]);
    }
    for (long long z = zs0; z < ze; ++z) {
      const int cs = st;
      int ns = st + 1;
      unsigned nph = ph;
      if (ns == NB) {
        ns = 0;
        nph ^= 1u;
      }
      T yr[YROW ? RPL : 1][L::EPL];
      if constexpr (YROW) {
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
#pragma unroll
          for (int e = 0; e < L::EPL; ++e) yr[k][e] = Ar<T>::zero();
          if (yext && live[k]) {
            const int rr = slot + k * SLOTS;
            const long long i = z * F + (long long)(y0 + rr / PL_TX) * m + x0 + rr % PL_TX;
            if (i < n) row_load_ex_rw<T, S>(yext + (size_t)i * S, g, yr[k]);
          }
        }
      }
      bwait(full + ns, nph);  // window z + 1
      const T* wc = win + (size_t)cs * C::WR * S;
      const T* wn = win + (size_t)ns * C::WR * S;
      const T* sv = vals + (size_t)cs * PL_TY * C::VL;
      const T* sy = ybuf + (size_t)cs * ny * PL_TY * C::YL;
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int rr = slot + k * SLOTS;
        const int yl = rr / PL_TX, xl = rr % PL_TX;
        T nx[L::EPL], pm[L::EPL], p1[L::EPL], q1[L::EPL], qm[L::EPL];
        row_load_ex_rw<T, S>(wn + woff[k], g, nx);
        row_load_ex_rw<T, S>(wc + woff[k] - C::WX * S, g, pm);
        row_load_ex_rw<T, S>(wc + woff[k] - S, g, p1);
        row_load_ex_rw<T, S>(wc + woff[k] + S, g, q1);
        row_load_ex_rw<T, S>(wc + woff[k] + C::WX * S, g, qm);
        if (live[k]) {
          const long long i = z * F + (long long)(y0 + yl) * m + x0 + xl;
          const long long i0 = z * F + (long long)(y0 + yl) * m + x0;
          const int sh = (sizeof(T) == 8) ? (int)(i0 & 1) : 0;
          const T* v = sv + (size_t)yl * C::VL + (size_t)(sh + xl) * PL_K;
          T x[L::EPL];
#pragma unroll
          for (int e = 0; e < L::EPL; ++e) {
            T acc = Ar<T>::zero();
            acc = Ar<T>::fma(v[0], prev[k][e], acc);
            acc = Ar<T>::fma(v[1], pm[e], acc);
            acc = Ar<T>::fma(v[2], p1[e], acc);
            acc = Ar<T>::fma(v[3], cur[k][e], acc);
            acc = Ar<T>::fma(v[4], q1[e], acc);
            acc = Ar<T>::fma(v[5], qm[e], acc);
            acc = Ar<T>::fma(v[6], nx[e], acc);
            x[e] = acc;
          }
          if (i < n) {
            row_store_ex_cs<T, S>(reinterpret_cast<T*>(a.Q) + (size_t)i * S, g, x);
            if (m0 != RED_NONE || m1 != RED_NONE) {
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const int md = q ? m1 : m0;
                if (md == RED_NONE) continue;
                const int yk = red_ykind(md);
                T yy[L::EPL];
                const T yv = yk == 1 ? sy[((size_t)yslot[q] * PL_TY + yl) * C::YL + sh + xl] : Ar<T>::zero();
#pragma unroll
                for (int e = 0; e < L::EPL; ++e) {
                  if constexpr (YROW) yy[e] = yk == 0 ? x[e] : (yk == 1 ? yv : (q == qext ? yr[k][e] : cur[k][e]));
                  else yy[e] = yk == 0 ? x[e] : yv;
                }
                if (q == 0) red_acc<T, S, false>(acc0, x, yy);
                else red_acc<T, S, false>(acc1, x, yy);
              }
            }
          }
        }
#pragma unroll
        for (int e = 0; e < L::EPL; ++e) {
          prev[k][e] = cur[k][e];
          cur[k][e] = nx[e];
        }
      }
      release();  // window z (its last reader was this step)
    }
    release();  // window ze: only its centre rows were read
  }
  if (a.nred > 0) {
    double* red_smem = reinterpret_cast<double*>(vals);  // the stages are no longer read
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    red_dispatch_flush<T, S, false>(m0, acc0, a.partials, a.pstride, a.red[0].poff, S, red_smem, 1, NW, 1);
    if (a.nred > 1)
      red_dispatch_flush<T, S, false>(m1, acc1, a.partials, a.pstride, a.red[1].poff, S, red_smem, 1, NW, 1);
  }
}

// ---------------------------------------------------------------- host side
template <typename T, int S>
static int launch_band_t(const BandArgs& a0, int nsm, cudaStream_t st, int* grid_out) {
  using C = BandCfg<T, S>;
  BandArgs a = a0;
  int nfar = 0;
  for (int k = 0; k < a.K; ++k) nfar += a.far_slot[k] >= 0;
  static const int env_d = getenv("SRK_BAND_D") ? atoi(getenv("SRK_BAND_D")) : 0;    // tuning knobs
  static const int env_tr = getenv("SRK_BAND_TR") ? atoi(getenv("SRK_BAND_TR")) : 0;
  a.D = (env_d >= 2 && env_d <= BAND_DMAX) ? env_d : 3;
  static const int env_x = getenv("SRK_BAND_X") ? atoi(getenv("SRK_BAND_X")) : 0;
  a.xflags = env_x;
  a.tr = (env_tr >= 16 && env_tr <= C::TR && (C::TR % env_tr) == 0) ? env_tr : C::TR;
  a.cap = a.D * a.tr + 2 * a.H;
  int ny = 0;
  for (int q = 0; q < a.nred; ++q) {
    const int yk = (a.red[q].mode == RED_NORM2 || a.red[q].mode == RED_COLNORM2) ? 0 : (a.red[q].mode == RED_SUMVEC ? 1 : 2);
    if (yk && (!a.red[q].yext || ((uintptr_t)a.red[q].yext & 15))) return (int)cudaErrorNotSupported;
    if (yk && a.red[q].ysrc >= 0) return (int)cudaErrorNotSupported;  // (SpMM reductions read Q and yext only)
    a.ystage[q] = yk;  // staged by the copy engine (measured: early global loads were slower)
    ny += yk ? 1 : 0;
  }
  const size_t smem = band_smem<T, S>(a.K, nfar, a.cap, ny, a.D, a.tr);
  if (smem > 220 * 1024) return (int)cudaErrorNotSupported;
  static const int env_nw = getenv("SRK_BAND_NW") ? atoi(getenv("SRK_BAND_NW")) : 0;
  const int nw = env_nw == 8 ? 8 : 16;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(band_kernel<T, S, 5, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(band_kernel<T, S, 7, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(band_kernel<T, S, BAND_KMAX, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(band_kernel<T, S, 5, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(band_kernel<T, S, 7, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(band_kernel<T, S, BAND_KMAX, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  }
  const long long ntiles = (a.n + a.tr - 1) / a.tr;
  // chunks of ct tiles: long enough that the 2H-row near window is loaded once per
  // chunk (~12% extra at 2H = 8 tiles), short enough for the sweep front to stay in L2
  a.ct = std::max(4, (int)((8LL * 2 * a.H + a.tr - 1) / a.tr));
  const long long nchunks = (ntiles + a.ct - 1) / a.ct;
  const int per_sm = (nw == 8 && smem <= 110 * 1024) ? 2 : 1;
  const int grid = (int)std::max<long long>(1, std::min<long long>((long long)nsm * per_sm, nchunks));
  if (grid_out) {  // grid query only (the caller sizes the partials first)
    *grid_out = grid;
    return 0;
  }
  static const bool use_cp = getenv("SRK_BAND_CP") != nullptr;  // cp.async feed (measured slower)
  if (use_cp) {
    static std::atomic<unsigned long long> attr2{0};
    if (first_on_device(attr2)) {
      cudaFuncSetAttribute(band_cp_kernel<T, S, 5, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      cudaFuncSetAttribute(band_cp_kernel<T, S, 7, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      cudaFuncSetAttribute(band_cp_kernel<T, S, BAND_KMAX, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    }
    const int g1 = (int)std::max<long long>(1, std::min<long long>(nsm, nchunks));
    if (a.K == 5) band_cp_kernel<T, S, 5, 16><<<g1, 512, smem, st>>>(a);
    else if (a.K == 7) band_cp_kernel<T, S, 7, 16><<<g1, 512, smem, st>>>(a);
    else band_cp_kernel<T, S, BAND_KMAX, 16><<<g1, 512, smem, st>>>(a);
    return (int)cudaGetLastError();
  }
  // the diagonal count as a compile-time trip count for the 2D / 3D stencils
  if (nw == 8) {
    if (a.K == 5) band_kernel<T, S, 5, 8><<<grid, 32 * 9, smem, st>>>(a);
    else if (a.K == 7) band_kernel<T, S, 7, 8><<<grid, 32 * 9, smem, st>>>(a);
    else band_kernel<T, S, BAND_KMAX, 8><<<grid, 32 * 9, smem, st>>>(a);
  } else {
    if (a.K == 5) band_kernel<T, S, 5, 16><<<grid, 32 * 17, smem, st>>>(a);
    else if (a.K == 7) band_kernel<T, S, 7, 16><<<grid, 32 * 17, smem, st>>>(a);
    else band_kernel<T, S, BAND_KMAX, 16><<<grid, 32 * 17, smem, st>>>(a);
  }
  return (int)cudaGetLastError();
}


// 7-point pattern {-F, -m, -1, 0, 1, m, F}, F a multiple of m (band_plane_kernel)
bool band_plane_pattern(const Mat::Band& b) {
  static const int env = getenv("SRK_BAND_PLANE") ? atoi(getenv("SRK_BAND_PLANE")) : 1;
  if (!env || b.K != PL_K) return false;
  const long long F = b.off[6], m = b.off[5];
  if (b.off[0] != -F || b.off[1] != -m || b.off[2] != -1 || b.off[3] != 0 || b.off[4] != 1) return false;
  return m >= 2 && F > m && F % m == 0;
}

template <typename T, int S>
static int launch_plane_t(const BandArgs& ba, const Mat::Band& b, int nsm, cudaStream_t st, int* grid_out) {
  constexpr int NW = 16;
  PlaneArgs a{};
  a.dia = ba.dia;
  a.P = ba.P;
  a.Q = ba.Q;
  a.n = ba.n;
  a.F = b.off[6];
  a.m = b.off[5];
  a.ny = (int)(a.F / a.m);
  a.nz = (a.n + a.F - 1) / a.F;
  a.ntx = (a.m + PL_TX - 1) / PL_TX;
  a.nty = (a.ny + PL_TY - 1) / PL_TY;
  a.nred = ba.nred;
  int ny = 0, next = 0, nrow = 0;
  for (int q = 0; q < a.nred; ++q) {
    a.red[q] = ba.red[q];
    const int md = a.red[q].mode;
    const int yk = (md == RED_NORM2 || md == RED_COLNORM2) ? 0 : (md == RED_SUMVEC ? 1 : 2);
    if (yk && (!a.red[q].yext || ((uintptr_t)a.red[q].yext & 15) || a.red[q].ysrc >= 0))
      return (int)cudaErrorNotSupported;
    if (yk == 2 && a.red[q].yext != a.P && ++next > 1) return (int)cudaErrorNotSupported;  // one external row operand
    nrow += yk == 2;
    a.ystage[q] = yk == 1;  // SUMVEC vectors are staged per plane by the copy engine
    ny += yk == 1;
  }
  a.partials = ba.partials;
  a.pstride = ba.pstride;
  a.done = ba.done;
  static const int env_nb = getenv("SRK_PLANE_NB") ? atoi(getenv("SRK_PLANE_NB")) : 0;
  a.NB = 0;
  for (int nb = (env_nb >= 3 && env_nb <= PL_NBMAX) ? env_nb : PL_NBMAX; nb >= 3; --nb)
    if (plane_smem<T, S>(nb, ny) <= 220 * 1024) {
      a.NB = nb;
      break;
    }
  if (!a.NB) return (int)cudaErrorNotSupported;
  // plane segment length: fewest window loads per CTA (ceil(items / grid) rounds of ZL + 2
  // windows), ties to the longer segment
  const long long ntile = (long long)a.ntx * a.nty;
  static const int env_zl = getenv("SRK_PLANE_ZL") ? atoi(getenv("SRK_PLANE_ZL")) : 0;
  long long best = -1;
  for (long long zl = 1; zl <= a.nz; ++zl) {
    const long long nzs = (a.nz + zl - 1) / zl;
    const long long items = ntile * nzs;
    const long long grid = std::min<long long>(nsm, items);
    const long long cost = (items + grid - 1) / grid * (zl + 2);
    if (env_zl > 0 ? zl == std::min<long long>(env_zl, a.nz) : (best < 0 || cost <= best)) {
      best = cost;
      a.zl = (int)zl;
    }
  }
  a.nzs = (int)((a.nz + a.zl - 1) / a.zl);
  a.nitems = ntile * a.nzs;
  const int grid = (int)std::min<long long>(nsm, a.nitems);
  if (grid_out) {
    *grid_out = grid;
    return 0;
  }
  const size_t smem = plane_smem<T, S>(a.NB, ny);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(band_plane_kernel<T, S, NW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(band_plane_kernel<T, S, NW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  }
  if (nrow) band_plane_kernel<T, S, NW, true><<<grid, 32 * (NW + 1), smem, st>>>(a);
  else band_plane_kernel<T, S, NW, false><<<grid, 32 * (NW + 1), smem, st>>>(a);
  return (int)cudaGetLastError();
}


// ---------------------------------------------------------------------------
// Banded vector product (s = 1, no fused reduction): the economic variants' one A^H-vector
// product per iteration. One row per thread, RT rows per thread, every load of a
// thread's rows issued before the first FMA: the K diagonal values of row i (contiguous, [n][K]
// row-major; a warp's 32 rows are one contiguous 32 K-value span, so the K strided loads of a warp
// touch the same sectors: L1 hits after the first) and p[i + d_k], coalesced across the warp for
// every k, whose K readers run within neighbouring tiles (L1 / L2 hits): DRAM = K values + p + q per
// row (72 B for the 7-point stencil against 104 B for the CSR arrays). Summation in ascending
// offset (= CSR order), as in the other band kernels. (A first version staged a CTA tile's values
// through shared memory with two barriers per tile: 0.74 ms on config 3 against the CSR kernel's
// 0.385 ms — the staging and the p loads ran back to back instead of overlapping.)
template <typename T, int KT>
__global__ void __launch_bounds__(256) band_vec_kernel(const T* __restrict__ dia, const T* __restrict__ p, T* __restrict__ q,
                                                       long long n, int Krt, BandOffs offs, const int* done) {
  if (done && *done) return;
  constexpr int RT = 2;
  const int K = KT > 0 ? KT : Krt;
  constexpr int KM = KT > 0 ? KT : BAND_KMAX;
  const long long stride = (long long)gridDim.x * 256 * RT;
  for (long long r0 = (long long)blockIdx.x * 256 * RT; r0 < n; r0 += stride) {
    T dv[RT][KM], pv[RT][KM];
#pragma unroll
    for (int u = 0; u < RT; ++u) {
      const long long i = r0 + u * 256 + threadIdx.x;
#pragma unroll
      for (int k = 0; k < KM; ++k) {
        const long long jj = i + offs.d[k];
        const bool in = k < K && i < n;
        dv[u][k] = in ? __ldcs(dia + i * K + k) : Ar<T>::zero();
        pv[u][k] = (in && jj >= 0 && jj < n) ? __ldg(p + jj) : Ar<T>::zero();
      }
    }
#pragma unroll
    for (int u = 0; u < RT; ++u) {
      const long long i = r0 + u * 256 + threadIdx.x;
      T acc = Ar<T>::zero();
#pragma unroll
      for (int k = 0; k < KM; ++k)
        if (k < K) acc = Ar<T>::fma(dv[u][k], pv[u][k], acc);
      if (i < n) q[i] = acc;
    }
  }
}

template <typename T>
static int launch_band_vec(const BandArgs& a, int nsm, cudaStream_t st, int* grid_out) {
  const long long need = (a.n + 511) / 512;
  const int grid = (int)std::max<long long>(1, std::min<long long>(need, (long long)nsm * 8));
  if (grid_out) {
    *grid_out = grid;
    return 0;
  }
  BandOffs offs{};
  for (int k = 0; k < a.K; ++k) offs.d[k] = a.off[k];
  const T* dia = reinterpret_cast<const T*>(a.dia);
  const T* p = reinterpret_cast<const T*>(a.P);
  T* q = reinterpret_cast<T*>(a.Q);
  if (a.K == 7) band_vec_kernel<T, 7><<<grid, 256, 0, st>>>(dia, p, q, a.n, a.K, offs, a.done);
  else if (a.K == 5) band_vec_kernel<T, 5><<<grid, 256, 0, st>>>(dia, p, q, a.n, a.K, offs, a.done);
  else band_vec_kernel<T, 0><<<grid, 256, 0, st>>>(dia, p, q, a.n, a.K, offs, a.done);
  return (int)cudaGetLastError();
}

bool band_supported(bool cplx, int s) {
  if (cplx) return s == 1 || s == 4 || s == 8;
  return s == 1 || s == 2 || s == 4 || s == 8 || s == 16;  // (s = 1 real: band_vec_kernel, no fused reduction)
}


// Q = A P over the banded form (Mat::Band); reductions as in the CSR kernel (non-FULL).
// Returns cudaErrorNotSupported when the width / diagonal set does not fit (the caller
// then runs the CSR kernel).
int launch_band(bool cplx, int s, const Mat::Band& b, const void* P, void* Q, long long n, const Red* red, int nred,
                double* partials, int pstride, const int* done, int nsm, cudaStream_t st, int* grid_out) {
  if (!band_supported(cplx, s) || b.K == 0 || nred > 2) return (int)cudaErrorNotSupported;
  BandArgs a{};
  a.dia = b.val;
  a.npad = b.npad;
  a.K = b.K;
  static const bool no_vec = getenv("SRK_NO_BAND_VEC") != nullptr;  // A/B switch
  if (s == 1 && !cplx) {  // the economic variants' vector product
    if (nred > 0 || no_vec) return (int)cudaErrorNotSupported;
    for (int k = 0; k < b.K; ++k) a.off[k] = b.off[k];
    a.P = P;
    a.Q = Q;
    a.n = n;
    a.done = done;
    return launch_band_vec<double>(a, nsm, st, grid_out);
  }
  if (band_plane_pattern(b)) {  // the 7-point pattern: the plane-marching kernel
    BandArgs pa = a;
    pa.P = P;
    pa.Q = Q;
    pa.n = n;
    pa.nred = nred;
    for (int i = 0; i < nred; ++i) pa.red[i] = red[i];
    pa.partials = partials;
    pa.pstride = pstride;
    pa.done = done;
    int r = (int)cudaErrorNotSupported;
    if (cplx) {
      switch (s) {
        case 1: r = launch_plane_t<double2, 1>(pa, b, nsm, st, grid_out); break;
        case 4: r = launch_plane_t<double2, 4>(pa, b, nsm, st, grid_out); break;
        case 8: r = launch_plane_t<double2, 8>(pa, b, nsm, st, grid_out); break;
      }
    } else {
      switch (s) {
        case 2: r = launch_plane_t<double, 2>(pa, b, nsm, st, grid_out); break;
        case 4: r = launch_plane_t<double, 4>(pa, b, nsm, st, grid_out); break;
        case 8: r = launch_plane_t<double, 8>(pa, b, nsm, st, grid_out); break;
        case 16: r = launch_plane_t<double, 16>(pa, b, nsm, st, grid_out); break;
      }
    }
    if (r != (int)cudaErrorNotSupported) return r;
  }
  const int hcap = band_hcap(s * (cplx ? 16 : 8));
  a.H = 0;
  for (int k = 0; k < b.K; ++k)
    if (std::abs(b.off[k]) <= hcap) a.H = std::max(a.H, std::abs(b.off[k]));
  int nf = 0;
  for (int k = 0; k < b.K; ++k) {
    a.off[k] = b.off[k];
    a.far_slot[k] = std::abs(b.off[k]) > a.H ? nf++ : -1;
  }
  if (nf > BAND_FMAX) return (int)cudaErrorNotSupported;
  a.P = P;
  a.Q = Q;
  a.n = n;
  a.nred = nred;
  for (int i = 0; i < nred; ++i) a.red[i] = red[i];
  a.partials = partials;
  a.pstride = pstride;
  a.done = done;
  if (cplx) {
    switch (s) {
      case 1: return launch_band_t<double2, 1>(a, nsm, st, grid_out);
      case 4: return launch_band_t<double2, 4>(a, nsm, st, grid_out);
      case 8: return launch_band_t<double2, 8>(a, nsm, st, grid_out);
    }
  } else {
    switch (s) {
      case 2: return launch_band_t<double, 2>(a, nsm, st, grid_out);
      case 4: return launch_band_t<double, 4>(a, nsm, st, grid_out);
      case 8: return launch_band_t<double, 8>(a, nsm, st, grid_out);
      case 16: return launch_band_t<double, 16>(a, nsm, st, grid_out);
    }
  }
  return (int)cudaErrorNotSupported;
}

// ------------------------------------------------------------ a0: band detection
// Every nonzero's diagonal d = j - i goes into a set of at most BAND_KMAX slots (CAS
// insertion; the set is tiny, so after the first rows every thread only reads it).
__global__ static void band_offsets_kernel(const int* rp, const int* ci, long long n, long long* slots, int* overflow) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    for (int p = rp[i]; p < rp[i + 1]; ++p) {
      const long long d = (long long)ci[p] - i;
      bool found = false;
      for (int q = 0; q < BAND_KMAX && !found; ++q) {
        long long cur = *(volatile long long*)(slots + q);
        if (cur == d) { found = true; break; }
        if (cur == LLONG_MIN) {
          const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(slots + q),
                                                    (unsigned long long)LLONG_MIN, (unsigned long long)d);
          if ((long long)prev == LLONG_MIN || (long long)prev == d) found = true;
        }
      }
      if (!found) *overflow = 1;
    }
  }
}

template <typename T>
__global__ static void band_fill_kernel(const int* rp, const int* ci, const T* val, long long n, const int* off, int K,
                                        long long npad, T* dia) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    for (int p = rp[i]; p < rp[i + 1]; ++p) {
      const long long d = (long long)ci[p] - i;
      for (int k = 0; k < K; ++k)
        if (off[k] == d) dia[(size_t)i * K + k] = val[p];
    }
}

// Builds b from a CSR (device arrays); returns 0 and b.K = 0 if the operator is not banded
// (more than BAND_KMAX diagonals, or offsets beyond int range).
int build_band(bool cplx, long long n, const int* rp, const int* ci, const void* val, Mat::Band& b, cudaStream_t st) {
  b = Mat::Band{};
  long long* slots = nullptr;
  int* ovf = nullptr;
  if (cudaMalloc(&slots, sizeof(long long) * BAND_KMAX) != cudaSuccess) return (int)cudaErrorMemoryAllocation;
  if (cudaMalloc(&ovf, sizeof(int)) != cudaSuccess) {
    cudaFree(slots);
    return (int)cudaErrorMemoryAllocation;
  }
  std::vector<long long> h(BAND_KMAX, LLONG_MIN);
  cudaMemcpyAsync(slots, h.data(), sizeof(long long) * BAND_KMAX, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(ovf, 0, sizeof(int), st);
  const int grid = (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8));
  band_offsets_kernel<<<grid, 256, 0, st>>>(rp, ci, n, slots, ovf);
  int o = 0;
  cudaMemcpyAsync(h.data(), slots, sizeof(long long) * BAND_KMAX, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&o, ovf, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(slots);
  cudaFree(ovf);
  if (e != cudaSuccess) return (int)e;
  if (o) return 0;
  std::vector<long long> offs;
  for (long long d : h)
    if (d != LLONG_MIN) offs.push_back(d);
  std::sort(offs.begin(), offs.end());
  if (offs.empty()) return 0;
  for (long long d : offs)
    if (d > INT_MAX / 2 || d < -INT_MAX / 2) return 0;
  const size_t esz = cplx ? 16 : 8;
  b.K = (int)offs.size();
  b.npad = (n + 1023) / 1024 * 1024;
  for (int k = 0; k < b.K; ++k) b.off[k] = (int)offs[k];
  if (cudaMalloc(&b.val, esz * b.npad * b.K) != cudaSuccess) {
    b = Mat::Band{};
    return (int)cudaErrorMemoryAllocation;
  }
  int* doff = nullptr;
  if (cudaMalloc(&doff, sizeof(int) * b.K) != cudaSuccess) {
    cudaFree(b.val);
    b = Mat::Band{};
    return (int)cudaErrorMemoryAllocation;
  }
  cudaMemcpyAsync(doff, b.off, sizeof(int) * b.K, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(b.val, 0, esz * b.npad * b.K, st);
  if (cplx) band_fill_kernel<double2><<<grid, 256, 0, st>>>(rp, ci, (const double2*)val, n, doff, b.K, b.npad, (double2*)b.val);
  else band_fill_kernel<double><<<grid, 256, 0, st>>>(rp, ci, (const double*)val, n, doff, b.K, b.npad, (double*)b.val);
  e = cudaStreamSynchronize(st);
  cudaFree(doff);
  return e == cudaSuccess ? 0 : (int)e;
}

}  // namespace srk
