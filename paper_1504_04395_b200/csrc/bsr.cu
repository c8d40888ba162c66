// bsr.cu — block-sparse (BSR, 12 x 12 complex blocks) SpMM Q = A P for the
// lattice operator of config 4 ("convert to ... BSR-12
// (lattice)"; PAPER.md P:752-778 Ex. 4's 12 dof/site Wilson-type operator, and the
// read-A-once block product P:66-74).
//
// Why blocks: in scalar CSR every one of a row's 97 entries gathers a whole P row
// (s = 12 complex = 192 B), i.e. ~18.6 KB of L2->SM traffic per row; in BSR a
// 12 x 12 block multiplies the 12 contiguous rows of P_J once (2.3 KB per block,
// ~1.7 KB per row), and no column index is stored per scalar entry.
//
// One warp per block row I: for every block J of the row the warp stages the
// block (12 x 12 complex, contiguous) and P_J (12 rows x S complex, contiguous)
// in its shared-memory double buffer with cp.async (the next block in flight
// while the current one is multiplied), and multiplies on the FP64 tensor cores:
// the complex product is the real one
//   [Q_r Q_i](12 x 2S, interleaved) += [B_r B_i](12 x 24, interleaved) * Bm(24 x 2S)
// with Bm[2k][c'] = P[k][c'], Bm[2k+1][2c] = -Im P[k][c], Bm[2k+1][2c+1] = Re P[k][c]
// (formed in the fragment load), M = 12 padded to 16, so 2 x (2S/8) x 6 DMMAs
// m8n8k4 per block. unit_diag adds the identity block (Q_I += P_I) in the epilogue.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "kernels.cuh"

namespace srk {

namespace {

constexpr int BS = 12;         // block size (rows = cols)
constexpr int BROW = 28;       // smem row stride of a staged block (doubles): 24 + 4 pad, 2-way banks
constexpr int BBLK = BS * BROW;  // doubles per staged block
constexpr int BSR_CFG_DEFAULT = 3;  // see launch_s (measured: scripts/bsr_probe.py, profiles/r02_bsr_probe.txt)

// 16-byte async copy with an L2 eviction policy: the blocks of A stream through
// once (evict_first) while the rows of P are re-read by the neighbouring block rows
// (evict_last), so A does not push P out of L2
__device__ __forceinline__ void cpa16(double* smem, const double* gmem, unsigned long long pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "l"(pol));
}
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int S>
struct BCfg {
  static constexpr int NR = 2 * S;            // real columns of P / Q
  static constexpr int NT = NR / 8;           // N tiles
  static constexpr int PBLK = BS * NR;        // doubles of a staged P block
  static constexpr int STAGE = BBLK + PBLK;   // one buffer
  static constexpr int WARP_SMEM = 2 * STAGE; // double buffer (doubles)
  static constexpr int WARPS = 8;
  static constexpr int SMEM = WARPS * WARP_SMEM * 8;
};

template <int S>
__global__ void __launch_bounds__(256, S >= 16 ? 1 : 2) bsr12_kernel(BsrArgs a) {
  if (a.done && *a.done) return;
  using C = BCfg<S>;
  extern __shared__ __align__(16) double bsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wbuf = bsm + (size_t)warp * C::WARP_SMEM;
  const double* __restrict__ val = reinterpret_cast<const double*>(a.val);
  const double* __restrict__ P = reinterpret_cast<const double*>(a.P);
  double* __restrict__ Q = reinterpret_cast<double*>(a.Q);
  const long long nb = a.nb;
  const long long gw = (long long)blockIdx.x * C::WARPS + warp;
  const long long nw = (long long)gridDim.x * C::WARPS;
  const int fr = lane >> 2, fk = lane & 3;
  // B-fragment swizzle of the complex -> real lift (odd k' rows: (-Im, Re) pairs)
  const int t = fk & 1;
  const int poff = t ? (fr ^ 1) : fr;
  // -Im P: flip the sign bit on the integer side (keeps the FP64 pipe for DMMAs)
  const unsigned long long psgn = (t && !(fr & 1)) ? 0x8000000000000000ULL : 0ULL;

  const unsigned long long pol_a = policy_evict_first(), pol_p = policy_evict_last();
  // stage block j (values) and the P rows of its block column into buffer b
  auto stage = [&](int j, int b) {
    double* bs = wbuf + (size_t)b * C::STAGE;
    double* ps = bs + BBLK;
    const double* bv = val + (size_t)j * (BS * BS * 2);
    const double* pj = P + (size_t)a.bci[j] * BS * C::NR;
    for (int c = lane; c < BS * 12; c += 32) {  // 12 rows x 12 chunks of 16 B
      const int r = c / 12, q = c % 12;
      cpa16(bs + r * BROW + 2 * q, bv + r * 24 + 2 * q, pol_a);
    }
    for (int c = lane; c < C::PBLK / 2; c += 32) cpa16(ps + 2 * c, pj + 2 * c, pol_p);
  };

  // epilogue reductions: per lane, over the Q entries it owns (rows fr and 8 + fr,
  // complex columns n * 4 + fk): scalar modes in rs[r], per-column modes in rc[r][n]
  const int nred = a.nred;
  int rmode[2];
  const double* ry[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    rmode[r] = r < nred ? a.red[r].mode : RED_NONE;
    ry[r] = r < nred ? reinterpret_cast<const double*>(a.red[r].yext) : nullptr;
  }
  double2 rs[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  double2 rc[2][C::NT];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int n = 0; n < C::NT; ++n) rc[r][n] = make_double2(0.0, 0.0);

  for (long long I = gw; I < nb; I += nw) {
    const int jb = __ldg(a.brp + I), je = __ldg(a.brp + I + 1);
    double acc[2][C::NT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < C::NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    if (je > jb) stage(jb, 0);
    cp_commit();
    // epilogue operands requested now, consumed after the row's last block: the
    // unit-diagonal P_I entries and reduction 0's Y entries at this lane's places
    double2 pI[2][C::NT], y0[2][C::NT];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int row = m * 8 + fr;
      const size_t base = ((size_t)I * BS + (row < BS ? row : 0)) * C::NR;
#pragma unroll
      for (int n = 0; n < C::NT; ++n) {
        const int col = n * 8 + 2 * fk;
        pI[m][n] = make_double2(0.0, 0.0);
        y0[m][n] = make_double2(0.0, 0.0);
        if (row < BS) {
          if (a.unit_diag) pI[m][n] = __ldg(reinterpret_cast<const double2*>(P + base + col));
          const int md = rmode[0];
          if (md == RED_SUMVEC) {
            if (n == 0) y0[m][0] = __ldg(reinterpret_cast<const double2*>(ry[0]) + (size_t)I * BS + row);
          } else if (md == RED_DIAG || md == RED_TRACE) {
            y0[m][n] = __ldg(reinterpret_cast<const double2*>(ry[0] + base + col));
          }
        }
      }
    }
    for (int j = jb; j < je; ++j) {
      const int b = (j - jb) & 1;
      if (j + 1 < je) stage(j + 1, b ^ 1);
      cp_commit();
      cp_wait<1>();
      __syncwarp();
      const double* bs = wbuf + (size_t)b * C::STAGE;
      const double* ps = bs + BBLK;
#pragma unroll
      for (int ks = 0; ks < 6; ++ks) {
        const int kr = ks * 4 + fk;  // real k' of this lane's fragments
        const double a0 = bs[fr * BROW + kr];
        const double a1 = fr < 4 ? bs[(8 + fr) * BROW + kr] : 0.0;
        const int prow = kr >> 1;
#pragma unroll
        for (int n = 0; n < C::NT; ++n) {
          const double bb = __longlong_as_double(__double_as_longlong(ps[prow * C::NR + n * 8 + poff]) ^ (long long)psgn);
          dmma(acc[0][n], a0, bb);
          dmma(acc[1][n], a1, bb);
        }
      }
      __syncwarp();  // buffer b is restaged at j + 2
    }
    // epilogue: Q rows 12 I + row (row < 12), (+ P_I for the unit diagonal)
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int row = m * 8 + fr;
      if (row < BS) {
        const size_t base = ((size_t)I * BS + row) * C::NR;
#pragma unroll
        for (int n = 0; n < C::NT; ++n) {
          const int col = n * 8 + 2 * fk;
          double2 v = make_double2(acc[m][n][0], acc[m][n][1]);
          if (a.unit_diag) {
            v.x += pI[m][n].x;
            v.y += pI[m][n].y;
          }
          *reinterpret_cast<double2*>(Q + base + col) = v;
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int md = rmode[r];
            if (md == RED_NONE) continue;
            if (md == RED_NORM2 || md == RED_COLNORM2) {
              const double q2 = v.x * v.x + v.y * v.y;
              if (md == RED_NORM2) rs[r].x += q2;
              else rc[r][n].x += q2;
            } else {
              // conj(y) * q with y the Y entry at the same place (SUMVEC: the row's vector entry)
              const double2 y = r == 0 ? (md == RED_SUMVEC ? y0[m][0] : y0[m][n])
                                       : (md == RED_SUMVEC ? __ldg(reinterpret_cast<const double2*>(ry[r]) + (size_t)I * BS + row)
                                                           : __ldg(reinterpret_cast<const double2*>(ry[r] + base + col)));
              const double2 pr = make_double2(y.x * v.x + y.y * v.y, y.x * v.y - y.y * v.x);
              if (md == RED_DIAG) {
                rc[r][n].x += pr.x;
                rc[r][n].y += pr.y;
              } else {
                rs[r].x += pr.x;
                rs[r].y += pr.y;
              }
            }
          }
        }
      }
    }
  }
  if (nred == 0) return;
  // CTA partials in the layout of red_len: fixed-order warp butterflies, then the
  // warps summed in index order (deterministic)
  __syncthreads();  // every warp is done with its staging buffers
  double* red_sm = bsm;  // [warp][len] doubles
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (r >= nred) break;
    const int md = rmode[r];
    const int len = red_len(md, S, true);
    double* w = red_sm + (size_t)warp * len;
    if (md == RED_DIAG || md == RED_COLNORM2) {
#pragma unroll
      for (int n = 0; n < C::NT; ++n) {
        double2 v = rc[r][n];
#pragma unroll
        for (int m = 4; m < 32; m <<= 1) {  // over fr: lanes with equal fk hold the same columns
          v.x += __shfl_xor_sync(0xffffffffu, v.x, m);
          v.y += __shfl_xor_sync(0xffffffffu, v.y, m);
        }
        if (fr == 0) {
          const int c = n * 4 + fk;
          if (md == RED_DIAG) {
            w[2 * c] = v.x;
            w[2 * c + 1] = v.y;
          } else {
            w[c] = v.x;
          }
        }
      }
    } else {
      double2 v = rs[r];
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, m);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, m);
      }
      if (lane == 0) {
        w[0] = v.x;
        if (md != RED_NORM2) w[1] = v.y;
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
      double acc = 0.0;
      for (int q = 0; q < C::WARPS; ++q) acc += red_sm[q * len + j];
      a.partials[(size_t)blockIdx.x * a.pstride + a.red[r].poff + j] = acc;
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------------------
// Round 2: the product without the M = 12 -> 16 padding. The complex block product is the
// real contraction
//   [B_r; B_i] (24 x 12)  *  [P_r | P_i] (12 x 2S)   ->   B_r P_r, B_r P_i, B_i P_r, B_i P_i
// M = 24 (three 8-row tiles, no padding), K = 12 (three k-steps), N = 2S, i.e. 9 * 2S/8 DMMAs per
// block (27 at S = 12) against 12 * 2S/8 (36) for the [B_r B_i] * lift(P) form above, and no sign
// flips; Q_r = B_r P_r - B_i P_i and Q_i = B_r P_i + B_i P_r are formed once per block ROW from
// the four accumulator sets. Tiles are chosen so that almost every fragment pair is one 16-byte
// shared-memory load and the combination is lane-local:
//   M tile 0 = B_r rows 0-7, M tile 1 = B_i rows 0-7 (lane row fr: one double2 = (Re, Im) of
//   B[fr][k] feeds both), M tile 2 = rows 8-11 with lane row 8 + fr/2 and part fr & 1 (B_r in
//   even-fr lanes, B_i in odd: one exchange with lane ^ 4 per block row);
//   N tiles in pairs: tile "re" = Re of complex columns 8j..8j+7, tile "im" = Im of the same
//   (lane column fr: one double2 of the interleaved P row feeds both), so a lane owns the complex
//   columns 8j + 2fk, 8j + 2fk + 1; a remaining group of 4 complex columns (S = 4, 12) is one tile
//   over the interleaved (Re, Im) columns, owning complex column 8 NP + fk.
// The block (2304 contiguous bytes) is staged unpadded — row stride 24 doubles is conflict-free
// for these fragment loads —, the 12 P rows with stride 2S + 4. Staging is by bulk copies
// (`cp.async.bulk`, one per lane: the block + 12 rows) into a per-warp two-stage mbarrier ring
// that runs ahead across block-row boundaries (the next row's first block is in flight during
// this row's last).
template <int S, int NWARP = 8, int NSTAGE = 2, bool EST = false, bool PAD = true>
struct B2Cfg {
  static constexpr int NR = 2 * S;
  static constexpr int NP = NR / 16;         // N-tile pairs
  static constexpr int NS = (NR % 16) / 8;   // single N tile (4 complex columns)
  static constexpr int NC = 2 * NP + NS;     // complex columns a lane owns per row
  // staged P row stride (doubles): NR + 4 (= 4 or 12 mod 16: conflict-free fragment loads, one copy
  // per row) or NR (one copy per block, 2-way conflicts on the P fragments)
  static constexpr int PST = PAD ? NR + 4 : NR;
  static constexpr bool PADDED = PAD;
  static constexpr int ABLK = BS * BS * 2;   // 288 doubles, unpadded
  static constexpr int STAGE = ABLK + BS * PST;
  static constexpr int NSTG = NSTAGE;         // ring stages per warp
  static constexpr int WARPS = NWARP;
  static constexpr bool ESTG = EST;           // epilogue operands (P_I, Y_I) staged by bulk copy too
  static constexpr int EBUF = EST ? 2 * BS * NR : 0;  // doubles per warp
  static constexpr int WARP_D = NSTG * STAGE + EBUF;
  static constexpr int SMEM = WARPS * WARP_D * 8 + WARPS * (NSTG + 1) * 8;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITB_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITB_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, unsigned bytes, unsigned long long* bar,
                                         unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <int S, int NWARP, int NSTAGE, bool EST, bool PAD>
__global__ void __launch_bounds__(32 * NWARP, S >= 16 ? 1 : 2) bsr12_kernel2(BsrArgs a) {
  if (a.done && *a.done) return;
  using C = B2Cfg<S, NWARP, NSTAGE, EST, PAD>;
  extern __shared__ __align__(16) double bsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wbuf = bsm + (size_t)warp * C::WARP_D;
  double* ebuf = wbuf + (size_t)C::NSTG * C::STAGE;  // [P_I rows | Y_I rows] (ESTG)
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(bsm + (size_t)C::WARPS * C::WARP_D) + warp * (C::NSTG + 1);
  unsigned long long* ebar = bars + C::NSTG;
  const double* __restrict__ val = reinterpret_cast<const double*>(a.val);
  const double* __restrict__ P = reinterpret_cast<const double*>(a.P);
  double* __restrict__ Q = reinterpret_cast<double*>(a.Q);
  const long long nb = a.nb;
  const long long gw = (long long)blockIdx.x * C::WARPS + warp;
  const long long nw = (long long)gridDim.x * C::WARPS;
  const int fr = lane >> 2, fk = lane & 3;
  const unsigned long long pol_a = policy_evict_first(), pol_p = policy_evict_last();

  if (lane == 0) {
    for (int q = 0; q <= C::NSTG; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + q)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // producer side: the warp's blocks in order, across its block rows (Ip, jp, jpe = next to issue)
  // (positions k = gw, gw + nw, ... of the visiting order; block row = order[k], or k)
  const int* __restrict__ order = a.order;
  auto row_of = [&](long long k) -> long long { return order ? (long long)__ldg(order + k) : k; };
  long long Ip = gw;
  int jp = 0, jpe = 0;
  auto seek = [&]() {  // move (Ip, jp) to the next existing block at or after the position
    while (Ip < nb && jp >= jpe) {
      Ip += nw;
      if (Ip < nb) {
        const long long r = row_of(Ip);
        jp = __ldg(a.brp + r);
        jpe = __ldg(a.brp + r + 1);
      }
    }
  };
  if (Ip < nb) {
    const long long r = row_of(Ip);
    jp = __ldg(a.brp + r);
    jpe = __ldg(a.brp + r + 1);
    seek();
  }
  constexpr unsigned ABYTES = C::ABLK * 8, PBYTES = C::NR * 8;
  auto issue = [&](unsigned cnt) {  // block jp into stage cnt % NSTG
    const int st = (int)(cnt % C::NSTG);
    double* bs = wbuf + (size_t)st * C::STAGE;
    unsigned long long* bar = bars + st;
    if constexpr (C::PADDED) {
      // (a bulk copy is a per-warp instruction with uniform operands: copies issued by different
      // lanes are serialised by a loop over the active lanes, ~10 instructions per copy)
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                     "r"(ABYTES + BS * PBYTES)
                     : "memory");
        bulk_g2s(bs, val + (size_t)jp * C::ABLK, ABYTES, bar, pol_a);
      } else if (lane <= BS) {
        const double* pj = P + ((size_t)__ldg(a.bci + jp) * BS + (lane - 1)) * C::NR;
        bulk_g2s(bs + C::ABLK + (lane - 1) * C::PST, pj, PBYTES, bar, pol_p);
      }
    } else {
      if (lane == 0) {  // two copies per block: the block and its 12 contiguous P rows
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                     "r"(ABYTES + BS * PBYTES)
                     : "memory");
        bulk_g2s(bs, val + (size_t)jp * C::ABLK, ABYTES, bar, pol_a);
        bulk_g2s(bs + C::ABLK, P + (size_t)__ldg(a.bci + jp) * BS * C::NR, BS * PBYTES, bar, pol_p);
      }
    }
    ++jp;
    seek();
  };
  unsigned issued = 0, used = 0, rows_done = 0;

  // complex column of owned slot ci
  auto ccol = [&](int ci) { return ci < 2 * C::NP ? 8 * (ci >> 1) + 2 * fk + (ci & 1) : 8 * C::NP + fk; };
  const bool own2 = !(fr & 1);  // this lane finalises row 8 + fr/2

  const int nred = a.nred;
  int rmode[2];
  const double* ry[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    rmode[r] = r < nred ? a.red[r].mode : RED_NONE;
    ry[r] = r < nred ? reinterpret_cast<const double*>(a.red[r].yext) : nullptr;
  }
  double2 rs[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  double2 rc[2][C::NC];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int n = 0; n < C::NC; ++n) rc[r][n] = make_double2(0.0, 0.0);

  for (long long kI = gw; kI < nb; kI += nw) {
    const long long I = row_of(kI);
    const int jb = __ldg(a.brp + I), je = __ldg(a.brp + I + 1);
    // accP[mt][j][part of P][e], accS[mt][part]
    double accP[3][C::NP > 0 ? C::NP : 1][2][2];
    double accS[3][2];
#pragma unroll
    for (int mt = 0; mt < 3; ++mt) {
#pragma unroll
      for (int j = 0; j < C::NP; ++j) accP[mt][j][0][0] = accP[mt][j][0][1] = accP[mt][j][1][0] = accP[mt][j][1][1] = 0.0;
      accS[mt][0] = accS[mt][1] = 0.0;
    }
    // epilogue operands requested now, consumed after the row's last block: the unit-diagonal
    // operand P_I and reduction 0's Y rows (or y entries) — by bulk copy into the warp's epilogue
    // buffer (ESTG), else P_I in registers and Y read in the epilogue (prefetching both in
    // registers spilled at S = 12)
    const int md0 = rmode[0];
    const bool y0rows = md0 == RED_DIAG || md0 == RED_TRACE, y0vec = md0 == RED_SUMVEC;
    double2 pI[2][C::ESTG ? 1 : C::NC];
    if constexpr (C::ESTG) {
      constexpr unsigned RB = BS * C::NR * 8;
      if (lane == 0) {
        const unsigned bytes = (a.unit_diag ? RB : 0u) + (y0rows ? RB : (y0vec ? (unsigned)(BS * 16) : 0u));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(ebar)), "r"(bytes) : "memory");
        if (a.unit_diag) bulk_g2s(ebuf, P + (size_t)I * BS * C::NR, RB, ebar, pol_p);
      } else if (lane == 1) {
        if (y0rows) bulk_g2s(ebuf + BS * C::NR, ry[0] + (size_t)I * BS * C::NR, RB, ebar, pol_a);
        else if (y0vec) bulk_g2s(ebuf + BS * C::NR, ry[0] + (size_t)I * BS * 2, BS * 16, ebar, pol_a);
      }
    } else {
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int row = m ? 8 + (fr >> 1) : fr;
        const bool act = m ? own2 : true;
        const size_t base = ((size_t)I * BS + row) * C::NR;
#pragma unroll
        for (int ci = 0; ci < C::NC; ++ci) {
          pI[m][ci] = make_double2(0.0, 0.0);
          if (act && a.unit_diag) pI[m][ci] = __ldg(reinterpret_cast<const double2*>(P + base + 2 * ccol(ci)));
        }
      }
    }
    for (int j = jb; j < je; ++j) {
      // keep the ring full: blocks used .. used + NSTG - 1 (this row's or later rows'); the stage of
      // block used - 1 was released by the __syncwarp that ended its multiplication
      while (Ip < nb && issued < used + C::NSTG) issue(issued++);
      const int st = (int)(used % C::NSTG);
      mbar_wait(bars + st, (used / C::NSTG) & 1);
      ++used;
      const double* bs = wbuf + (size_t)st * C::STAGE;
      const double* ps = bs + C::ABLK;
#pragma unroll
      for (int ks = 0; ks < 3; ++ks) {
        const int k = ks * 4 + fk;
        const double2 a01 = *reinterpret_cast<const double2*>(bs + (fr * BS + k) * 2);
        const double a2 = bs[((8 + (fr >> 1)) * BS + k) * 2 + (fr & 1)];
#pragma unroll
        for (int jn = 0; jn < C::NP; ++jn) {
          const double2 b = *reinterpret_cast<const double2*>(ps + k * C::PST + 16 * jn + 2 * fr);
          dmma(accP[0][jn][0], a01.x, b.x);
          dmma(accP[0][jn][1], a01.x, b.y);
          dmma(accP[1][jn][0], a01.y, b.x);
          dmma(accP[1][jn][1], a01.y, b.y);
          dmma(accP[2][jn][0], a2, b.x);
          dmma(accP[2][jn][1], a2, b.y);
        }
        if (C::NS) {
          const double b = ps[k * C::PST + 16 * C::NP + fr];
          dmma(accS[0], a01.x, b);
          dmma(accS[1], a01.y, b);
          dmma(accS[2], a2, b);
        }
      }
      __syncwarp();  // this stage is refilled by the next issue
    }
    // combine: q[m][ci] = (Q_r, Q_i) of row (m ? 8 + fr/2 : fr), complex column ccol(ci)
    double2 q[2][C::NC];
#pragma unroll
    for (int ci = 0; ci < C::NC; ++ci) {
      double x0, y0_, x1, y1, x2, y2;  // (B P_r, B P_i) of M tiles 0 (B_r), 1 (B_i), 2 (mixed)
      if (ci < 2 * C::NP) {
        const int jn = ci >> 1, e = ci & 1;
        x0 = accP[0][jn][0][e]; y0_ = accP[0][jn][1][e];
        x1 = accP[1][jn][0][e]; y1 = accP[1][jn][1][e];
        x2 = accP[2][jn][0][e]; y2 = accP[2][jn][1][e];
      } else {
        x0 = accS[0][0]; y0_ = accS[0][1];
        x1 = accS[1][0]; y1 = accS[1][1];
        x2 = accS[2][0]; y2 = accS[2][1];
      }
      q[0][ci] = make_double2(x0 - y1, y0_ + x1);
      const double xo = __shfl_xor_sync(0xffffffffu, x2, 4), yo = __shfl_xor_sync(0xffffffffu, y2, 4);
      q[1][ci] = make_double2(x2 - yo, y2 + xo);  // meaningful in the even-fr lanes (B_r there, B_i in lane ^ 4)
    }
    if constexpr (C::ESTG) mbar_wait(ebar, rows_done & 1);
    ++rows_done;
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int row = m ? 8 + (fr >> 1) : fr;
      if (m && !own2) continue;
      const size_t base = ((size_t)I * BS + row) * C::NR;
#pragma unroll
      for (int ci = 0; ci < C::NC; ++ci) {
        const int col = 2 * ccol(ci);
        double2 v = q[m][ci];
        if (a.unit_diag) {
          const double2 pi = C::ESTG ? *reinterpret_cast<const double2*>(ebuf + row * C::NR + col) : pI[m][C::ESTG ? 0 : ci];
          v.x += pi.x;
          v.y += pi.y;
        }
        *reinterpret_cast<double2*>(Q + base + col) = v;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int md = rmode[r];
          if (md == RED_NONE) continue;
          if (md == RED_NORM2 || md == RED_COLNORM2) {
            const double q2 = v.x * v.x + v.y * v.y;
            if (md == RED_NORM2) rs[r].x += q2;
            else rc[r][ci].x += q2;
          } else {
            double2 y;
            if (C::ESTG && r == 0)
              y = *reinterpret_cast<const double2*>(ebuf + BS * C::NR + (md == RED_SUMVEC ? 2 * row : row * C::NR + col));
            else
              y = md == RED_SUMVEC ? __ldg(reinterpret_cast<const double2*>(ry[r]) + (size_t)I * BS + row)
                                   : __ldg(reinterpret_cast<const double2*>(ry[r] + base + col));
            const double2 pr = make_double2(y.x * v.x + y.y * v.y, y.x * v.y - y.y * v.x);
            if (md == RED_DIAG) {
              rc[r][ci].x += pr.x;
              rc[r][ci].y += pr.y;
            } else {
              rs[r].x += pr.x;
              rs[r].y += pr.y;
            }
          }
        }
      }
    }
    if constexpr (C::ESTG) __syncwarp();  // the epilogue buffer is rewritten by the next row's request
  }
  if (nred == 0) return;
  __syncthreads();  // every warp is done with its staging buffers
  double* red_sm = bsm;  // [warp][len] doubles
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (r >= nred) break;
    const int md = rmode[r];
    const int len = red_len(md, S, true);
    double* w = red_sm + (size_t)warp * len;
    if (md == RED_DIAG || md == RED_COLNORM2) {
#pragma unroll
      for (int ci = 0; ci < C::NC; ++ci) {
        double2 v = rc[r][ci];
#pragma unroll
        for (int m = 4; m < 32; m <<= 1) {  // over fr: lanes with equal fk own the same columns
          v.x += __shfl_xor_sync(0xffffffffu, v.x, m);
          v.y += __shfl_xor_sync(0xffffffffu, v.y, m);
        }
        if (fr == 0) {
          const int c = ccol(ci);
          if (md == RED_DIAG) {
            w[2 * c] = v.x;
            w[2 * c + 1] = v.y;
          } else {
            w[c] = v.x;
          }
        }
      }
    } else {
      double2 v = rs[r];
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, m);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, m);
      }
      if (lane == 0) {
        w[0] = v.x;
        if (md != RED_NORM2) w[1] = v.y;
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
      double acc = 0.0;
      for (int qq = 0; qq < C::WARPS; ++qq) acc += red_sm[qq * len + j];
      a.partials[(size_t)blockIdx.x * a.pstride + a.red[r].poff + j] = acc;
    }
    __syncthreads();
  }
}

template <int S, int NWARP, int NSTAGE, bool EST, bool PAD = true>
int launch_k2(const BsrArgs& a, int grid, cudaStream_t st) {
  using C2 = B2Cfg<S, NWARP, NSTAGE, EST, PAD>;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(bsr12_kernel2<S, NWARP, NSTAGE, EST, PAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C2::SMEM);
  if (grid < 0) {  // resident warps per SM
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bsr12_kernel2<S, NWARP, NSTAGE, EST, PAD>, 32 * NWARP, C2::SMEM);
    return occ * NWARP;
  }
  bsr12_kernel2<S, NWARP, NSTAGE, EST, PAD><<<grid, 32 * NWARP, C2::SMEM, st>>>(a);
  return (int)cudaGetLastError();
}

// launch configuration of the M = 24 form: (warps per CTA, ring stages per warp, epilogue staging).
// SRK_BSR_CFG selects one for measurements (scripts/bsr_probe.py); read per launch.
static int bsr_cfg() {
  const char* e = getenv("SRK_BSR_CFG");
  return e ? atoi(e) : BSR_CFG_DEFAULT;
}

template <int S>
int launch_s(const BsrArgs& a, int grid, cudaStream_t st) {
  using C = BCfg<S>;
  const bool old = getenv("SRK_BSR_OLD") != nullptr;  // A/B switch (read per launch): the padded [B_r B_i] * lift(P) form
  if (old) {
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr)) cudaFuncSetAttribute(bsr12_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (grid < 0) {
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bsr12_kernel<S>, 256, C::SMEM);
      return occ * 8;
    }
    bsr12_kernel<S><<<grid, 256, C::SMEM, st>>>(a);
    return (int)cudaGetLastError();
  }
  switch (bsr_cfg()) {
    case 1: return launch_k2<S, 8, 2, false, false>(a, grid, st);  // one P copy per block (unpadded)
    case 2: return launch_k2<S, 6, 2, true, true>(a, grid, st);
    case 3: return launch_k2<S, 6, 2, true, false>(a, grid, st);
    case 4: return launch_k2<S, 6, 3, false, false>(a, grid, st);
    case 5: return launch_k2<S, 4, 4, true, true>(a, grid, st);     // fewer warps, deeper ring (measured slower)
    default: return launch_k2<S, 8, 2, false, true>(a, grid, st);
  }
}

}  // namespace

// warps per CTA of the configuration a launch will use (the engine sizes the grid with it)
int bsr_warps_per_cta() {
  if (getenv("SRK_BSR_OLD")) return 8;
  switch (bsr_cfg()) {
    case 2: case 3: case 4: return 6;
    case 5: return 4;
    default: return 8;
  }
}

bool bsr_supported(int bs, bool cplx, int s) { return bs == BS && cplx && (s == 4 || s == 8 || s == 12 || s == 16); }

// grid < 0: returns the resident CTAs per SM
int launch_bsr(const BsrArgs& a, int s, int grid, cudaStream_t st) {
  switch (s) {
    case 4: return launch_s<4>(a, grid, st);
    case 8: return launch_s<8>(a, grid, st);
    case 12: return launch_s<12>(a, grid, st);
    case 16: return launch_s<16>(a, grid, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace srk
