// blk_mma.cu — the block methods' updates with s x s coefficients on the FP64
// tensor cores (the Bl updates "represent
// BLAS3 GEMM operations"). out_o = sum_t src_t * C_ot with every coefficient lifted
// to a W x W real matrix in shared memory (ONE / SCALAR / DIAG as multiples of the
// identity or diagonal, s x s as given, transposed-conjugated or conjugated as asked;
// complex blocks through the interleaved real lift
//   [x_re x_im] * [[C_re, C_im], [-C_im, C_re]]  on column pairs (2k, 2k+1)),
// then per warp 8-row tiles as m8n8k4 DMMAs: A fragments straight from the input
// rows (or, for a chained output, shuffled out of its accumulators), B fragments
// from the staged coefficient. All outputs of a tile are formed before any is
// stored (in-place updates are safe). The norm / trace / diagonal / vector-sum
// reductions are accumulated in the accumulator layout; s x s Grams are left to the
// tensor-core Gram kernel by the engine.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"

namespace srk {

namespace {

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// stage = nin consecutive 8-row tiles (one per input, 8 w doubles each, contiguous in the
// row-major blocks) copied by the bulk-copy engine; completion counted on the stage's mbarrier
__device__ __forceinline__ void issue_stage(const UpdArgs& a, int nin, int w, long long tile, double* dst,
                                            unsigned long long* bar) {
  const unsigned bytes = (unsigned)(8 * w * 8);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes * nin)
               : "memory");
  for (int b = 0; b < nin; ++b)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst + (size_t)b * 8 * w)),
                 "l"(reinterpret_cast<const double*>(a.in[b]) + (size_t)tile * 8 * w), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

template <int W>
__global__ void __launch_bounds__(256, 2) upd_mma_kernel(UpdArgs a, int cplx, int nterm, int stg) {
  if (a.done && *a.done) return;
  constexpr int NT = W / 8;   // 8-column tiles
  extern __shared__ __align__(16) double msm[];
  __shared__ int tslot[MAX_OUT][MAX_SRC];
  const int s = a.s;
  const int w = cplx ? 2 * s : s;  // real row width
  const bool vec2 = (w & 1) == 0;  // 16-byte row segments
  const long long n = a.n;
  const int nout = a.nout, nin = a.nin, nred = a.nred;
  // a.cslot[o][src] holds the term's staged-matrix index (-1: absent term)
  if (threadIdx.x < MAX_OUT * MAX_SRC)
    tslot[threadIdx.x / MAX_SRC][threadIdx.x % MAX_SRC] = a.cslot[threadIdx.x / MAX_SRC][threadIdx.x % MAX_SRC];
  __syncthreads();
  // ---- stage every term as a W x W real matrix (row k = input column, col c = output column)
  for (int t = 0; t < nterm; ++t) {
    int o = 0, src = 0;
    for (int q = 0; q < MAX_OUT * MAX_SRC; ++q)
      if (tslot[q / MAX_SRC][q % MAX_SRC] == t) {
        o = q / MAX_SRC;
        src = q % MAX_SRC;
      }
    const Coef cf = a.cf[o][src];
    double* M = msm + (size_t)t * W * W;  // stored transposed: M[c * W + k]
    for (int idx = threadIdx.x; idx < W * W; idx += blockDim.x) {
      const int c = idx / W, k = idx % W;
      double v = 0.0;
      if (k < w && c < w) {
        const int kk = cplx ? k / 2 : k, cc = cplx ? c / 2 : c;  // complex element indices
        // complex value of the coefficient at (kk, cc)
        double re = 0.0, im = 0.0;
        if (cf.kind == CK_ONE) {
          re = (kk == cc) ? 1.0 : 0.0;
        } else if (cf.kind == CK_SCALAR) {
          if (kk == cc) {
            re = a.ws[cf.off];
            im = cplx ? a.ws[cf.off + 1] : 0.0;
          }
        } else if (cf.kind == CK_DIAG) {
          if (kk == cc) {
            re = a.ws[cf.off + (cplx ? 2 * kk : kk)];
            im = cplx ? a.ws[cf.off + 2 * kk + 1] : 0.0;
          }
        } else {  // CK_FULL: out[c] += x[k] M[k][c] (herm: M^H)
          const int r0 = cf.herm ? cc : kk, c0 = cf.herm ? kk : cc;
          const size_t e = (size_t)r0 * s + c0;
          re = cplx ? a.ws[cf.off + 2 * e] : a.ws[cf.off + e];
          im = cplx ? a.ws[cf.off + 2 * e + 1] : 0.0;
          if (cf.herm) im = -im;
        }
        if (cf.conj) im = -im;
        if (cf.neg) {
          re = -re;
          im = -im;
        }
        if (!cplx) {
          v = re;
        } else {
          const int tk = k & 1, tc = c & 1;  // real lift: [[re, im], [-im, re]] on (k, c) pairs
          v = (tk == 0) ? (tc == 0 ? re : im) : (tc == 0 ? -im : re);
        }
      }
      M[idx] = v;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const long long ntile = (n + 7) / 8;
  const long long nfull = n / 8;  // tiles with 8 live rows: the ones staged by bulk copies
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  // per-warp ring of stg stages (stg = 0: inputs read straight from global memory)
  const size_t stage_len = (size_t)nin * 8 * w;
  double* ring = msm + (size_t)nterm * W * W + (size_t)warp * stg * stage_len;
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(msm + (size_t)nterm * W * W + (size_t)(blockDim.x >> 5) * stg * stage_len) +
      warp * stg;
  const long long first = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  if (stg && lane == 0) {
    for (int q = 0; q < stg; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bars + q)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (stg && lane == 0)
    for (int q = 0; q < stg; ++q) {
      const long long t = first + q * nwarps;
      if (t < nfull) issue_stage(a, nin, w, t, ring + q * stage_len, bars + q);
    }
  // reduction accumulators (per lane): scalar modes in rs, per-column modes in rc[nt][pair]
  int rmode[MAX_RED], rx[MAX_RED], ry[MAX_RED];
#pragma unroll
  for (int r = 0; r < MAX_RED; ++r) {
    rmode[r] = r < nred ? a.red[r].mode : RED_NONE;
    rx[r] = r < nred ? a.red[r].xsrc : -2;
    ry[r] = r < nred ? a.red[r].ysrc : -2;
  }
  double rs[MAX_RED][2];
  double rc[MAX_RED][NT][2];
#pragma unroll
  for (int r = 0; r < MAX_RED; ++r) {
    rs[r][0] = rs[r][1] = 0.0;
#pragma unroll
    for (int t = 0; t < NT; ++t) rc[r][t][0] = rc[r][t][1] = 0.0;
  }

  long long k = 0;
  for (long long tile = first; tile < ntile; tile += nwarps, ++k) {
    const long long row = tile * 8 + fr;  // this lane's A-fragment and accumulator row
    const bool live = row < n;
    const bool piped = stg && tile < nfull;
    const int stage = piped ? (int)(k % stg) : 0;
    if (piped) mbar_wait_parity(bars + stage, (unsigned)((k / stg) & 1));
    // input b's row for this lane: the staged tile, or global memory
    auto in_row = [&](int b) -> const double* {
      return piped ? ring + stage * stage_len + (size_t)b * 8 * w + (size_t)fr * w
                   : reinterpret_cast<const double*>(a.in[b]) + (size_t)row * w;
    };
    double acc[MAX_OUT][NT][2];
#pragma unroll
    for (int o = 0; o < MAX_OUT; ++o) {
#pragma unroll
      for (int t = 0; t < NT; ++t) acc[o][t][0] = acc[o][t][1] = 0.0;
      if (o < nout) {
        // inputs
#pragma unroll
        for (int b = 0; b < MAX_IN; ++b) {
          const int ts = b < nin ? tslot[o][b] : -1;
          if (ts < 0) continue;
          const double* X = in_row(b);
          const double* M = msm + (size_t)ts * W * W;
          // k order permuted within each 8-column group: k-steps 2j, 2j+1 take, for lane
          // fk, the columns 8j + 2fk and 8j + 2fk + 1 (one 16-byte load of A, one of B)
          double2 av[NT];
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const int col = j * 8 + 2 * fk;
            if (vec2) {
              av[j] = (live && col < w) ? *reinterpret_cast<const double2*>(X + col) : make_double2(0.0, 0.0);
            } else {
              av[j].x = (live && col < w) ? X[col] : 0.0;
              av[j].y = (live && col + 1 < w) ? X[col + 1] : 0.0;
            }
          }
          // consecutive DMMAs go to different accumulators (NT independent chains)
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            double2 bv[NT];
#pragma unroll
            for (int t = 0; t < NT; ++t) bv[t] = *reinterpret_cast<const double2*>(M + (t * 8 + fr) * W + j * 8 + 2 * fk);
#pragma unroll
            for (int t = 0; t < NT; ++t) dmma(acc[o][t], av[j].x, bv[t].x);
#pragma unroll
            for (int t = 0; t < NT; ++t) dmma(acc[o][t], av[j].y, bv[t].y);
          }
        }
        // earlier outputs of this tile (C fragment -> A fragment by shuffles)
#pragma unroll
        for (int p = 0; p < MAX_OUT; ++p) {
          if (p >= o) break;
          const int ts = tslot[o][MAX_IN + p];
          if (ts < 0) continue;
          const double* M = msm + (size_t)ts * W * W;
          // with the permuted k order the A values of an earlier output are this lane's
          // own accumulator entries (columns 8j + 2fk, 8j + 2fk + 1): no shuffles
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            double2 bv[NT];
#pragma unroll
            for (int tt = 0; tt < NT; ++tt) bv[tt] = *reinterpret_cast<const double2*>(M + (tt * 8 + fr) * W + j * 8 + 2 * fk);
#pragma unroll
            for (int tt = 0; tt < NT; ++tt) dmma(acc[o][tt], acc[p][j][0], bv[tt].x);
#pragma unroll
            for (int tt = 0; tt < NT; ++tt) dmma(acc[o][tt], acc[p][j][1], bv[tt].y);
          }
        }
      }
    }
    // ---- store every output, then the reductions (inputs were all read above)
#pragma unroll
    for (int o = 0; o < MAX_OUT; ++o) {
      if (o >= nout || !a.out[o] || !live) continue;
      double* Y = reinterpret_cast<double*>(a.out[o]);
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int col = t * 8 + 2 * fk;
        if (col + 1 < w && (w & 1) == 0) {
          *reinterpret_cast<double2*>(Y + (size_t)row * w + col) = make_double2(acc[o][t][0], acc[o][t][1]);
        } else {
          if (col < w) Y[(size_t)row * w + col] = acc[o][t][0];
          if (col + 1 < w) Y[(size_t)row * w + col + 1] = acc[o][t][1];
        }
      }
    }
    if (nred && live) {
#pragma unroll
      for (int r = 0; r < MAX_RED; ++r) {
        const int md = rmode[r];
        if (md == RED_NONE) continue;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int col = t * 8 + 2 * fk;
          if (col >= w) continue;
          // x values at (row, col), (row, col + 1)
          double x0 = 0.0, x1 = 0.0;
          if (rx[r] >= SRC_OUT) {
#pragma unroll
            for (int o = 0; o < MAX_OUT; ++o)
              if (rx[r] == SRC_OUT + o) {
                x0 = acc[o][t][0];
                x1 = acc[o][t][1];
              }
          } else {
            const double* X = in_row(rx[r]);
            x0 = X[col];
            x1 = col + 1 < w ? X[col + 1] : 0.0;
          }
          if (md == RED_NORM2 || md == RED_COLNORM2) {
            const double q = x0 * x0 + x1 * x1;
            if (md == RED_NORM2) rs[r][0] += q;
            else if (cplx) rc[r][t][0] += q;  // one complex column per pair
            else {
              rc[r][t][0] += x0 * x0;
              rc[r][t][1] += x1 * x1;
            }
            continue;
          }
          double y0 = 0.0, y1 = 0.0;
          if (md == RED_SUMVEC) {
            const double* yv = reinterpret_cast<const double*>(a.red[r].yext);
            if (cplx) {
              y0 = yv[2 * row];
              y1 = yv[2 * row + 1];
            } else {
              y0 = y1 = yv[row];
            }
          } else if (ry[r] >= SRC_OUT) {
#pragma unroll
            for (int o = 0; o < MAX_OUT; ++o)
              if (ry[r] == SRC_OUT + o) {
                y0 = acc[o][t][0];
                y1 = acc[o][t][1];
              }
          } else {
            const double* Yp = ry[r] >= 0 ? in_row(ry[r]) : reinterpret_cast<const double*>(a.red[r].yext) + (size_t)row * w;
            y0 = Yp[col];
            y1 = col + 1 < w ? Yp[col + 1] : 0.0;
          }
          // conj(y) * x
          double pr, pi;
          if (cplx) {
            pr = y0 * x0 + y1 * x1;
            pi = y0 * x1 - y1 * x0;
            if (md == RED_DIAG) {
              rc[r][t][0] += pr;
              rc[r][t][1] += pi;
            } else {
              rs[r][0] += pr;
              rs[r][1] += pi;
            }
          } else {
            if (md == RED_DIAG) {
              rc[r][t][0] += y0 * x0;
              rc[r][t][1] += y1 * x1;
            } else {
              rs[r][0] += y0 * x0 + y1 * x1;
            }
          }
        }
      }
    }
    if (piped) {
      __syncwarp();  // every lane's reads of this stage are done
      const long long nt = tile + (long long)stg * nwarps;
      if (lane == 0 && nt < nfull) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_stage(a, nin, w, nt, ring + stage * stage_len, bars + stage);
      }
    }
  }
  if (nred == 0) return;
  // ---- CTA partials in the red_len layout: warp butterflies, then warps in order
  __syncthreads();
  double* rsm = msm;  // the staged coefficients are no longer needed
#pragma unroll
  for (int r = 0; r < MAX_RED; ++r) {
    if (r >= nred) break;
    const int md = rmode[r];
    const int len = red_len(md, s, cplx);
    double* wv = rsm + (size_t)warp * len;
    if (md == RED_DIAG || md == RED_COLNORM2) {
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        double v0 = rc[r][t][0], v1 = rc[r][t][1];
#pragma unroll
        for (int m = 4; m < 32; m <<= 1) {  // over fr: lanes with equal fk hold the same columns
          v0 += __shfl_xor_sync(0xffffffffu, v0, m);
          v1 += __shfl_xor_sync(0xffffffffu, v1, m);
        }
        if (fr == 0) {
          const int col = t * 8 + 2 * fk;
          if (cplx) {
            const int c = col / 2;
            if (c < s) {
              if (md == RED_DIAG) {
                wv[2 * c] = v0;
                wv[2 * c + 1] = v1;
              } else {
                wv[c] = v0;
              }
            }
          } else {
            if (col < s) wv[col] = v0;
            if (col + 1 < s) wv[col + 1] = v1;
          }
        }
      }
    } else {
      double v0 = rs[r][0], v1 = rs[r][1];
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, m);
        v1 += __shfl_xor_sync(0xffffffffu, v1, m);
      }
      if (lane == 0) {
        wv[0] = v0;
        if (len > 1) wv[1] = v1;
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
      double acc = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) acc += rsm[q * len + j];
      a.partials[(size_t)blockIdx.x * a.pstride + a.red[r].poff + j] = acc;
    }
    __syncthreads();
  }
}

// stages of the per-warp input ring: as many as fit (up to 4) in half an SM's shared
// memory, so that two CTAs stay resident; 0 (direct global loads) when fewer than 2 fit
// or an input is not 16-byte aligned (bulk-copy requirement). SRK_UPD_STAGES overrides.
int pick_stages(const UpdArgs& a, int w, int W, int nterm) {
  if (a.nin == 0) return 0;
  for (int b = 0; b < a.nin; ++b)
    if (reinterpret_cast<uintptr_t>(a.in[b]) & 15) return 0;
  static int env = [] {
    const char* e = getenv("SRK_UPD_STAGES");
    return e ? atoi(e) : -1;
  }();
  const size_t per = (size_t)8 * a.nin * 8 * w * 8 + 8;  // 8 warps, one stage each, + mbarrier
  const size_t budget = 110 * 1024 - (size_t)nterm * W * W * 8;
  int stg = (int)std::min<size_t>(4, budget / per);
  if (env >= 0) stg = env;
  return stg >= 2 ? stg : 0;
}

size_t smem_bytes(int W, int w, int nterm, int nin, int stg) {
  const size_t pipe = (size_t)nterm * W * W * 8 + (size_t)8 * stg * ((size_t)nin * 8 * w * 8 + 8);
  return std::max<size_t>(pipe, (size_t)8 * 2 * 64 * 8);
}

template <int W>
int launch_w(const UpdArgs& a, int cplx, int nterm, int grid, cudaStream_t st) {
  const int w = a.s * (cplx ? 2 : 1);
  const int stg = pick_stages(a, w, W, nterm);
  const size_t smem = smem_bytes(W, w, nterm, a.nin, stg);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(upd_mma_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  if (grid < 0) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, upd_mma_kernel<W>, 256, smem);
    return occ;
  }
  upd_mma_kernel<W><<<grid, 256, smem, st>>>(a, cplx, nterm, stg);
  return (int)cudaGetLastError();
}

}  // namespace

// real row width w = s (or 2s complex) <= 32; a.cslot[o][src] = the term's index in
// [0, nterm) or -1; grid < 0 -> resident CTAs per SM
int upd_mma_width(int w) { return w <= 8 ? 8 : (w <= 16 ? 16 : (w <= 32 ? 32 : 0)); }
size_t upd_mma_smem(int w, int nterm) {
  const int W = upd_mma_width(w);
  return std::max<size_t>((size_t)nterm * W * W * 8, (size_t)8 * 2 * 64 * 8);
}
int launch_upd_mma(const UpdArgs& a, bool cplx, int nterm, int grid, cudaStream_t st) {
  const int w = a.s * (cplx ? 2 : 1);
  switch (upd_mma_width(w)) {
    case 8: return launch_w<8>(a, cplx, nterm, grid, st);
    case 16: return launch_w<16>(a, cplx, nterm, grid, st);
    case 32: return launch_w<32>(a, cplx, nterm, grid, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace srk
