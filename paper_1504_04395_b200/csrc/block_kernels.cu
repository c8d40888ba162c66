// block_kernels.cu — fixed-order second-stage reduction and the dtype dispatch
// of the hot-path kernels (templates in block_kernels.cuh).
#include "kernels.cuh"

namespace srk {

// ============================================================================
// Deterministic second stage: ws[woff + j] = sum_b partials[b*pstride + poff + j]
// One warp per output value; lanes stride over CTAs; fixed xor tree.
// ============================================================================
__global__ void fin_kernel(FinArgs a) {
  if (a.done && *a.done) return;
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int j = wid;
  for (int q = 0; q < a.nseg; ++q) {
    if (j < a.seg[q].len) {
      double acc = 0.0;
      for (int b = lane; b < a.nblk; b += 32) acc += a.partials[(size_t)b * a.pstride + a.seg[q].poff + j];
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
      if (lane == 0) a.ws[a.seg[q].woff + j] = acc;
      return;
    }
    j -= a.seg[q].len;
  }
}

// ============================================================================
// dispatch
// ============================================================================
int launch_spmm_f64(int cap, bool full, const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st);
int launch_spmm_c128(int cap, bool full, const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st);
int launch_upd_f64(int cap, bool full, const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st);
int launch_upd_c128(int cap, bool full, const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st);

__host__ __device__ constexpr int pow2c(int x) { return x <= 1 ? 1 : 2 * pow2c((x + 1) / 2); }

int cap_for(int s) {
  // (2: an exact-width instance for s = 2 — the team-per-row kernel with 16-byte P rows,
  // config 5's s = 2 ran 3x slower than s = 1 on the generic width-4 instance)
  const int caps[] = {1, 2, 4, 8, 12, 16, 32, 64};
  for (int c : caps)
    if (s <= c) return c;
  return -1;
}

// rows handled by one 256-thread CTA per grid-stride step (one row per lane group)
int rows_per_cta(int cap, bool cplx) {
  int esz = cplx ? 16 : 8;
  int epc = (esz == 16) ? 1 : ((cap % 2 == 0) ? 2 : 1);
  int nch = (cap + epc - 1) / epc;
  int G = pow2c(nch);
  if (G > 32) G = 32;
  return 8 * (32 / G);
}

int launch_spmm(bool cplx, int cap, bool full, const SpmmArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  return cplx ? launch_spmm_c128(cap, full, a, grid, block, smem, st) : launch_spmm_f64(cap, full, a, grid, block, smem, st);
}

int launch_upd(bool cplx, int cap, bool full, const UpdArgs& a, int grid, int block, size_t smem, cudaStream_t st) {
  return cplx ? launch_upd_c128(cap, full, a, grid, block, smem, st) : launch_upd_f64(cap, full, a, grid, block, smem, st);
}

// block-method instances (s x s coefficients) up to capacity 32; the in-kernel s x s
// Gram up to 16 (wider ones are routed to the tensor-core Gram by the engine)
bool full_supported(bool cplx, int cap) { (void)cplx; return cap <= 32; }
bool full_red_supported(bool cplx, int cap) { (void)cplx; return cap <= 16; }

int padded_width(int cap, bool cplx) {
  const int esz = cplx ? 16 : 8;
  const int epc = (esz == 16) ? 1 : ((cap % 2 == 0) ? 2 : 1);
  const int nch = (cap + epc - 1) / epc;
  int G = pow2c(nch);
  if (G > 32) G = 32;
  const int cpl = (nch + G - 1) / G;
  return G * epc * cpl;
}

int launch_fin(const FinArgs& a, cudaStream_t st) {
  int total = 0;
  for (int q = 0; q < a.nseg; ++q) total += a.seg[q].len;
  if (total == 0) return 0;
  const int warps_per_cta = 8;
  int grid = (total + warps_per_cta - 1) / warps_per_cta;
  fin_kernel<<<grid, warps_per_cta * 32, 0, st>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace srk
