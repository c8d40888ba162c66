// tma_probe.cu — checks the sm_100a TMA primitives used by spmm_tma.cuh in
// isolation (gather4 of 4 rows of a 2D FP64 tensor; 1D bulk copy), printing the
// first words landed in shared memory. Tuning aid only.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>

#include "spmm_tma.cuh"  // scripts/ (experiment, not part of the library)

using namespace srk;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void probe(const __grid_constant__ TmaDesc map, const double* src, double* out, int mode) {
  __shared__ __align__(128) double buf[4 * 16];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode == 0) {
      mbar_expect_tx_arrive(&bar, 4 * 16 * 8);
      tma_gather4(buf, &map, 0, 5, 2, 9, 0, &bar);
    } else {
      mbar_expect_tx_arrive(&bar, 4 * 16 * 8);
      bulk_g2s(buf, src + 32, 4 * 16 * 8, &bar);
    }
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int boxrows = argc > 1 ? atoi(argv[1]) : 1;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;
  const int n = 16, s = 16;
  double h[n * s];
  for (int i = 0; i < n * s; ++i) h[i] = i;
  double *P, *out;
  CK(cudaMalloc(&P, sizeof(h)));
  CK(cudaMalloc(&out, 64 * 8));
  CK(cudaMemcpy(P, h, sizeof(h), cudaMemcpyHostToDevice));
  TmaDesc d;
  cuuint64_t dims[2] = {(cuuint64_t)s, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)s * 8};
  cuuint32_t box[2] = {(cuuint32_t)s, (cuuint32_t)boxrows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(reinterpret_cast<CUtensorMap*>(&d), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P, dims, strides, box,
                                      es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode boxrows=%d mode=%d: %d\n", boxrows, mode, (int)r);
  probe<<<1, 32>>>(d, P, out, mode);
  CK(cudaDeviceSynchronize());
  double o[64];
  CK(cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost));
  for (int rr = 0; rr < 4; ++rr) printf("row %d: %g %g ... %g\n", rr, o[rr * 16], o[rr * 16 + 1], o[rr * 16 + 15]);
  return 0;
}
